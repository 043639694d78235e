// tlbbench.cu -- does the phase-C record gather pay for TLB reach?
// 148 CTAs x 39 random 16 KB records (94 MB, the config-2 phase-C volume),
// NS=8 bulk-copy ring, from a pool of P bytes (470 MB = 2 experts' records,
// up to 8 GB = 4 layers' experts), pool touched vs untouched since the last
// launch.  L2 cleaned by a 256 MB read between launches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tlbbench tools/tlbbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2505_05950_b200/csrc/floe_ptx.cuh"

constexpr int NS = 8;
constexpr uint32_t REC = 16384;

__global__ void __launch_bounds__(256, 1) gather(const uint8_t *pool, const uint64_t *idx,
                                                 uint32_t per_cta, uint32_t *sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS];
  const uint64_t *my = idx + (uint64_t)blockIdx.x * per_cta;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
    for (uint32_t i = 0; i < per_cta && i < NS; ++i) {
      floe_ptx::mbar_arrive_expect_tx(&full[i], REC);
      floe_ptx::bulk_g2s(smem + i * REC, pool + my[i] * REC, REC, &full[i]);
    }
  }
  __syncthreads();
  uint32_t acc = 0;
  for (uint32_t i = 0; i < per_cta; ++i) {
    const uint32_t s = i % NS;
    floe_ptx::mbar_wait(&full[s], (i / NS) & 1u);
    acc ^= reinterpret_cast<const uint32_t *>(smem + s * REC)[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0 && i + NS < per_cta) {
      floe_ptx::mbar_arrive_expect_tx(&full[s], REC);
      floe_ptx::bulk_g2s(smem + s * REC, pool + my[i + NS] * REC, REC, &full[s]);
    }
  }
  if (acc == 0x1234567u) *sink = acc;
}

__global__ void touch(const uint4 *p, uint64_t n16, uint32_t *sink) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc ^= p[i].x;
  if (acc == 0x1234567u) *sink = acc;
}

int main() {
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t big = 8ull << 30;
  uint8_t *pool, *flush;
  uint32_t *sink;
  uint64_t *didx;
  cudaMalloc(&pool, big);
  cudaMalloc(&flush, 256ull << 20);
  cudaMalloc(&sink, 4);
  cudaMemset(pool, 1, big);
  const uint32_t per = 39, n = per * sm;
  cudaMalloc(&didx, 8ull * n);
  cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * REC);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  uint64_t st = 88172645463325252ull;
  for (uint64_t pool_mb : {470ull, 2048ull, 8192ull}) {
    const uint64_t nrec = (pool_mb << 20) / REC;
    for (int mode = 0; mode < 2; ++mode) {  // 0: TLB warm (pool just swept), 1: 8 GB swept since
      float tot = 0;
      for (int r = 0; r < 6; ++r) {
        std::vector<uint64_t> h(n);
        for (auto &x : h) {
          st ^= st << 13; st ^= st >> 7; st ^= st << 17;
          x = st % nrec;
        }
        cudaMemcpy(didx, h.data(), 8ull * n, cudaMemcpyHostToDevice);
        if (mode == 0) touch<<<sm * 4, 256>>>((const uint4 *)pool, (pool_mb << 20) / 16, sink);
        else touch<<<sm * 4, 256>>>((const uint4 *)pool, big / 16, sink);
        touch<<<sm * 4, 256>>>((const uint4 *)flush, (256ull << 20) / 16, sink);  // clean L2
        cudaEventRecord(a);
        gather<<<sm, 256, NS * REC>>>(pool, didx, per, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r) tot += ms;
      }
      const float us = tot / 5 * 1e3f;
      printf("pool %5llu MB, %s: %7.2f us  (%6.1f GB/s)  err=%s\n", (unsigned long long)pool_mb,
             mode ? "8 GB swept since (TLB cold)" : "pool swept (TLB warm)     ", us,
             (double)n * REC / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
