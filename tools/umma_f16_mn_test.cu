// umma_f16_mn_test.cu -- validates tcgen05.mma kind::f16 with an MN-major
// (N-contiguous) B operand, SWIZZLE_NONE: D[128 x N] (f32, TMEM) = A[128 x K]
// (f16, K-major) * B[K x N] (f16, N contiguous per k).  Tries the layout /
// descriptor variants and prints mismatches for each.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_f16_mn_test tools/umma_f16_mn_test.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 32, K = 32;  // two K=16 MMAs

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}
// A K-major: (row, k) -> (row%8)*16 + (k%8)*2 + (k/8)*128 + (row/8)*(K/8*128)
__device__ __forceinline__ uint32_t offA(uint32_t r, uint32_t k) {
  return (r % 8) * 16 + (k % 8) * 2 + (k / 8) * 128 + (r / 8) * (K / 8 * 128);
}
// B MN-major: core matrix = 8 k x 8 n (16 B along n); n-cores step cn, k-cores step ck
__device__ __forceinline__ uint32_t offB(uint32_t k, uint32_t n, uint32_t cn, uint32_t ck) {
  return (k % 8) * 16 + (n % 8) * 2 + (n / 8) * cn + (k / 8) * ck;
}

__global__ void kern(const __half *A, const __half *B, float *D, uint32_t cn, uint32_t ck,
                     uint32_t lbo, uint32_t sbo, uint32_t kstep) {
  __shared__ __align__(1024) uint8_t sa[M * K * 2];
  __shared__ __align__(1024) uint8_t sb[K * N * 2 + 4096];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const uint32_t t = threadIdx.x, warp = t / 32, lane = t % 32;
  for (uint32_t i = t; i < M * K; i += blockDim.x)
    *reinterpret_cast<__half *>(sa + offA(i / K, i % K)) = A[i];
  for (uint32_t i = t; i < K * N; i += blockDim.x)
    *reinterpret_cast<__half *>(sb + offB(i / N, i % N, cn, ck)) = B[i];  // B[k][n]
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t dt = tmem_base;
  if (t == 0) {
    // D f32 (1<<4), A f16 (0<<7), B f16 (0<<10), A K-major (bit 15 = 0), B MN-major (bit 16 = 1)
    const uint32_t idesc = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int kb = 0; kb < K / 16; ++kb) {
      const uint64_t da = make_desc(smem_u32(sa) + kb * 256, 128, K / 8 * 128);
      const uint64_t db = make_desc(smem_u32(sb) + kb * kstep, lbo, sbo);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
          "l"(da), "l"(db), "r"(idesc), "r"((uint32_t)kb));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(&mbar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(dt + ((warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < N; ++n) D[(warp * 32 + lane) * N + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(dt));
}

int main() {
  std::vector<__half> A(M * K), B(K * N);
  std::vector<float> Af(M * K), Bf(K * N);
  srand(3);
  for (int i = 0; i < M * K; ++i) { Af[i] = (rand() % 17 - 8) / 8.0f; A[i] = __float2half(Af[i]); }
  for (int i = 0; i < K * N; ++i) { Bf[i] = (rand() % 17 - 8) / 4.0f; B[i] = __float2half(Bf[i]); }
  std::vector<float> ref(M * N, 0.0f);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) ref[m * N + n] += Af[m * K + k] * Bf[k * N + n];
  __half *dA, *dB;
  float *dD;
  cudaMalloc(&dA, 2 * M * K);
  cudaMalloc(&dB, 2 * K * N);
  cudaMalloc(&dD, 4 * M * N);
  cudaMemcpy(dA, A.data(), 2 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 2 * K * N, cudaMemcpyHostToDevice);
  // layout strides (cn = n-core step, ck = k-core step) and descriptor (lbo, sbo), kstep per MMA (16 k = 2 k-cores)
  struct V { uint32_t cn, ck, lbo, sbo, kstep; const char *name; } vs[] = {
      {128, 512, 128, 512, 1024, "n-cores 128, k-cores 512; LBO=n(128) SBO=k(512)"},
      {128, 512, 512, 128, 1024, "n-cores 128, k-cores 512; LBO=k(512) SBO=n(128)"},
      {256, 128, 256, 128, 256, "k-cores 128, n-cores 256; LBO=n(256) SBO=k(128)"},
      {256, 128, 128, 256, 256, "k-cores 128, n-cores 256; LBO=k(128) SBO=n(256)"},
  };
  for (auto &v : vs) {
    cudaMemset(dD, 0, 4 * M * N);
    kern<<<1, 128>>>(dA, dB, dD, v.cn, v.ck, v.lbo, v.sbo, v.kstep);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> got(M * N);
    cudaMemcpy(got.data(), dD, 4 * M * N, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i) bad += fabsf(got[i] - ref[i]) > 1e-3f;
    printf("%-52s err=%s mismatches %d / %d (D[0][0..2] %g %g %g ref %g %g %g)\n", v.name,
           cudaGetErrorString(e), bad, M * N, got[0], got[1], got[2], ref[0], ref[1], ref[2]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
