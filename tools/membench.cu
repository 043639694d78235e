// membench.cu -- HBM streaming microbenchmark on B200: how many bytes per SM
// must be in flight, and in what form, to reach the copy roofline?
//   bulk  : one CTA per SM, cp.async.bulk chunks of C bytes into an NS ring
//   ldg   : plain 128-bit loads, U per thread in flight, G CTAs per SM
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/membench tools/membench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <vector>

#include "../paper_2505_05950_b200/csrc/floe_ptx.cuh"

template <int NS>
__global__ void __launch_bounds__(256, 1) bulk_stream(const uint8_t *src, uint64_t bytes,
                                                      uint32_t chunk, uint32_t *sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS];
  const uint64_t per = bytes / gridDim.x;
  const uint8_t *base = src + per * blockIdx.x;
  const uint32_t n = (uint32_t)(per / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
    for (uint32_t i = 0; i < n && i < (uint32_t)NS; ++i) {
      floe_ptx::mbar_arrive_expect_tx(&full[i], chunk);
      floe_ptx::bulk_g2s(smem + (size_t)i * chunk, base + (size_t)i * chunk, chunk, &full[i]);
    }
  }
  __syncthreads();
  uint32_t acc = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t s = i % NS;
    floe_ptx::mbar_wait(&full[s], (i / NS) & 1u);
    const uint4 *p = reinterpret_cast<const uint4 *>(smem + (size_t)s * chunk);
    for (uint32_t k = threadIdx.x; k < chunk / 16; k += 256) acc ^= p[k].x;
    __syncthreads();
    if (threadIdx.x == 0 && i + NS < n) {
      floe_ptx::mbar_arrive_expect_tx(&full[s], chunk);
      floe_ptx::bulk_g2s(smem + (size_t)s * chunk, base + (size_t)(i + NS) * chunk, chunk,
                         &full[s]);
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

// Records of `rec` bytes at scattered offsets (like kept gate|down records),
// ring of NS stages refilled R at a time after a block barrier (K2's shape).
template <int NS, int R>
__global__ void __launch_bounds__(256, 1) bulk_records(const uint8_t *src, const uint32_t *idx,
                                                       uint32_t n_total, uint32_t rec,
                                                       uint32_t *sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS];
  const uint32_t begin = (uint32_t)((uint64_t)n_total * blockIdx.x / gridDim.x);
  const uint32_t end = (uint32_t)((uint64_t)n_total * (blockIdx.x + 1) / gridDim.x);
  const uint32_t n = end - begin;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
    for (uint32_t i = 0; i < n && i < (uint32_t)NS; ++i) {
      floe_ptx::mbar_arrive_expect_tx(&full[i], rec);
      floe_ptx::bulk_g2s(smem + (size_t)i * rec, src + (size_t)idx[begin + i] * rec, rec, &full[i]);
    }
  }
  __syncthreads();
  uint32_t acc = 0;
  for (uint32_t i0 = 0; i0 < n; i0 += R) {
    for (int r = 0; r < R && i0 + r < n; ++r) {
      const uint32_t i = i0 + r, s = i % NS;
      floe_ptx::mbar_wait(&full[s], (i / NS) & 1u);
      const uint4 *p = reinterpret_cast<const uint4 *>(smem + (size_t)s * rec);
      for (uint32_t k = threadIdx.x; k < rec / 16; k += 256) acc ^= p[k].x;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int r = 0; r < R; ++r) {
        const uint32_t i = i0 + r, nx = i + NS;
        if (i < n && nx < n) {
          const uint32_t s = i % NS;
          floe_ptx::mbar_arrive_expect_tx(&full[s], rec);
          floe_ptx::bulk_g2s(smem + (size_t)s * rec, src + (size_t)idx[begin + nx] * rec, rec,
                             &full[s]);
        }
      }
  }
  if (acc == 0x12345678u) *sink = acc;
}

template <int U>
__global__ void ldg_stream(const uint4 *src, uint64_t n16, uint32_t *sink) {
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t j = i + u * stride;
      if (j < n16) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(src + j));
      } else {
        v[u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t bytes = 1ull << 30;  // 1 GiB, far larger than L2
  uint8_t *buf;
  uint32_t *sink;
  cudaMalloc(&buf, bytes + (1 << 20));
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch, uint64_t nbytes) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    return nbytes / (best * 1e-3) / 1e9;
  };
  // bulk ring: chunk x depth
  const uint32_t chunks[] = {4096, 8192, 16384, 32768, 65536};
  for (uint32_t c : chunks) {
    for (int ns : {2, 4, 8, 12}) {
      const uint64_t smem = (uint64_t)ns * c;
      if (smem > 200 * 1024) continue;
      double gbs = 0;
      const uint64_t nb = (bytes / sm / c) * c * sm;
      auto run = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        gbs = timeit([&] { kern<<<sm, 256, smem>>>(buf, nb, c, sink); }, nb);
      };
      if (ns == 2) run(bulk_stream<2>);
      if (ns == 4) run(bulk_stream<4>);
      if (ns == 8) run(bulk_stream<8>);
      if (ns == 12) run(bulk_stream<12>);
      printf("bulk chunk %6u B x %2d stages (%3llu KB/SM in flight): %7.1f GB/s  err=%s\n", c, ns,
             (unsigned long long)(smem / 1024), gbs, cudaGetErrorString(cudaGetLastError()));
    }
  }
  const uint64_t n16 = bytes / 16;
  for (int ctas : {1, 2, 4, 8}) {
    double g4 = timeit([&] { ldg_stream<4><<<sm * ctas, 256>>>((const uint4 *)buf, n16, sink); }, bytes);
    double g8 = timeit([&] { ldg_stream<8><<<sm * ctas, 256>>>((const uint4 *)buf, n16, sink); }, bytes);
    double g16 = timeit([&] { ldg_stream<16><<<sm * ctas, 256>>>((const uint4 *)buf, n16, sink); }, bytes);
    printf("ldg  %d CTA/SM x 256 thr: U=4 %7.1f  U=8 %7.1f  U=16 %7.1f GB/s\n", ctas, g4, g8, g16);
  }
  // small-footprint reads (like one expert-token: 65 MB) cold from HBM:
  // per-launch time with the L2 flushed (256 MiB memset) before each launch.
  uint8_t *flush;
  cudaMalloc(&flush, 256u << 20);
  int mode = 0;  // 0: dirty flush (memset), 1: clean flush (read), 2: none
  auto cold = [&](auto launch) {
    float tot = 0.0f;
    for (int r = 0; r < 6; ++r) {
      if (mode == 0) cudaMemsetAsync(flush, r, 256u << 20);
      if (mode == 1) ldg_stream<8><<<sm * 2, 256>>>((const uint4 *)flush, (256u << 20) / 16, sink);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r) tot += ms;
    }
    return tot / 5 * 1e3f;  // us
  };
  for (mode = 0; mode < 3; ++mode) {
    printf("---- L2 before each launch: %s\n", mode == 0 ? "dirty (memset 256 MiB)"
                                              : mode == 1 ? "clean (read 256 MiB)" : "no flush");
    const uint32_t c = 16384;
    const uint64_t smem = 8ull * c;
    cudaFuncSetAttribute(bulk_stream<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (uint64_t mb : {4, 16, 33, 65, 94, 164}) {
      const uint64_t nb = ((mb << 20) / sm / c) * c * sm;
      float us_b = cold([&] { bulk_stream<8><<<sm, 256, smem>>>(buf, nb, c, sink); });
      float us_l = cold([&] { ldg_stream<8><<<sm * 2, 256>>>((const uint4 *)buf, nb / 16, sink); });
      printf("cold %4llu MB: bulk16Kx8 %7.2f us (%6.1f GB/s)   ldg2x8 %7.2f us (%6.1f GB/s)\n",
             (unsigned long long)mb, us_b, nb / (us_b * 1e-6) / 1e9, us_l,
             nb / (us_l * 1e-6) / 1e9);
    }
    float us0 = cold([&] { ldg_stream<8><<<sm, 256>>>((const uint4 *)buf, 0, sink); });
    printf("empty launch (cold): %.2f us\n", us0);
  }
  // K2-shaped traffic: 5760 scattered 16 KB records out of 2 x 14336 (94 MB)
  {
    mode = 1;
    const uint32_t rec = 16384, pool = 2 * 14336, n = 5760;
    std::vector<uint32_t> hidx(n);
    uint64_t st = 12345;
    std::vector<uint8_t> used(pool, 0);
    for (uint32_t i = 0; i < n;) {
      st = st * 6364136223846793005ull + 1442695040888963407ull;
      const uint32_t c = (uint32_t)((st >> 33) % pool);
      if (!used[c]) {
        used[c] = 1;
        hidx[i++] = c;
      }
    }
    std::vector<uint32_t> sorted = hidx;
    std::sort(sorted.begin(), sorted.end());
    uint32_t *didx;
    cudaMalloc(&didx, 4ull * n);
    for (int variant = 0; variant < 2; ++variant) {
      cudaMemcpy(didx, variant ? sorted.data() : hidx.data(), 4ull * n, cudaMemcpyHostToDevice);
      auto runk = [&](auto kern, int ns, int r) {
        const uint32_t smem = ns * rec;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float us = cold([&] { kern<<<sm, 256, smem>>>(buf, didx, n, rec, sink); });
        printf("records %s NS=%2d R=%d: %7.2f us (%6.1f GB/s) err=%s\n",
               variant ? "sorted " : "random ", ns, r, us, (double)n * rec / (us * 1e-6) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
      };
      runk(bulk_records<8, 1>, 8, 1);
      runk(bulk_records<8, 4>, 8, 4);
      runk(bulk_records<12, 4>, 12, 4);
      runk(bulk_records<12, 1>, 12, 1);
    }
  }
  return 0;
}
