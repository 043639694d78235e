// gridbar_bench.cu -- cost of a grid-wide barrier among 148 persistent CTAs
// (one per SM) on sm_100a, several arrival/poll flavours.  Each CTA runs N
// barriers back to back; thread 0 arrives/polls, the CTA joins with
// __syncthreads.  Reports ns per barrier and the exit spread (max - min
// exit time over CTAs of one barrier, from %globaltimer).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridbar_bench tools/gridbar_bench.cu
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int MODE>
__global__ void bar_kernel(unsigned long long *bar, unsigned long long *flags, int n,
                           unsigned long long *exits /* [n][G] */) {
  const uint32_t G = gridDim.x, b = blockIdx.x;
  for (int i = 0; i < n; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long target = (unsigned long long)(i + 1) * G;
      if (MODE == 0) {  // fence + atomicAdd + ld.acquire spin (current)
        __threadfence();
        atomicAdd(bar, 1ull);
        unsigned long long v;
        do {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
        } while (v < target);
      } else if (MODE == 1) {  // red.release + ld.acquire spin
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        unsigned long long v;
        do {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
        } while (v < target);
      } else if (MODE == 2) {  // red.release + relaxed spin + fence.acquire
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        unsigned long long v;
        do {
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
        } while (v < target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (MODE == 3) {  // per-CTA flags, CTA 0 gathers then broadcasts
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + 16 * b), "l"((unsigned long long)(i + 1)) : "memory");
        if (b == 0) {
          for (uint32_t c = 0; c < G; ++c) {
            unsigned long long v;
            do {
              asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + 16 * c) : "memory");
            } while (v < (unsigned long long)(i + 1));
          }
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(bar), "l"((unsigned long long)(i + 1)) : "memory");
        }
        unsigned long long v;
        do {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
        } while (v < (unsigned long long)(i + 1));
      } else if (MODE == 4) {  // atom.add.release (returning) + acquire spin, no separate fence
        unsigned long long old;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(bar) : "memory");
        unsigned long long v = old + 1;
        while (v < target)
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
      }
      exits[(size_t)i * G + b] = gt();
    }
    __syncthreads();
  }
}

template <int MODE>
void run(const char *name, int G) {
  const int n = 200;
  unsigned long long *bar, *flags, *exits;
  cudaMalloc(&bar, 8);
  cudaMalloc(&flags, 8 * 16 * G);
  cudaMalloc(&exits, 8ull * n * G);
  cudaMemset(bar, 0, 8);
  cudaMemset(flags, 0, 8 * 16 * G);
  void *args[] = {&bar, &flags, (void *)&n, &exits};
  cudaEvent_t a, c;
  cudaEventCreate(&a);
  cudaEventCreate(&c);
  // warm
  cudaLaunchCooperativeKernel((void *)bar_kernel<MODE>, G, 256, args, 0, 0);
  cudaDeviceSynchronize();
  cudaMemset(bar, 0, 8);
  cudaMemset(flags, 0, 8 * 16 * G);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void *)bar_kernel<MODE>, G, 256, args, 0, 0);
  cudaEventRecord(c);
  cudaEventSynchronize(c);
  float ms;
  cudaEventElapsedTime(&ms, a, c);
  std::vector<unsigned long long> h((size_t)n * G);
  cudaMemcpy(h.data(), exits, 8ull * n * G, cudaMemcpyDeviceToHost);
  double spread = 0, step = 0;
  for (int i = 10; i < n; ++i) {
    auto lo = *std::min_element(h.begin() + (size_t)i * G, h.begin() + (size_t)(i + 1) * G);
    auto hi = *std::max_element(h.begin() + (size_t)i * G, h.begin() + (size_t)(i + 1) * G);
    auto lop = *std::min_element(h.begin() + (size_t)(i - 1) * G, h.begin() + (size_t)i * G);
    spread += hi - lo;
    step += lo - lop;
  }
  printf("%-44s G=%d: %7.1f ns/barrier (event), %7.1f ns (min-exit to min-exit), exit spread %7.1f ns  err=%s\n",
         name, G, ms * 1e6 / n, step / (n - 10), spread / (n - 10), cudaGetErrorString(cudaGetLastError()));
  cudaFree(bar);
  cudaFree(flags);
  cudaFree(exits);
}

int main() {
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  for (int G : {sm, 74, 8}) {
    run<0>("fence+atomicAdd+ld.acquire spin", G);
    run<1>("red.release+ld.acquire spin", G);
    run<2>("red.release+relaxed spin+fence", G);
    run<3>("flags -> CTA0 gather -> broadcast", G);
    run<4>("atom.add.release + ld.acquire spin", G);
  }
  return 0;
}
