// mmabench.cu -- per-SM throughput of the legacy warp-level integer MMAs on
// sm_100a (candidates for K1's exact integer dot products):
//   IMMA m16n8k32 s8.s8 -> s32   (512 MACs per warp instruction)
//   IMMA m16n8k64 u4.s4 -> s32   (1024 MACs per warp instruction)
// Each warp runs 8 independent accumulator chains.  Prints MACs/clk/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mmabench tools/mmabench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int ITERS = 2048;

__global__ void k_imma8(int *out, int seed) {
  uint32_t a0 = seed + threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55,
           b1 = a0 ^ 0x33;
  int c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = i + j;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 0x7fffffff) out[0] = s;
}

__global__ void k_imma4(int *out, int seed) {
  uint32_t a0 = seed + threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55,
           b1 = a0 ^ 0x33;
  int c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = i + j;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k64.row.col.s32.u4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 0x7fffffff) out[0] = s;
}

__global__ void k_hmma(int *outi, int seed) {
  uint32_t a0 = seed + threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55,
           b1 = a0 ^ 0x33;
  float c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = i + j;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5f) outi[0] = (int)s;
}

template <typename K>
void bench(const char *name, K kern, double macs_per_inst) {
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void *out;
  cudaMalloc(&out, 4);
  for (int warps : {4, 8, 16, 32}) {
    kern<<<sm, 32 * warps>>>((int *)out, 1);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<sm, 32 * warps>>>((int *)out, 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double insts = (double)sm * warps * ITERS * 8;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-28s warps/SM %2d: %8.1f MACs/clk/SM  (%.2f warp-inst/clk/SM) err=%s\n", name, warps,
           insts * macs_per_inst / cyc / sm, insts / cyc / sm,
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  bench("IMMA m16n8k32 s8", k_imma8, 16.0 * 8 * 32);
  bench("IMMA m16n8k64 u4.s4", k_imma4, 16.0 * 8 * 64);
  bench("HMMA m16n8k16 f16->f32", k_hmma, 16.0 * 8 * 16);
  return 0;
}
