// umma_i8_test.cu -- validates a hand-built tcgen05.mma kind::i8 call on sm_100a:
// D[128 x N] (s32, TMEM) = A[128 x K] (u8, smem, K-major) * B[N x K]^T (s8, smem,
// K-major), SWIZZLE_NONE canonical layout (8-row x 16-byte core matrices),
// for the two LBO/SBO assignments; prints mismatches per variant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_test tools/umma_i8_test.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 16, K = 64;  // two K=32 MMAs

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// byte offset of (row, k) in a K-major SWIZZLE_NONE operand
__host__ __device__ inline uint32_t kmaj_off(uint32_t row, uint32_t k, uint32_t lbo, uint32_t sbo) {
  return (row % 8) * 16 + (k % 16) + (k / 16) * lbo + (row / 8) * sbo;
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__global__ void k(const uint8_t *A, const int8_t *B, int32_t *D, uint32_t lboA, uint32_t sboA,
                  uint32_t lboB, uint32_t sboB) {
  __shared__ __align__(1024) uint8_t sa[M * K];
  __shared__ __align__(1024) uint8_t sb[N * K];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const uint32_t t = threadIdx.x, warp = t / 32, lane = t % 32;
  for (uint32_t i = t; i < M * K; i += blockDim.x) {
    const uint32_t r = i / K, kk = i % K;
    sa[kmaj_off(r, kk, lboA, sboA)] = A[i];
  }
  for (uint32_t i = t; i < N * K; i += blockDim.x) {
    const uint32_t r = i / K, kk = i % K;
    sb[kmaj_off(r, kk, lboB, sboB)] = (uint8_t)B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // generic-proxy smem writes -> visible to the async (tensor) proxy
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t dt = tmem_base;
  if (t == 0) {
    // idesc: D s32 (2 << 4), A u8 (0 << 7), B s8 (1 << 10), K-major both, N>>3 << 17, M>>4 << 24
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);
    for (int kb = 0; kb < K / 32; ++kb) {
      // K=32 bytes per MMA = two core matrices along K: advance by 2*lbo
      const uint64_t da = make_desc(smem_u32(sa) + kb * 2 * lboA, lboA, sboA);
      const uint64_t db = make_desc(smem_u32(sb) + kb * 2 * lboB, lboB, sboB);
      const uint32_t acc = kb > 0 ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&mbar)));
  }
  // wait for the MMAs
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w reads TMEM lanes 32w..32w+31 (rows), 16 columns
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(dt + ((warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const uint32_t row = warp * 32 + lane;
  for (int n = 0; n < N; ++n) D[row * N + n] = (int32_t)r[n];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(dt));
}

int main() {
  std::vector<uint8_t> A(M * K);
  std::vector<int8_t> B(N * K);
  srand(1);
  for (auto &a : A) a = rand() % 4;
  for (auto &b : B) b = (int8_t)(rand() % 256 - 128);
  std::vector<int32_t> ref(M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      int s = 0;
      for (int kk = 0; kk < K; ++kk) s += (int)A[m * K + kk] * (int)B[n * K + kk];
      ref[m * N + n] = s;
    }
  uint8_t *dA;
  int8_t *dB;
  int32_t *dD;
  cudaMalloc(&dA, M * K);
  cudaMalloc(&dB, N * K);
  cudaMalloc(&dD, 4 * M * N);
  cudaMemcpy(dA, A.data(), M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), N * K, cudaMemcpyHostToDevice);
  // A: K=64 bytes = 4 core matrices along K; B the same
  struct V { uint32_t la, sa, lb, sb; const char *name; } vs[] = {
      {128, 512, 128, 512, "LBO=128 (K step) SBO=512 (8-row step)"},
      {1024 * 2, 128, 256, 128, "LBO=K-step far, SBO=128 (rows packed)"},
  };
  for (auto &v : vs) {
    cudaMemset(dD, 0, 4 * M * N);
    k<<<1, 128>>>(dA, dB, dD, v.la, v.sa, v.lb, v.sb);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int32_t> got(M * N);
    cudaMemcpy(got.data(), dD, 4 * M * N, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i) bad += got[i] != ref[i];
    printf("%-44s err=%s mismatches %d / %d  (D[0][0..3] = %d %d %d %d ref %d %d %d %d)\n", v.name,
           cudaGetErrorString(e), bad, M * N, got[0], got[1], got[2], got[3], ref[0], ref[1], ref[2],
           ref[3]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
