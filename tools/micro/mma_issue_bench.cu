// Microbenchmark: cost of issuing tcgen05.mma (kind::f16, M128, K16) from one warp, for several
// issue styles and N, on every SM.  Prints cycles per MMA (issue loop + drain) — compare with the
// tensor-pipe floor 128*N/256 cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_issue tools/micro/mma_issue_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_plain(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
// 8 MMAs (K = 128) in one asm block under one elect; A/B descriptors advance by 32 bytes (>>4 = 2)
// inside each 64-wide atom and by `atom` bytes between atoms.
template <int ATOM>
__device__ __forceinline__ void mma8_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 a4, %1, %5;\n\tadd.s64 a5, a4, 2;\n\tadd.s64 a6, a4, 4;\n\tadd.s64 a7, a4, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "add.s64 b4, %2, %5;\n\tadd.s64 b5, b4, 2;\n\tadd.s64 b6, b4, 4;\n\tadd.s64 b7, b4, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, 1;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc0), "n"(ATOM >> 4));
}

template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t mbar;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  if (warp == 1) {
    constexpr uint32_t id = idesc_bf16(128, N, 0, 0);
    constexpr uint32_t ATOM = 128 * 128;                 // [128 rows][64 cols] bf16 atom
    const uint64_t da = sdesc(sb, 16, 1024), db = sdesc(sb + 32768, 16, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t dst = tmem + (it & 1) * 256;
      if (MODE == 0) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          mma_elect(dst, da + off, db + off, id, kk > 0);
        }
      } else if (MODE == 1) {
        mma8_elect<ATOM>(dst, da, db, id, 0);
      } else if (MODE == 2) {
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
            mma_plain(dst, da + off, db + off, id, kk > 0);
          }
        }
        __syncwarp();
      }
    }
    long long t1 = clock64();
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
    asm volatile(
        "{\n\t.reg .pred d;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n\t@!d bra W;\n\t}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&mbar)) : "memory");
    long long t2 = clock64();
    if (lane == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int MODE, int N>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; cudaMalloc(&d, sms * 2 * sizeof(long long));
  cudaFuncSetAttribute(k<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024 + 1024);
  const int iters = 2000;
  k<MODE, N><<<sms, 128, 66 * 1024 + 1024>>>(d, 10);
  k<MODE, N><<<sms, 128, 66 * 1024 + 1024>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
  long long h[2 * 148];
  cudaMemcpy(h, d, sizeof(long long) * 2 * sms, cudaMemcpyDeviceToHost);
  double a = 0, b = 0;
  for (int i = 0; i < sms; ++i) { a += h[2 * i]; b += h[2 * i + 1]; }
  a /= sms * (double)iters * 8; b /= sms * (double)iters * 8;
  printf("%-28s N=%3d  issue %.1f cyc/MMA  total %.1f cyc/MMA  (floor %d)\n", name, N, a, b, 128 * N / 256);
  cudaFree(d);
}

int main() {
  run<0, 64>("per-MMA elect asm");
  run<1, 64>("8 MMAs in one asm, 1 elect");
  run<2, 64>("lane-0 branch");
  run<0, 128>("per-MMA elect asm");
  run<1, 128>("8 MMAs in one asm, 1 elect");
  run<2, 128>("lane-0 branch");
  run<0, 256>("per-MMA elect asm");
  run<1, 256>("8 MMAs in one asm, 1 elect");
  return 0;
}
