// Microbenchmark: tcgen05.mma throughput per SM for the operand modes the attention kernel can
// use (kind::f16, K16 per instruction, 8 instructions per group):
//   SS  cta_group::1  M128 N64/N128     A, B from smem            (S = Q K^T today)
//   TS  cta_group::1  M128 N64/N128     A from TMEM, B from smem  (PV today; S with Q in TMEM)
//   SS  cta_group::2  M256 N128         A per CTA, B split over the CTA pair
//   SS  cta_group::1  M128 N128 while two other warps stream st.shared (smem contention)
// Prints cycles per instruction vs the floor 128*N/256 (per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_modes tools/micro/mma_modes_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// MODE 0: SS cg1; 1: TS cg1; 2: SS cg2 (M256); 3: SS cg1 + smem store traffic
template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ volatile uint32_t stop;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool CG2 = MODE == 2;
  for (int i = threadIdx.x; i < 98304 / 4; i += 128) ((uint32_t*)smem)[i] = 0;
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (CG2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&holder)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&holder)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG2) cluster_sync(); else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  const bool leader = !CG2 || cta_rank() == 0;
  if (warp == 1 && leader) {
    constexpr uint32_t id = idesc_bf16(CG2 ? 256 : 128, N, 0, 0);
    constexpr uint32_t ATOM = 128 * 128;
    const uint64_t da = sdesc(sb, 16, 1024), db = sdesc(sb + 32768, 16, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t dst = tmem + (it & 1) * 128;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
        const uint32_t acc = kk > 0;
        if (MODE == 1) {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dst),
              "r"(tmem + 256 + kk * 8), "l"(db + off), "r"(id), "r"(acc));
        } else if (CG2) {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dst),
              "l"(da + off), "l"(db + off), "r"(id), "r"(acc));
        } else {
          asm volatile(
              "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dst),
              "l"(da + off), "l"(db + off), "r"(id), "r"(acc));
        }
      }
    }
    long long t1 = clock64();
    if (CG2)
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(mb),
          "h"((uint16_t)3) : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(mb) : "memory");
    asm volatile(
        "{\n\t.reg .pred d;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n\t@!d bra W;\n\t}" ::"r"(mb) : "memory");
    long long t2 = clock64();
    stop = 1;
    if (lane == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0; }
  } else if (CG2 && warp == 1) {
    asm volatile(
        "{\n\t.reg .pred d;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], 0;\n\t@!d bra W;\n\t}" ::"r"(mb) : "memory");
    if (lane == 0) { out[blockIdx.x * 2] = 0; out[blockIdx.x * 2 + 1] = 0; }
  } else if (MODE == 3 && warp >= 2) {
    // smem write traffic (like TMA fills): 16 B per lane per store into [64 KB, 96 KB)
    uint4 v = make_uint4(lane, 1, 2, 3);
    uint4* dst = (uint4*)(smem + 65536) + (warp - 2) * 1024;
    while (!stop) {
#pragma unroll 8
      for (int i = 0; i < 32; ++i) dst[(i * 32 + lane) & 1023] = v;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CG2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    if (CG2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int MODE, int N>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d; cudaMalloc(&d, sms * 2 * sizeof(long long));
  const int smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(k<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms / 2 * 2);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = MODE == 2 ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k<MODE, N>, d, 10);
  cudaLaunchKernelEx(&cfg, k<MODE, N>, d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s N=%d: %s\n", name, N, cudaGetErrorString(e)); exit(1); }
  long long h[2 * 148];
  cudaMemcpy(h, d, sizeof(long long) * 2 * cfg.gridDim.x, cudaMemcpyDeviceToHost);
  double a = 0, b = 0; int n = 0;
  for (unsigned i = 0; i < cfg.gridDim.x; ++i) if (h[2 * i + 1]) { a += h[2 * i]; b += h[2 * i + 1]; ++n; }
  a /= n * (double)iters * 8; b /= n * (double)iters * 8;
  // per SM: a cg2 instruction does 2x the work of a cg1 one on two SMs -> same per-SM floor
  printf("%-34s N=%3d  issue %.1f  total %.1f cyc/instr  (per-SM floor %d)\n", name, N, a, b, 128 * N / 256);
  cudaFree(d);
}

int main() {
  run<0, 64>("SS cg1 M128");
  run<0, 128>("SS cg1 M128");
  run<1, 64>("TS cg1 M128 (A in TMEM)");
  run<1, 128>("TS cg1 M128 (A in TMEM)");
  run<3, 128>("SS cg1 M128 + st.shared traffic");
  run<2, 128>("SS cg2 M256 (B split over pair)");
  run<2, 256>("SS cg2 M256 (B split over pair)");
  return 0;
}
