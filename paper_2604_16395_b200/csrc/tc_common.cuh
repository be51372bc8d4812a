// Shared device helpers of the tcgen05 attention kernel (attn_tc.cu; also included by the
// measured-and-rejected CTA-pair experiment tools/experiments/attn_pair.cu):
// PTX wrappers (mbarrier, TMA, tcgen05 MMA / TMEM), the exp2 / softmax building blocks,
// and the driver entry point for tensor-map encoding.  Included by one TU each (anonymous
// namespace: every kernel TU gets its own inline copies).
#pragma once
#include "s2l_internal.h"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#ifndef S2L_POLY_PAIRS
#define S2L_POLY_PAIRS 2   // of every 8 exp2 pairs, this many on the FMA pipe (polynomial)
#endif
#ifndef S2L_POLY_PAIRS_FP8
#define S2L_POLY_PAIRS_FP8 1   // the FP8-pool kernel's share
#endif

namespace s2l {
namespace {

constexpr int kD = 128;
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr uint32_t kTileBytes = kBM * kD * 2;  // 32 KB: a 128 x 128 bf16 operand tile
constexpr uint32_t kAtom = 16384;              // one [128 rows][64 cols] SW128 column of atoms
#ifndef S2L_RESCALE_THRESH
#define S2L_RESCALE_THRESH 8.0f
#endif
#ifndef S2L_POLY_DEG
#define S2L_POLY_DEG 3          // degree of the FMA-pipe 2^f polynomial (experiment: 2)
#endif
constexpr float kRescaleThresh = S2L_RESCALE_THRESH;   // log2 units: rescale when max grows 256x

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Blocking wait with a watchdog: a protocol bug traps (kernel error) after ~2^26 timed-out
// try_waits (seconds) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  uint32_t n = 0;
  while (!mbar_try(bar, parity)) {
    if (++n == (1u << 26)) __trap();
  }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, uint32_t bar,
                                            int32_t x, int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(tmap), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, uint32_t bar,
                                            int32_t x, int32_t y, int32_t z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void* tmap, uint32_t bar,
                                            int32_t x, int32_t y, int32_t z, int32_t w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(w), "r"(bar)
      : "memory");
}
// TMA store smem -> global (bulk async-group of the issuing thread).
__device__ __forceinline__ void tma_store_2d(const void* tmap, uint32_t src, int32_t x, int32_t y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tmap),
               "r"(x), "r"(y), "r"(src)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const void* tmap, uint32_t src, int32_t x, int32_t y, int32_t z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tmap),
               "r"(x), "r"(y), "r"(z), "r"(src)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the smem sources of this thread's committed stores may be overwritten
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// this thread's committed stores are complete (visible in global memory)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor kind::f16: D f32, A/B bf16 (or f16 with f16 = true), dense.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn, bool f16 = false) {
  return (1u << 4) | (f16 ? 0u : (1u << 7) | (1u << 10)) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

#define S2L_R32(x) "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), \
    "=r"(x[6]), "=r"(x[7]), "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]),   \
    "=r"(x[13]), "=r"(x[14]), "=r"(x[15]), "=r"(x[16]), "=r"(x[17]), "=r"(x[18]),            \
    "=r"(x[19]), "=r"(x[20]), "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]),            \
    "=r"(x[25]), "=r"(x[26]), "=r"(x[27]), "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
#define S2L_W32(x) "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), \
    "r"(x[7]), "r"(x[8]), "r"(x[9]), "r"(x[10]), "r"(x[11]), "r"(x[12]), "r"(x[13]),          \
    "r"(x[14]), "r"(x[15]), "r"(x[16]), "r"(x[17]), "r"(x[18]), "r"(x[19]), "r"(x[20]),      \
    "r"(x[21]), "r"(x[22]), "r"(x[23]), "r"(x[24]), "r"(x[25]), "r"(x[26]), "r"(x[27]),      \
    "r"(x[28]), "r"(x[29]), "r"(x[30]), "r"(x[31])

// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets its lane's columns.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : S2L_R32(r)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31, %32};" ::"r"(taddr),
      S2L_W32(r)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe for a pair (offloads MUFU.EX2, the softmax bottleneck at d = 128):
// round-to-nearest split x = n + f with the 1.5*2^23 trick, f in [-0.5, 0.5], degree-3
// polynomial for 2^f (relative error <= 7.6e-5, fitted to 2^f on [-0.5, 0.5]), exponent
// added as an integer (n << 23).  x is clamped to >= -127 (result ~0 there); callers use it
// only on tiles without masked (-inf) scores.
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 y = __fadd2_rn(x, magic);
  const float2 t = __fadd2_rn(y, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-t.x, -t.y));
#if S2L_POLY_DEG == 2
  // experiment: degree 2 (relative error <= 1.73e-3, about bf16's half ulp)
  float2 q = __ffma2_rn(f, make_float2(0.23842709f, 0.23842709f), make_float2(0.70344443f, 0.70344443f));
  q = __ffma2_rn(q, f, make_float2(1.000443f, 1.000443f));
#else
  float2 q = __ffma2_rn(f, make_float2(0.0551704f, 0.0551704f), make_float2(0.24260826f, 0.24260826f));
  q = __ffma2_rn(q, f, make_float2(0.69326098f, 0.69326098f));
  q = __ffma2_rn(q, f, make_float2(0.99992833f, 0.99992833f));
#endif
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(y.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(y.y) << 23)));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// P -> bf16x2 (round to nearest even) for the PV MMA.
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// P -> the MMA's operand type: bf16x2 (kHalf = false) or f16x2 (the FP8-KV kernel, whose MMAs
// run on f16 operands), round to nearest even.
template <bool kHalf = false>
__device__ __forceinline__ uint32_t pack_p(float lo, float hi) {
  return kHalf ? pack_f16(lo, hi) : pack_bf16(lo, hi);
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

 // p = 2^(s*scale - m) for 64 columns (32 pairs per phase, the FMA-pipe polynomial spread
// over every 8/kPolyPer8-th pair): more independent work per phase for the single softmax warp of an SMSP
// (tools/micro/softmax_bench2.cu: ~10 % fewer cycles per tile than 32-column phases).
template <bool kMasked, int kPolyPer8, bool kHalf = false>
__device__ __forceinline__ float2 chunk_p64(const uint32_t* v, float2 acc, int vis, int base,
                                            float2 sc2, float2 nm2, uint32_t (&pk)[32]) {
  float2 x[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    float s0 = __uint_as_float(v[2 * c]), s1 = __uint_as_float(v[2 * c + 1]);
    if (kMasked) {
      if (base + 2 * c > vis) s0 = -INFINITY;
      if (base + 2 * c + 1 > vis) s1 = -INFINITY;
    }
    x[c] = __ffma2_rn(make_float2(s0, s1), sc2, nm2);
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const bool poly = !kMasked && kPolyPer8 > 0 &&
                      ((kPolyPer8 == 1 || kPolyPer8 == 2 || kPolyPer8 == 4) ? (c % (8 / (kPolyPer8 ? kPolyPer8 : 1))) == 0
                                                                             : (c & 7) < kPolyPer8);
    if (poly) x[c] = exp2_poly2(x[c]);
    else x[c] = make_float2(fast_exp2(x[c].x), fast_exp2(x[c].y));
  }
  float2 a[4] = {acc, make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    a[c & 3] = __fadd2_rn(a[c & 3], x[c]);
    pk[c] = pack_p<kHalf>(x[c].x, x[c].y);
  }
  return __fadd2_rn(__fadd2_rn(a[0], a[1]), __fadd2_rn(a[2], a[3]));
}
// p = 2^(s*scale - m) for 32 columns of an unmasked tile (16 pairs), the FMA-pipe polynomial
// on kPolyPer8 of every 8 pairs, spread evenly (pair c is polynomial iff (c*kPolyPer8) mod 8 <
// kPolyPer8); returns the running pair sum, writes 16 packed bf16x2.
template <int kPolyPer8, bool kHalf = false>
__device__ __forceinline__ float2 chunk_p32(const uint32_t* v, float2 acc, float2 sc2, float2 nm2,
                                            uint32_t (&pk)[16]) {
  float2 x[16];
#pragma unroll
  for (int c = 0; c < 16; ++c)
    x[c] = __ffma2_rn(make_float2(__uint_as_float(v[2 * c]), __uint_as_float(v[2 * c + 1])), sc2, nm2);
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    if (((c * kPolyPer8) & 7) < kPolyPer8) x[c] = exp2_poly2(x[c]);
    else x[c] = make_float2(fast_exp2(x[c].x), fast_exp2(x[c].y));
  }
  float2 a[2] = {acc, make_float2(0.f, 0.f)};
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    a[c & 1] = __fadd2_rn(a[c & 1], x[c]);
    pk[c] = pack_p<kHalf>(x[c].x, x[c].y);
  }
  return __fadd2_rn(a[0], a[1]);
}
// Row max of 32 columns with 8 independent chains (short dependency latency).
template <bool kMasked>
__device__ __forceinline__ void max32(const uint32_t* sv, int vis, int base, float (&t)[8]) {
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    float x = __uint_as_float(sv[c]);
    if (kMasked && base + c > vis) x = -INFINITY;
    t[c & 7] = fmaxf(t[c & 7], x);
  }
}


__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}


// Warp-wide MMA issue: every lane of the MMA warp executes the loop with warp-uniform
// operands (kept in uniform registers); elect.sync picks one lane (always the same, lane 0,
// with the full warp converged) to issue tcgen05.mma / tcgen05.commit.
__device__ __forceinline__ void mma_ss_elect(uint32_t d_tmem, uint64_t a, uint64_t b,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn(const char** err) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !ptr) {
      *err = "cuTensorMapEncodeTiled entry point not found";
      return nullptr;
    }
    fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
  }
  return fn;
}


}  // namespace
}  // namespace s2l
