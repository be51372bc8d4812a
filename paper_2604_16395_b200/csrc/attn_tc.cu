// Paged chunked-prefill attention on the 5th-generation tensor cores (sm_100a):
// tcgen05.mma with TMEM accumulators, operands staged in shared memory by TMA.
//
// What it computes (a4; readings Z1-Z3): for an item with query rows at
// absolute positions q_pos .. q_pos+n_q-1, row t and q head h attend causally to keys
// 0 .. q_pos+t of kv head g = h / G (G = h_q/h_kv), softmax scale 1/sqrt(128), K/V read from
// the paged pool through the request's block table.
//
// Tiling (one CTA = one 128-row Q tile of one (item, kv head)):
//   * GQA packing: tile row r = (token t0 + r/G, q head g*G + r%G), so the G heads that share
//     a kv head share every K/V tile (one TMA of Q: box {64, G, 128/G} over [rows][h_q][d]).
//   * KV tiles of 128 keys; each 16-token (k-token) block is one TMA box {64, k} per d-half
//     at row (((block*L + layer)*2 + K|V)*h_kv + g)*k of the pool viewed as [rows][128].
//     Boxes land at 2 KB (k*128 B) offsets, giving the canonical K-major SWIZZLE_128B
//     layout [d-half][128 keys][64] without a gather.
//   * S = Q·K^T: 8 x tcgen05.mma M=128 N=128 K=16 (A, B K-major SW128) into TMEM
//     (two S buffers of 128 columns, so S_{j+1} runs on the tensor core while the softmax
//     warps work on S_j).
//   * softmax warps (4 warps, thread = TMEM lane = row) tcgen05.ld S, mask, online softmax
//     in fp32 with exp2 (log2 e folded into the scale), lazy rescale of O (only when the row
//     max grows by > 2^8), write P as bf16 into shared memory in the K-major SW128 layout.
//   * O += P·V: 8 x tcgen05.mma M=128 N=128 K=16, A = P (K-major), B = V (MN-major SW128,
//     V is [keys][d] with d contiguous, LBO = 16 KB between d-halves) into TMEM O.
//   * epilogue: tcgen05.ld O, divide by the row sum, bf16 store; optional LSE.
// Warp roles: 0 = TMA producer, 1 = MMA issuer (one thread), 2 = TMEM allocator,
// 4..7 = softmax / correction / epilogue.  Pipelines: K ring x2, V ring x2 (TMA -> MMA),
// S x2 (MMA -> softmax), P x1 and O (softmax <-> MMA), all mbarrier-based.
#include "s2l_internal.h"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

namespace s2l {
namespace {

constexpr int kD = 128;
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kThreads = 256;
constexpr uint32_t kTileBytes = kBM * kD * 2;  // 32 KB: a 128 x 128 bf16 operand tile
constexpr uint32_t kAtom = 16384;              // one [128 rows][64 cols] SW128 column of atoms

constexpr uint32_t OFF_Q = 0;
constexpr uint32_t OFF_K = OFF_Q + kTileBytes;
constexpr uint32_t OFF_V = OFF_K + 2 * kTileBytes;
constexpr uint32_t OFF_P = OFF_V + 2 * kTileBytes;
constexpr uint32_t OFF_BAR = OFF_P + kTileBytes;
enum : uint32_t {
  B_Q = 0, B_KF = 1, B_KE = 3, B_VF = 5, B_VE = 7, B_SF = 9, B_SE = 11, B_PF = 13, B_OD = 14,
  NUM_BARS = 15
};
constexpr uint32_t OFF_TMEM = OFF_BAR + NUM_BARS * 8;
constexpr uint32_t SMEM_BYTES = OFF_TMEM + 16 + 1024;  // + slack for 1024-B alignment
constexpr uint32_t TMEM_COLS = 512;                    // S0 [0,128) S1 [128,256) O [256,384)
constexpr uint32_t TMEM_O = 256;
constexpr float kRescaleThresh = 8.0f;                 // log2 units: rescale when max grows 256x

struct TcParams {
  const AttnItemDev* items;
  const int32_t* table;
  __nv_bfloat16* o;
  float* lse;
  int32_t n_items, max_blocks, layer, L, h_q, h_kv, kb, group;
  float scale_log2;
};

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
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
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
// Instruction descriptor kind::f16: D f32, A/B bf16, dense.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
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
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmap_q,
                   const __grid_constant__ CUtensorMap tmap_kv, const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  const uint32_t sQ = sb + OFF_Q, sK = sb + OFF_K, sV = sb + OFF_V, sP = sb + OFF_P;
  auto bar = [&](uint32_t i) { return sb + OFF_BAR + 8u * i; };
  uint32_t* tmem_holder = (uint32_t*)(smem + OFF_TMEM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- work unit: (item, kv head, Q tile), items sorted longest-first, last tile first
  const int32_t unit = blockIdx.x;
  int32_t lo = 0, hi = p.n_items - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (p.items[mid].unit_begin <= unit) lo = mid; else hi = mid - 1;
  }
  const AttnItemDev it = p.items[lo];
  const int32_t local = unit - it.unit_begin;
  const int32_t tile = it.tiles - 1 - local / p.h_kv;
  const int32_t kvh = local % p.h_kv;
  const int32_t G = p.group;
  const int32_t toks = kBM / G;
  const int32_t tok0 = tile * toks;
  const int32_t tok_last = min(tok0 + toks, it.n_q) - 1;
  const int64_t key_last = it.q_pos + tok_last;
  const int32_t nT = (int32_t)(key_last / kBN) + 1;
  const int64_t kv_len = it.q_pos + it.n_q;
  const int32_t nblk_valid = (int32_t)((kv_len + p.kb - 1) / p.kb);

  if (threadIdx.x == 0) {
    mbar_init(bar(B_Q), 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(B_KF + s), 1);
      mbar_init(bar(B_KE + s), 1);
      mbar_init(bar(B_VF + s), 1);
      mbar_init(bar(B_VE + s), 1);
      mbar_init(bar(B_SF + s), 1);
      mbar_init(bar(B_SE + s), 128);
    }
    mbar_init(bar(B_PF), 128);
    mbar_init(bar(B_OD), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_q) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_kv) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      mbar_expect_tx(bar(B_Q), kTileBytes);
      const int32_t z = (int32_t)(it.q_row + tok0);
      tma_load_3d(sQ, &tmap_q, bar(B_Q), 0, kvh * G, z);
      tma_load_3d(sQ + kAtom, &tmap_q, bar(B_Q), 64, kvh * G, z);
    }
    const int32_t nb_tile = kBN / p.kb;
    const int32_t* trow = p.table + (int64_t)it.slot * p.max_blocks;
    const int32_t rows_per_block = p.L * 2 * p.h_kv * p.kb;
    const int32_t row_k = ((p.layer * 2 + 0) * p.h_kv + kvh) * p.kb;
    const int32_t row_v = ((p.layer * 2 + 1) * p.h_kv + kvh) * p.kb;
    for (int32_t j = 0; j < nT; ++j) {
      const int s = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      int32_t bid = 0;
      if (lane < nb_tile) {
        const int32_t b = j * nb_tile + lane;
        bid = __ldg(trow + (b < nblk_valid ? b : 0));
      }
      const int32_t id = __shfl_sync(0xffffffffu, bid, lane >> 1);
      const int32_t blk_i = lane >> 1, half = lane & 1;
      // K_j
      mbar_wait(bar(B_KE + s), ph ^ 1);
      if (lane == 0) mbar_expect_tx(bar(B_KF + s), kTileBytes);
      __syncwarp();
      if (lane < 2 * nb_tile)
        tma_load_2d(sK + s * kTileBytes + half * kAtom + blk_i * p.kb * 128, &tmap_kv,
                    bar(B_KF + s), half * 64, id * rows_per_block + row_k);
      // V_j
      mbar_wait(bar(B_VE + s), ph ^ 1);
      if (lane == 0) mbar_expect_tx(bar(B_VF + s), kTileBytes);
      __syncwarp();
      if (lane < 2 * nb_tile)
        tma_load_2d(sV + s * kTileBytes + half * kAtom + blk_i * p.kb * 128, &tmap_kv,
                    bar(B_VF + s), half * 64, id * rows_per_block + row_v);
    }
  } else if (warp == 1) {
    // ================= MMA issuer (one thread) =================
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16(kBM, kBN, 0, 0);  // Q K-major, K K-major
      constexpr uint32_t idesc_o = idesc_bf16(kBM, kD, 0, 1);   // P K-major, V MN-major
      mbar_wait(bar(B_Q), 0);
      auto issue_s = [&](int32_t i) {
        const int s = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        mbar_wait(bar(B_KF + s), ph);
        mbar_wait(bar(B_SE + s), ph ^ 1);
        tc_fence_after();
        const uint32_t kbase = sK + s * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_bf16(tmem + s * 128, sdesc(sQ + off, 16, 1024), sdesc(kbase + off, 16, 1024),
                   idesc_s, kk > 0);
        }
        mma_commit(bar(B_SF + s));
        mma_commit(bar(B_KE + s));
      };
      issue_s(0);
      for (int32_t j = 0; j < nT; ++j) {
        if (j + 1 < nT) issue_s(j + 1);
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(bar(B_VF + s), ph);
        mbar_wait(bar(B_PF), j & 1);
        tc_fence_after();
        const uint32_t vbase = sV + s * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kBN / 16; ++kk) {
          const uint32_t aoff = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_bf16(tmem + TMEM_O, sdesc(sP + aoff, 16, 1024),
                   sdesc(vbase + kk * 16 * 128, kAtom, 1024), idesc_o, (j > 0 || kk > 0));
        }
        mma_commit(bar(B_VE + s));
        mma_commit(bar(B_OD));
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ================= softmax / correction / epilogue =================
    const int r = threadIdx.x - 128;                 // tile row == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    const int32_t tok = tok0 + r / G;
    const int32_t hq = kvh * G + r % G;
    const bool valid = tok < it.n_q;
    const int64_t limit = it.q_pos + (valid ? tok : tok_last);
    const float sl2 = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    uint32_t sv[128];
    for (int32_t j = 0; j < nT; ++j) {
      const int s = j & 1;
      mbar_wait(bar(B_SF + s), (j >> 1) & 1);
      tc_fence_after();
      {
        const uint32_t ta = tmem + lane_off + s * 128;
        tmem_ld32(ta, sv);
        tmem_ld32(ta + 32, sv + 32);
        tmem_ld32(ta + 64, sv + 64);
        tmem_ld32(ta + 96, sv + 96);
        tmem_wait_ld();
      }
      tc_fence_before();
      mbar_arrive(bar(B_SE + s));
      const int64_t key0 = (int64_t)j * kBN;
      if (key0 + kBN - 1 > limit) {
        const int32_t vis = (int32_t)(limit - key0);   // keys c <= vis are visible
#pragma unroll
        for (int c = 0; c < kBN; ++c)
          if (c > vis) sv[c] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kBN; ++c) mx = fmaxf(mx, __uint_as_float(sv[c]));
      mx *= sl2;
      const float m_new = (mx > m_run + kRescaleThresh) ? mx : m_run;
      if (j > 0) {
        mbar_wait(bar(B_OD), (j - 1) & 1);  // PV_{j-1} done: P buffer free, O stable
        tc_fence_after();
        const bool resc = m_new != m_run;
        if (__any_sync(0xffffffffu, resc)) {
          const float alpha = resc ? fast_exp2(m_run - m_new) : 1.f;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            const uint32_t ta = tmem + lane_off + TMEM_O + c * 32;
            tmem_ld32(ta, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            tmem_st32(ta, ov);
          }
          tmem_wait_st();
          l_run *= alpha;
        }
      }
      m_run = m_new;
      float sum = 0.f;
      const uint32_t prow = sP + r * 128;
#pragma unroll
      for (int chunk = 0; chunk < 16; ++chunk) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p0 = fast_exp2(fmaf(__uint_as_float(sv[chunk * 8 + 2 * e]), sl2, -m_run));
          const float p1 = fast_exp2(fmaf(__uint_as_float(sv[chunk * 8 + 2 * e + 1]), sl2, -m_run));
          sum += p0 + p1;
          w[e] = pack_bf16(p0, p1);
        }
        const uint32_t atom = chunk >> 3, cc = chunk & 7;
        st_shared_v4(prow + atom * kAtom + ((cc ^ (r & 7)) << 4), w[0], w[1], w[2], w[3]);
      }
      l_run += sum;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      mbar_arrive(bar(B_PF));
    }
    // epilogue
    mbar_wait(bar(B_OD), (nT - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l_run;
    __nv_bfloat16* orow = p.o + ((it.q_row + tok) * p.h_q + hq) * (int64_t)kD;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t ov[32];
      tmem_ld32(tmem + lane_off + TMEM_O + c * 32, ov);
      tmem_wait_ld();
      if (valid) {
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          w[e] = pack_bf16(__uint_as_float(ov[2 * e]) * inv, __uint_as_float(ov[2 * e + 1]) * inv);
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int e = 0; e < 4; ++e) dst[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
      }
    }
    if (valid && p.lse)
      p.lse[(it.q_row + tok) * p.h_q + hq] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
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

bool attn_tc_supported(const Geometry& g) {
  const int32_t G = g.h_q / g.h_kv;
  return g.d == kD && g.k >= 16 && g.k <= 128 && (kBM % G) == 0;
}

bool make_tmap_kv(void* out, const void* pool, int64_t total_rows, int32_t d, int32_t k,
                  const char** err) {
  auto fn = encode_fn(err);
  if (!fn) return false;
  if (total_rows >= (1ll << 31)) {
    *err = "pool has >= 2^31 rows";
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)total_rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)k};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn((CUtensorMap*)out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)pool, dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled(pool) failed";
    return false;
  }
  return true;
}

bool make_tmap_q(void* out, const void* q, int64_t q_rows, int32_t h_q, int32_t d, int32_t group,
                 const char** err) {
  auto fn = encode_fn(err);
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)h_q, (cuuint64_t)q_rows};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)h_q * d * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)group, (cuuint32_t)(kBM / group)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn((CUtensorMap*)out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)q, dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled(q) failed";
    return false;
  }
  return true;
}

cudaError_t launch_attn_tc(const Geometry& g, const AttnItemDev* items, int32_t n_items,
                           int32_t total_units, const int32_t* table, int32_t layer,
                           const void* tmap_q, const void* tmap_kv, void* o, float* lse,
                           cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (total_units <= 0) return cudaSuccess;
  TcParams p{};
  p.items = items;
  p.table = table;
  p.o = (__nv_bfloat16*)o;
  p.lse = lse;
  p.n_items = n_items;
  p.max_blocks = g.max_blocks;
  p.layer = layer;
  p.L = g.L;
  p.h_q = g.h_q;
  p.h_kv = g.h_kv;
  p.kb = g.k;
  p.group = g.h_q / g.h_kv;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)kD);
  CUtensorMap tq, tkv;
  memcpy(&tq, tmap_q, sizeof(CUtensorMap));
  memcpy(&tkv, tmap_kv, sizeof(CUtensorMap));
  attn_tc_kernel<<<total_units, kThreads, SMEM_BYTES, st>>>(tq, tkv, p);
  return cudaGetLastError();
}

}  // namespace s2l
