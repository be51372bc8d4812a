// Paged chunked-prefill attention on a CTA PAIR (tcgen05 cta_group::2, sm_100a).
//
// What it computes (a4; readings Z1-Z3): for an item with query rows at
// absolute positions q_pos .. q_pos+n_q-1, row t and q head h attend causally to keys
// 0 .. q_pos+t of kv head g = h / G (G = h_q/h_kv), softmax scale 1/sqrt(128), K/V read from
// the paged pool through the request's block table.  Same contract as attn_tc2_kernel
// (attn_tc.cu); this kernel is the one s2l_prefill_batch launches.
//
// Why a pair (the round-2 redesign): a CTA that ping-pongs two Q tiles through
// one SM's tensor core must alias P into S (TMEM holds S0, S1, O0, O1 = 512 columns), so
// S_i(j+1) cannot start before PV_i(j) has read P_i(j): softmax -> PV -> S -> softmax is a
// serial chain per tile, and the SS S-MMAs of two tiles plus K/V staging saturate shared memory.
// Here two CTAs on two SMs (a cluster of 2) run ONE work unit (item, kv head, pair of 128-row Q
// tiles), one tile each, and the leader CTA issues M = 256 MMAs for both:
//   * each CTA stages only half of every B operand: keys 64c..64c+63 of a K tile (S = Q K^T,
//     N = 128 keys split by N) and d-half c of a V tile (O += P V, N = 128 d split by N), so
//     TMA traffic and shared-memory operand reads per SM halve;
//   * TMEM per CTA (512 columns): S double buffer [0,256), P double buffer [256,384) (bf16,
//     128 keys = 64 columns), O [384,512).  S(j+1) is computed while the softmax works on S(j),
//     and P(j+1) is written while PV(j) still reads P(j): no chain through the tensor core.
//   * softmax: 8 warps per CTA, two per SMSP (warps q+4 and q+8 own TMEM lanes 32q..32q+31
//     and key halves 0-63 / 64-127 of those rows); the two halves exchange their maxima
//     through shared memory (a 64-thread named barrier) so both use the same running max.
// Warp roles per CTA: 0 = TMA producer (both CTAs), 1 = TMEM allocator + MMA issuer (leader),
// 4..11 = softmax / O rescale / epilogue.
#include "tc_common.cuh"

#include <cstring>
#include <mutex>

namespace s2l {
namespace {

namespace pr {
constexpr int kThreads = 384;
// setmaxnreg moves registers inside the CTA's launch allocation (384 x 168): warps 0-3 shrink,
// the eight softmax warps grow (the sums must fit or setmaxnreg.inc waits forever)
constexpr int kRegLaunch = 168, kRegCtrl = 88, kRegSoftmax = 208;
static_assert(128 * kRegCtrl + 256 * kRegSoftmax <= kThreads * kRegLaunch, "register pool");
constexpr uint32_t kHalf = 16384;                 // a K half [2 d-halves][64 keys][64] or a V half [128 keys][64]
constexpr int NST = 10;                           // ring slots: K_j at index 2j, V_j at 2j+1
constexpr uint32_t OFF_Q = 0;                     // this CTA's Q tile [2 d-halves][128 rows][64]
constexpr uint32_t OFF_RING = kTileBytes;
constexpr uint32_t OFF_XCH = OFF_RING + NST * kHalf;   // f32 scratch of the softmax warps
constexpr uint32_t OFF_BAR = OFF_XCH + 6 * 128 * 4;   // max hand-off [2][128] + epilogue [2][2][128]
enum : uint32_t {
  B_QF = 0,                 // leader: both CTAs' Q tiles landed (tx)
  B_RF = 1,                 // leader: ring slot s full, both CTAs' halves (tx)
  B_RE = B_RF + NST,        // each CTA: ring slot s free (MMA commit, multicast)
  B_SF = B_RE + NST,        // each CTA: S buffer b computed (commit, multicast)
  B_SR = B_SF + 2,          // leader: S buffer b read by all 16 softmax warps of the pair
  B_PL = B_SR + 2,          // leader: P buffer b keys 0-63 written (8 warps of the pair)
  B_PH = B_PL + 2,          // leader: P buffer b keys 64-127 written
  B_PE = B_PH + 2,          // each CTA: PV through P buffer b done (commit, multicast)
  B_OF = B_PE + 2,          // each CTA: the last PV done
  NBARS = B_OF + 1
};
constexpr uint32_t OFF_TMEMH = OFF_BAR + NBARS * 8;
constexpr uint32_t SMEM = OFF_TMEMH + 16 + 1024;  // + slack for the 1024-B alignment
constexpr uint32_t T_S = 0, T_P = 256, T_O = 384, TMEM_COLS = 512;
}  // namespace pr

struct PairParams {
  const AttnItemDev* items;
  const int32_t* table;
  __nv_bfloat16* o;
  float* lse;
  int32_t n_items, max_blocks, layer, L, h_q, h_kv, kb, group;
  float scale_log2;
  int32_t split_begin, split_s;  // tail-wave KV split (units >= split_begin run as split_s pieces)
  float* ws;                     // [pieces][2 tiles][128][128] partial O (unnormalised, fp32)
  float* ws_ml;                  // [pieces][2][128][2] running max (log2 units) and row sum
  int32_t* ws_cnt;               // [split units][2 tiles] arrival counters (self-resetting)
  uint32_t* trace;               // S2L_TRACE builds only: clock stamps of the first cluster's leader
  int32_t n_inl;                 // > 0: the items are inl[0 .. n_inl) (by value), not *items
  AttnItemDev inl[kInlineAttnItems];
};
#ifdef S2L_TRACE
// Timing experiment: the leader CTA of cluster 0 records (event, tile, step, clock); each
// writer (0 MMA, 1-2 softmax warps 4 / 8 lane 0, 3 producer) has its own region and counter.
__device__ __forceinline__ void ptrace(const PairParams& p, uint32_t& n, uint32_t writer, uint32_t ev, uint32_t j) {
  if (blockIdx.x != 0 || p.trace == nullptr || n >= 4000) return;
  uint32_t c;
  asm volatile("mov.u32 %0, %%clock;" : "=r"(c));
  uint32_t* e = p.trace + 16 + (writer * 4096 + n) * 2;
  e[0] = (ev << 24) | (j & 0xffff);
  e[1] = c;
  ++n;
  p.trace[writer] = n;
}
#define PTRACE(w, ev, j) ptrace(p, tr_n, w, ev, j)
#else
#define PTRACE(w, ev, j)
#endif
__device__ __forceinline__ AttnItemDev pitem_at(const PairParams& p, int32_t i) {
  return p.n_inl ? p.inl[i] : p.items[i];
}

// ---- cluster / cta_group::2 PTX ----------------------------------------------------------
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on an mbarrier of (possibly) another CTA of the cluster.  Default (CTA-scope)
// semantics, as CUTLASS's ClusterBarrier: the only data handed over through these barriers is
// TMEM, ordered by tcgen05.fence::before_thread_sync / after_thread_sync around the
// arrive / wait; release.cluster / acquire.cluster would add a GPU-scope MEMBAR per arrive and
// an L1 invalidate per wait (measured: 2x slower).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cbar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cbar) : "memory");
}
__device__ __forceinline__ void st_shared_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float ld_shared_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
// TMA loads of a CTA pair: the bytes land in this CTA's shared memory, the transaction count
// goes to the leader's mbarrier (cbar: shared::cluster address)
__device__ __forceinline__ void tma2_load_2d(uint32_t dst, const void* tmap, uint32_t cbar, int32_t x, int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(tmap), "r"(x), "r"(y), "r"(cbar)
      : "memory");
}
__device__ __forceinline__ void tma2_load_3d(uint32_t dst, const void* tmap, uint32_t cbar, int32_t x, int32_t y,
                                             int32_t z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(cbar)
      : "memory");
}
__device__ __forceinline__ void tma2_load_4d(uint32_t dst, const void* tmap, uint32_t cbar, int32_t x, int32_t y,
                                             int32_t z, int32_t w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(w), "r"(cbar)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma2_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// commit of the pair's MMAs issued so far: one arrival on the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void commit2_mc(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

// p = 2^(s*scale - m) for the 64 columns of one key half; returns the row-sum part and writes
// 32 packed bf16x2 (masked tiles: columns c > vis give p = 0, no polynomial share).
template <bool kMasked, int kPolyPer8>
__device__ __forceinline__ float half_p(const uint32_t* sv, int vis, float2 sc2, float2 nm2, uint32_t (&pk)[32]) {
  float2 acc = make_float2(0.f, 0.f);
  acc = chunk_p64<kMasked, kMasked ? 0 : kPolyPer8>(sv, acc, vis, 0, sc2, nm2, pk);
  return acc.x + acc.y;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pr::kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_kv,
                     const __grid_constant__ CUtensorMap tmap_kv4, const __grid_constant__ CUtensorMap tmap_kvh,
                     const __grid_constant__ PairParams p) {
  using namespace pr;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](uint32_t i) { return sb + OFF_BAR + 8u * i; };
  uint32_t* tmem_holder = (uint32_t*)(smem + OFF_TMEMH);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();                       // 0 = leader (issues the MMAs)
#ifdef S2L_TRACE
  uint32_t tr_n = 0;
#endif
  auto lbar = [&](uint32_t i) { return mapa(bar(i), 0); }; // the leader's copy of barrier i

  // ---- work unit: (item, kv head, pair of Q tiles), longest first; this CTA = tile `rank`
  int32_t unit = (int32_t)(blockIdx.x >> 1), piece = 0, npieces = 1;
  if (unit >= p.split_begin) {
    const int32_t b = unit - p.split_begin;
    unit = p.split_begin + b / p.split_s;
    piece = b % p.split_s;
    npieces = p.split_s;
  }
  int32_t lo = 0, hi = p.n_items - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (pitem_at(p, mid).unit_begin <= unit) lo = mid; else hi = mid - 1;
  }
  const AttnItemDev it = pitem_at(p, lo);
  const int32_t local = unit - it.unit_begin;
  const int32_t pairs = (it.tiles + 1) >> 1;
  const int32_t pair = pairs - 1 - local % pairs;          // head-major: a head's pairs are adjacent
  const int32_t kvh = local / pairs;
  const int32_t G = p.group;
  const int32_t toks = kBM / G;
  const int32_t tok0 = pair * 2 * toks;                    // first token of tile 0; tile 1 at +toks
  const int32_t tok_last = min(tok0 + 2 * toks, it.n_q) - 1;
  const int64_t key_last = it.q_pos + tok_last;
  const int32_t nT_all = (int32_t)(key_last / kBN) + 1;
  const int32_t jb = (int32_t)((int64_t)nT_all * piece / npieces);
  const int32_t nT = (int32_t)((int64_t)nT_all * (piece + 1) / npieces) - jb;
  const int64_t kv_len = it.q_pos + it.n_q;
  const int32_t nblk_valid = (int32_t)((kv_len + p.kb - 1) / p.kb);

  if (threadIdx.x == 0) {
    mbar_init(bar(B_QF), 1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(bar(B_RF + s), 1);
      mbar_init(bar(B_RE + s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(B_SF + b), 1);
      mbar_init(bar(B_SR + b), 8);
      mbar_init(bar(B_PL + b), 8);
      mbar_init(bar(B_PH + b), 8);
      mbar_init(bar(B_PE + b), 1);
    }
    mbar_init(bar(B_OF), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_q) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_kv) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_kv4) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_kvh) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();                                         // barriers initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_prologue();

  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtrl));
  if (warp == 0) {
    // ================= TMA producer (both CTAs: this CTA's halves) =================
    const uint32_t cqf = lbar(B_QF);
    if (lane == 0) {
      if (rank == 0) mbar_expect_tx(bar(B_QF), 2 * kTileBytes);   // both CTAs' Q tiles
      const int32_t z = (int32_t)(it.q_row + tok0 + rank * toks);
      tma2_load_3d(sb + OFF_Q, &tmap_q, cqf, 0, kvh * G, z);
      tma2_load_3d(sb + OFF_Q + kAtom, &tmap_q, cqf, 64, kvh * G, z);
    }
    const int32_t nb_tile = kBN / p.kb;                   // 1..8 blocks per 128-key tile
    const int32_t nb_half = nb_tile >= 2 ? nb_tile / 2 : 1;   // blocks holding this CTA's 64 keys
    const int32_t* trow = p.table + (int64_t)it.slot * p.max_blocks;
    const int32_t rows_per_block = p.L * 2 * p.h_kv * p.kb;
    const int32_t row_kv[2] = {((p.layer * 2 + 0) * p.h_kv + kvh) * p.kb,
                               ((p.layer * 2 + 1) * p.h_kv + kvh) * p.kb};
    const int32_t lkh[2] = {(p.layer * 2 + 0) * p.h_kv + kvh, (p.layer * 2 + 1) * p.h_kv + kvh};
    auto load_id = [&](int32_t jt) {                     // lane b < nb_tile: block b of tile jt
      const int32_t b = (jb + jt) * nb_tile + lane;
      return __ldg(trow + (b < nblk_valid ? b : 0));
    };
    int32_t next_id = (lane < nb_tile) ? load_id(0) : 0;
    for (int32_t j = 0; j < nT; ++j) {
      const int32_t cur_id = next_id;
      if (j + 1 < nT && lane < nb_tile) next_id = load_id(j + 1);
      int32_t ids[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) ids[b] = __shfl_sync(0xffffffffu, cur_id, b);
      const bool full = (jb + j + 1) * nb_tile <= nblk_valid;   // every block of the tile exists
#pragma unroll
      for (int kind = 0; kind < 2; ++kind) {
        const uint32_t idx = 2u * (uint32_t)j + kind;
        const uint32_t s = idx % NST, ph = (idx / NST) & 1;
        if (lane == 0) PTRACE(3, 30, idx);
        mbar_wait(bar(B_RE + s), ph ^ 1);
        if (lane == 0) {
          PTRACE(3, 31, idx);
          const uint32_t dst = sb + OFF_RING + s * kHalf;
          const uint32_t cf = lbar(B_RF + s);
          if (rank == 0) mbar_expect_tx(bar(B_RF + s), 2 * kHalf);   // both CTAs' halves
          if (kind == 0) {
            // K keys 64*rank .. +63 of the tile, both d-halves: [d-half][64 keys][64]
            if (p.kb == 128) {
              const int32_t y = ids[0] * rows_per_block + row_kv[0] + 64 * (int32_t)rank;
              tma2_load_2d(dst, &tmap_kvh, cf, 0, y);              // box {64, 64}
              tma2_load_2d(dst + 8192, &tmap_kvh, cf, 64, y);
            } else {
              const int32_t b0 = (int32_t)rank * nb_half;
              bool run = full;
#pragma unroll
              for (int b = 1; b < 8; ++b)
                if (b < nb_half) run = run && (ids[b0 + b] == ids[b0] + b);
              if (run) {
                tma2_load_4d(dst, &tmap_kvh, cf, 0, 0, lkh[0], ids[b0]);     // box {64, k, 1, 64/k}
                tma2_load_4d(dst + 8192, &tmap_kvh, cf, 64, 0, lkh[0], ids[b0]);
              } else {
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                  if (b < nb_half) {
                    const int32_t y = ids[b0 + b] * rows_per_block + row_kv[0];
                    tma2_load_2d(dst + b * p.kb * 128, &tmap_kv, cf, 0, y);
                    tma2_load_2d(dst + 8192 + b * p.kb * 128, &tmap_kv, cf, 64, y);
                  }
                }
              }
            }
          } else {
            // V d-half `rank` of all 128 keys: [128 keys][64]
            bool run = full;
#pragma unroll
            for (int b = 1; b < 8; ++b)
              if (b < nb_tile) run = run && (ids[b] == ids[0] + b);
            if (run) {
              tma2_load_4d(dst, &tmap_kv4, cf, 64 * (int32_t)rank, 0, lkh[1], ids[0]);   // box {64, k, 1, 128/k}
            } else {
#pragma unroll
              for (int b = 0; b < 8; ++b) {
                if (b < nb_tile) {
                  const int32_t y = ids[b] * rows_per_block + row_kv[1];
                  tma2_load_2d(dst + b * p.kb * 128, &tmap_kv, cf, 64 * (int32_t)rank, y);
                }
              }
            }
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 && rank == 0) {
    // ================= MMA issuer (leader; M = 256 over the pair) =================
    constexpr uint32_t idesc_s = idesc_bf16(256, kBN, 0, 0);
    constexpr uint32_t idesc_o = idesc_bf16(256, kD, 0, 1);
    const uint64_t dq = sdesc(sb + OFF_Q, 16, 1024);
    const uint64_t dr = sdesc(sb + OFF_RING, 16, 1024);    // K halves (K-major)
    const uint64_t dvr = sdesc(sb + OFF_RING, 8192, 1024); // V halves (MN-major, one atom wide)
    auto issue_s = [&](uint32_t b, uint32_t ks) {
      const uint64_t kd = dr + ((ks * kHalf) >> 4);
#pragma unroll
      for (int kk = 0; kk < kD / 16; ++kk) {
        const uint32_t oq = ((kk >> 2) * kAtom + (kk & 3) * 32) >> 4;
        const uint32_t ok = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
        mma2_ss(tmem + T_S + b * 128, dq + oq, kd + ok, idesc_s, kk > 0);
      }
      commit2_mc(bar(B_SF + b));
      commit2_mc(bar(B_RE + ks));
    };
    mbar_wait(bar(B_QF), 0);
    tc_fence_after();
    // Issue in readiness order: S(js) as soon as K_js has landed and softmax(js-2) has loaded
    // S buffer js&1 into registers (B_SR, early in that softmax step); PV(jp) as soon as the
    // halves of P(jp) are in TMEM.  (A fixed order S(j+2), PV(j) would hold S(j+2) back until
    // P(j) is done.)  The tensor pipe executes in issue order; S and PV touch disjoint TMEM.
    // mbarrier.test_wait never blocks (try_wait may suspend the thread for a while), so one
    // poll over several barriers stays cheap
    auto ready = [&](uint32_t b, uint32_t parity) {
      uint32_t ok;
      asm volatile(
          "{\n\t.reg .pred P1;\n\t"
          "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
          "selp.b32 %0, 1, 0, P1;\n\t}"
          : "=r"(ok)
          : "r"(b), "r"(parity)
          : "memory");
      return __all_sync(0xffffffffu, ok != 0);
    };
    int32_t js = 0, jp = 0, hp = 0;
    uint32_t vs = 0, spins = 0;
    while (jp < nT) {
      bool progress = false;
      if (js < nT) {
        const uint32_t idx = 2u * (uint32_t)js, ks = idx % NST;
        if (ready(bar(B_RF + ks), (idx / NST) & 1) &&
            (js < 2 || ready(bar(B_SR + (js & 1)), ((uint32_t)(js - 2) >> 1) & 1))) {
          tc_fence_after();
          if (lane == 0) PTRACE(0, 13, js);
          issue_s((uint32_t)js & 1, ks);
          ++js;
          progress = true;
        }
      }
      if (jp < js) {
        const uint32_t b = (uint32_t)jp & 1, ph = ((uint32_t)jp >> 1) & 1;
        if (hp == 0) {
          const uint32_t idx = 2u * (uint32_t)jp + 1;
          vs = idx % NST;
          if (ready(bar(B_RF + vs), (idx / NST) & 1) && ready(bar(B_PL + b), ph)) {
            tc_fence_after();
            if (lane == 0) PTRACE(0, 11, jp);
            const uint64_t vd = dvr + ((vs * kHalf) >> 4);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma2_ts(tmem + T_O, tmem + T_P + b * 64 + kk * 8, vd + ((kk * 16 * 128) >> 4), idesc_o,
                      (jp > 0 || kk > 0));
            hp = 1;
            progress = true;
          }
        }
        if (hp == 1 && ready(bar(B_PH + b), ph)) {
          tc_fence_after();
          if (lane == 0) PTRACE(0, 12, jp);
          const uint64_t vd = dvr + ((vs * kHalf) >> 4);
#pragma unroll
          for (int kk = 4; kk < 8; ++kk)
            mma2_ts(tmem + T_O, tmem + T_P + b * 64 + kk * 8, vd + ((kk * 16 * 128) >> 4), idesc_o, 1);
          commit2_mc(bar(B_PE + b));
          commit2_mc(bar(B_RE + vs));
          hp = 0;
          ++jp;
          progress = true;
        }
      }
      if (progress) spins = 0;
      else if (++spins == (1u << 26)) __trap();         // protocol watchdog (as mbar_wait)
    }
    commit2_mc(bar(B_OF));
    __syncwarp();
  } else if (warp >= 4) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    // ================= softmax / rescale / epilogue: rows 32q..32q+31 =================
    // Two warps per SMSP share these rows (TMEM lanes of quadrant q) and take alternate KV
    // steps: warp q+4 the even ones, warp q+8 the odd ones, so one warp's loads, max and
    // hand-off overlap the other's exponentials.  The running max travels between them
    // through shared memory (step j's max is read by the warp of step j+1, named barriers
    // 1+q / 5+q); each warp keeps its own partial row sum (scaled to the max it last saw),
    // combined in the epilogue.
    const int q = warp & 3, par = (warp - 4) >> 2;
    const int r = q * 32 + lane;                          // tile row == TMEM lane
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int32_t tok = tok0 + (int32_t)rank * toks + r / G;
    const int32_t hq = kvh * G + r % G;
    const bool valid = tok < it.n_q;
    const int64_t limit = it.q_pos + (valid ? tok : tok_last);
    const float sl2 = p.scale_log2;
    const uint32_t xm = sb + OFF_XCH;                     // f32 [step parity][128]: m after a step
    const uint32_t id_give = par ? 5 + q : 1 + q, id_take = par ? 1 + q : 5 + q;
    const uint32_t c_sr[2] = {lbar(B_SR + 0), lbar(B_SR + 1)};
    const uint32_t c_pl[2] = {lbar(B_PL + 0), lbar(B_PL + 1)};
    const uint32_t c_ph[2] = {lbar(B_PH + 0), lbar(B_PH + 1)};
    const uint32_t tO = tmem + lane_off + T_O;
    float m_w = -INFINITY, l_w = 0.f;                     // partial row sum, scaled to 2^-m_w
    for (int32_t j = par; j < nT; j += 2) {
      const uint32_t b = (uint32_t)j & 1;
      const uint32_t tS = tmem + lane_off + T_S + b * 128;
      const uint32_t tP = tmem + lane_off + T_P + b * 64;
      const bool tw = q == 0 && lane == 0;
      if (tw) PTRACE(1 + par, 20, j);
      mbar_wait(bar(B_SF + b), ((uint32_t)j >> 1) & 1);
      tc_fence_after();
      if (tw) PTRACE(1 + par, 21, j);
      const int64_t key0 = (int64_t)(jb + j) * kBN;
      const int64_t vis64 = limit - key0;                 // keys c <= vis of this tile visible
      const int32_t vis = (int32_t)(vis64 < -1 ? -1 : (vis64 > kBN ? kBN : vis64));
      const bool masked = __any_sync(0xffffffffu, vis < kBN - 1);
      uint32_t sv[128];
      float mt[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mt[i] = -INFINITY;
      tmem_ld32(tS, sv);
      tmem_ld32(tS + 32, sv + 32);
      tmem_wait_ld();
      tmem_ld32(tS + 64, sv + 64);                        // in flight during the first max half
      tmem_ld32(tS + 96, sv + 96);
      if (masked) { max32<true>(sv, vis, 0, mt); max32<true>(sv + 32, vis, 32, mt); }
      else { max32<false>(sv, vis, 0, mt); max32<false>(sv + 32, vis, 32, mt); }
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(c_sr[b]);        // S buffer b may be overwritten
      if (masked) { max32<true>(sv + 64, vis, 64, mt); max32<true>(sv + 96, vis, 96, mt); }
      else { max32<false>(sv + 64, vis, 64, mt); max32<false>(sv + 96, vis, 96, mt); }
      const float mx = fmaxf(fmaxf(fmaxf(mt[0], mt[1]), fmaxf(mt[2], mt[3])),
                             fmaxf(fmaxf(mt[4], mt[5]), fmaxf(mt[6], mt[7]))) * sl2;
      if (tw) PTRACE(1 + par, 22, j);
      float m_prev = -INFINITY;                           // the max after step j-1 (O's scale)
      if (j > 0) {
        asm volatile("bar.sync %0, 64;" ::"r"(id_take) : "memory");
        m_prev = ld_shared_f32(xm + 4u * ((b ^ 1) * 128 + r));
      }
      if (tw) PTRACE(1 + par, 25, j);
      const float m_new = (mx > m_prev + kRescaleThresh) ? mx : m_prev;
      if (j + 1 < nT) {                                   // hand the max to step j+1's warp
        st_shared_f32(xm + 4u * (b * 128 + r), m_new);
        asm volatile("bar.arrive %0, 64;" ::"r"(id_give) : "memory");
      }
      if (m_prev > m_w) {                                 // bring this warp's partial sum to m_prev
        l_w *= fast_exp2(m_w - m_prev);
        m_w = m_prev;
      }
      if (j >= 2) mbar_wait(bar(B_PE + b), ((uint32_t)j / 2 - 1) & 1);   // PV(j-2) read P buffer b
      if (j > 0 && __any_sync(0xffffffffu, m_new != m_prev)) {
        // O holds PV through step j-1, scaled to m_prev: rescale it once PV(j-1) is done
        mbar_wait(bar(B_PE + (b ^ 1)), ((uint32_t)(j - 1) / 2) & 1);
        tc_fence_after();
        const float alpha = (m_new != m_prev) ? fast_exp2(m_prev - m_new) : 1.f;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          uint32_t ov[16];
          tmem_ld16(tO + c * 16, ov);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            float2 x = __fmul2_rn(make_float2(__uint_as_float(ov[e]), __uint_as_float(ov[e + 1])),
                                  make_float2(alpha, alpha));
            ov[e] = __float_as_uint(x.x);
            ov[e + 1] = __float_as_uint(x.y);
          }
          tmem_st16(tO + c * 16, ov);
        }
      }
      if (m_new > m_w) {
        l_w *= (m_w == -INFINITY) ? 0.f : fast_exp2(m_w - m_new);
        m_w = m_new;
      }
      // a row with no visible key yet (possible in a split piece) keeps m = -inf and p = 0
      const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
      const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m_use, -m_use);
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t pk[32];
        acc = masked ? chunk_p64<true, 0>(sv + 64 * hh, acc, vis, 64 * hh, sc2, nm2, pk)
                     : chunk_p64<false, S2L_POLY_PAIRS>(sv + 64 * hh, acc, vis, 64 * hh, sc2, nm2, pk);
        tmem_st16(tP + 32 * hh, pk);
        tmem_st16(tP + 32 * hh + 16, pk + 16);
        tmem_wait_st();                                   // keys 64hh .. 64hh+63 of P in TMEM
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(hh == 0 ? c_pl[b] : c_ph[b]);
        if (tw) PTRACE(1 + par, 23 + hh, j);
      }
      l_w += acc.x + acc.y;
    }
    // ---- epilogue: combine the two warps' (m, l); each warp writes 64 of the 128 O columns
    mbar_wait(bar(B_OF), 0);
    tc_fence_after();
    const uint32_t ep = sb + OFF_XCH + 2 * 128 * 4;       // f32 [warp parity][2][128]
    st_shared_f32(ep + 4u * ((par * 2 + 0) * 128 + r), m_w);
    st_shared_f32(ep + 4u * ((par * 2 + 1) * 128 + r), l_w);
    asm volatile("bar.sync %0, 64;" ::"r"(9 + q) : "memory");
    const float m_o = ld_shared_f32(ep + 4u * (((par ^ 1) * 2 + 0) * 128 + r));
    const float l_o = ld_shared_f32(ep + 4u * (((par ^ 1) * 2 + 1) * 128 + r));
    const float m_run = fmaxf(m_w, m_o);
    const float l_all = (m_w == -INFINITY ? 0.f : l_w * fast_exp2(m_w - m_run)) +
                        (m_o == -INFINITY ? 0.f : l_o * fast_exp2(m_o - m_run));
    const int h = par;                                    // output columns 64h .. 64h+63
    const uint32_t tOh = tO + 64 * h;
    __nv_bfloat16* orow = p.o + ((it.q_row + tok) * p.h_q + hq) * (int64_t)kD + 64 * h;
    if (npieces == 1) {
      const float inv = 1.f / l_all;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[16];
        tmem_ld16(tOh + c * 16, ov);
        tmem_wait_ld();
        if (valid) {
          uint32_t w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            w[e] = pack_bf16(__uint_as_float(ov[2 * e]) * inv, __uint_as_float(ov[2 * e + 1]) * inv);
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
          dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
          dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      if (valid && p.lse && h == 0)
        p.lse[(it.q_row + tok) * p.h_q + hq] = (m_run + __log2f(l_all)) * 0.69314718055994531f;
    } else {
      // partial (unnormalised O, m, l) of this KV range -> workspace; the last piece merges
      const int32_t su = unit - p.split_begin;
      const int64_t prow = (((int64_t)su * npieces + piece) * 2 + rank) * 128 + r;
      float* wo = p.ws + prow * kD + 64 * h;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[16];
        tmem_ld16(tOh + c * 16, ov);
        tmem_wait_ld();
        float4* dst = reinterpret_cast<float4*>(wo + c * 16);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          dst[e] = make_float4(__uint_as_float(ov[4 * e]), __uint_as_float(ov[4 * e + 1]),
                               __uint_as_float(ov[4 * e + 2]), __uint_as_float(ov[4 * e + 3]));
      }
      if (h == 0) {
        p.ws_ml[prow * 2] = m_run;
        p.ws_ml[prow * 2 + 1] = l_all;
      }
      __threadfence();
      asm volatile("bar.sync 15, 256;" ::: "memory");      // all softmax warps of this CTA wrote
      uint32_t* flag = (uint32_t*)(smem + OFF_TMEMH + 8);
      if (threadIdx.x == 128) {
        const int32_t old = atomicAdd(p.ws_cnt + su * 2 + rank, 1);
        const uint32_t last = (old == npieces - 1) ? 1u : 0u;
        if (last) p.ws_cnt[su * 2 + rank] = 0;            // ready for the next launch
        *flag = last;
      }
      asm volatile("bar.sync 15, 256;" ::: "memory");
      if (*flag) {
        __threadfence();
        float M = -INFINITY;
        for (int k = 0; k < npieces; ++k) {
          const int64_t pr = (((int64_t)su * npieces + k) * 2 + rank) * 128 + r;
          M = fmaxf(M, __ldcg(p.ws_ml + pr * 2));
        }
        constexpr int kMaxPieces = 8;
        float wk[kMaxPieces];
        float Lsum = 0.f;
#pragma unroll
        for (int k = 0; k < kMaxPieces; ++k) {
          wk[k] = 0.f;
          if (k < npieces) {
            const int64_t pr = (((int64_t)su * npieces + k) * 2 + rank) * 128 + r;
            wk[k] = fast_exp2(__ldcg(p.ws_ml + pr * 2) - M);
            Lsum += wk[k] * __ldcg(p.ws_ml + pr * 2 + 1);
          }
        }
        const float inv = 1.f / Lsum;
#pragma unroll 1
        for (int c0 = 0; c0 < 64; c0 += 32) {
          float acc[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) acc[c] = 0.f;
#pragma unroll
          for (int k = 0; k < kMaxPieces; ++k) {
            if (k < npieces) {
              const float* po = p.ws + ((((int64_t)su * npieces + k) * 2 + rank) * 128 + r) * kD + 64 * h + c0;
#pragma unroll
              for (int c = 0; c < 32; c += 2) {
                const float2 x = __ldcg(reinterpret_cast<const float2*>(po + c));
                acc[c] += wk[k] * x.x;
                acc[c + 1] += wk[k] * x.y;
              }
            }
          }
          if (valid) {
#pragma unroll
            for (int c = 0; c < 32; c += 8) {
              uint4 v4 = make_uint4(pack_bf16(acc[c] * inv, acc[c + 1] * inv), pack_bf16(acc[c + 2] * inv, acc[c + 3] * inv),
                                    pack_bf16(acc[c + 4] * inv, acc[c + 5] * inv), pack_bf16(acc[c + 6] * inv, acc[c + 7] * inv));
              *reinterpret_cast<uint4*>(orow + c0 + c) = v4;
            }
          }
        }
        if (valid && p.lse && h == 0) p.lse[(it.q_row + tok) * p.h_q + hq] = (M + __log2f(Lsum)) * 0.69314718055994531f;
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  cluster_sync();                                         // both CTAs done with TMEM / smem
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

cudaError_t ensure_pair_attr() {
  static std::mutex mu;
  static bool done[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(attn_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pr::SMEM);
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

}  // namespace

cudaError_t launch_attn_pair(const Geometry& g, const AttnItemDev* items, const AttnItemDev* items_host,
                             int32_t n_items, int32_t total_units, int32_t split_begin, int32_t split_s,
                             float* ws, int32_t max_pieces, int32_t* ws_cnt, const int32_t* table,
                             int32_t layer, const void* tmap_q, const void* tmap_kv, void* o, float* lse,
                             cudaStream_t st) {
  cudaError_t e = ensure_pair_attr();
  if (e != cudaSuccess) return e;
  if (total_units <= 0) return cudaSuccess;
  PairParams p{};
  p.items = items;
  p.n_inl = 0;
  if (items_host && n_items <= kInlineAttnItems) {
    memcpy(p.inl, items_host, (size_t)n_items * sizeof(AttnItemDev));
    p.n_inl = n_items;
  }
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
  CUtensorMap tq, tkv, tkv4, tkvh;
  memcpy(&tq, tmap_q, sizeof(CUtensorMap));
  memcpy(&tkv, tmap_kv, sizeof(CUtensorMap));
  memcpy(&tkv4, (const char*)tmap_kv + 128, sizeof(CUtensorMap));
  memcpy(&tkvh, (const char*)tmap_kv + 256, sizeof(CUtensorMap));
  p.split_begin = total_units;
  p.split_s = 1;
  int32_t units = total_units;
  if (split_s > 1 && split_begin < total_units) {
    p.split_begin = split_begin;
    p.split_s = split_s;
    units = split_begin + (total_units - split_begin) * split_s;
  }
  p.ws = ws;
  p.ws_ml = ws ? ws + (int64_t)max_pieces * 2 * 128 * kD : nullptr;
  p.ws_cnt = ws_cnt;
  p.trace = attn_trace_buf();
  return launch_k(attn_pair_kernel, dim3(2 * units), dim3(pr::kThreads), pr::SMEM, st, tq, tkv, tkv4, tkvh, p);
}

}  // namespace s2l
