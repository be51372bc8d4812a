// Paged chunked-prefill attention on the 5th-generation tensor cores (sm_100a):
// tcgen05.mma with TMEM accumulators, operands staged in shared memory by TMA.
//
// What it computes (a4; readings Z1-Z3): for an item with query rows at
// absolute positions q_pos .. q_pos+n_q-1, row t and q head h attend causally to keys
// 0 .. q_pos+t of kv head g = h / G (G = h_q/h_kv), softmax scale 1/sqrt(128), K/V read from
// the paged pool through the request's block table.
//
// Tiling (one CTA = one work unit: a pair of 128-row Q tiles of one (item, kv head), or a
// KV-range piece of such a unit in the tail wave; details in DESIGN.md §6):
//   * GQA packing: tile row r = (token t0 + r/G, q head g*G + r%G), so the G heads that share
//     a kv head share every K/V tile (Q by TMA boxes {64, G, 128/G} over [rows][h_q][d]).
//   * KV tiles of 128 keys in the canonical K-major SWIZZLE_128B layout [d-half][128 keys][64]:
//     one 4-D TMA box per d-half when the tile's blocks have consecutive ids, else one 2-D box
//     {64, k} per block and d-half; one ring of 5 x 32-KB slots (K_j, V_j, K_j+1, ...) at the
//     base of shared memory, the two Q tiles after it.
//   * S_i = Q_i·K^T: 8 x tcgen05.mma M128 N128 K16 (SS) into TMEM S_i; O_i += P_i·V: 8 TS-MMAs
//     with P_i in TMEM (aliasing S_i's first 64 columns) and V MN-major from shared memory.
//     TMEM: S_0, S_1, O_0, O_1 (512 columns).  One MMA warp issues PV_0, S_0, PV_1, S_1 per KV
//     step, which keeps the two tiles' softmaxes half a step apart on the shared SMSPs.
//   * softmax (warpgroup per tile, thread = TMEM lane = row): stale-max exponentials against
//     the running max as the score chunks arrive, exact path (max, lazy O rescale when the max
//     grows by > 2^8) on the first, masked and violating tiles; exp2 on MUFU plus a
//     polynomial share on the FMA pipe; P packed to bf16 (f16 for FP8 pools) in two halves.
//   * epilogue: O / l from TMEM; full tiles staged in the freed Q buffer and written by TMA;
//     split pieces merge (O_k, m_k, l_k) through a coalesced workspace or straight from TMEM.
// Warp roles: 0 = TMA producer, 1 = MMA issuer + TMEM allocator, 2-3 = FP8 -> f16 converters
// (FP8 pools only), 4-7 / 8-11 = softmax + epilogue of Q tile 0 / 1.  All hand-offs are
// mbarriers; every wait traps after ~2^26 polls instead of hanging.
#include "tc_common.cuh"

#include <cstdlib>
#include <cstring>
#include <mutex>

// Build-time variants (experiments; defaults are the measured best).
#ifndef S2L_NST_BF16
#define S2L_NST_BF16 5        // K/V ring slots of the bf16 kernel (32 KB each)
#endif
#ifndef S2L_NST_FP8
#define S2L_NST_FP8 3         // converted (f16) K/V ring slots of the FP8 kernel
#endif
#ifndef S2L_F8ST
#define S2L_F8ST 4            // E4M3 staging slots of the FP8 kernel (16 KB each; 3 + 4 beat 4 + 2 by ~2 %)
#endif
#ifndef S2L_OUT_WAIT_READ
#define S2L_OUT_WAIT_READ 1
#endif

namespace s2l {
namespace {

constexpr uint32_t TMEM_COLS = 512;
#ifndef S2L_TMEM_MAP
#define S2L_TMEM_MAP 0          // experiment: 0 = S0 S1 O0 O1, 1 = S0 O0 S1 O1, 2 = O0 O1 S0 S1
#endif
// TMEM columns of tile i's S (P aliases its first 64 columns) and O accumulators
__host__ __device__ constexpr uint32_t tm_s(int i) {
  return S2L_TMEM_MAP == 1 ? 256u * i : (S2L_TMEM_MAP == 2 ? 256u + 128u * i : 128u * i);
}
__host__ __device__ constexpr uint32_t tm_o(int i) {
  return S2L_TMEM_MAP == 1 ? 256u * i + 128u : (S2L_TMEM_MAP == 2 ? 128u * i : 256u + 128u * i);
}

struct TcParams {
  const AttnItemDev* items;
  const int32_t* table;
  __nv_bfloat16* o;
  float* lse;
  int32_t n_items, max_blocks, layer, L, h_q, h_kv, kb, group;
  float scale_log2;
  // tail-wave KV split (v2): CTAs >= split_begin are pieces of units split into split_s
  // contiguous KV ranges; partials go to ws, the last piece of a unit merges (ws_cnt).
  int32_t split_begin, split_s;
  int32_t split_direct;   // 0: the last piece always merges from the workspace (tests)
  float* ws;       // [pieces][2][128][128] partial O (unnormalised, fp32)
  float* ws_ml;    // [pieces][2][128][2] running max (log2 units) and row sum
  int32_t* ws_cnt;
  uint32_t* trace;   // S2L_TRACE builds only: per-event SM clock stamps of CTA 0
  // fused append (NEXT-2, v2 only): the chunk's K/V (positions >= q_pos, block-aligned) are
  // read from the caller's rows of this layer (tmap_kin / tmap_vin: [rows][h_kv][d], row
  // q_row + t) instead of the pool, and each unit writes the blocks that start inside its own
  // token range to the pool (TMA store; a partial last block by plain stores into pool).
  int32_t fuse;
  __nv_bfloat16* pool;
  int32_t n_inl;     // > 0: the items are inl[0 .. n_inl) (by value), not *items
  AttnItemDev inl[kInlineAttnItems];
};
// Parameters of the fused-append instantiation (the input maps), kept out of the plain
// kernel's parameter block.  (Passing the chunk blocks' ids inline as well, so that the kernel
// could write their table entries instead of a patch launch, took the block past 4 KB and
// made every launch ~15 us slower: measured, `profiles/r01/next2_fused.txt`.)
struct TcParamsFused : TcParams {
  CUtensorMap tmap_kin, tmap_vin;     // box {64, 1, k}: one block of one kv head
  CUtensorMap tmap_kin_t, tmap_vin_t; // box {64, 1, 128}: a whole 128-key tile
  uint64_t fuse_mask;                 // bit i: item i's append is fused (others: from the pool)
};
template <bool kFuse> struct ParamsOf { using T = TcParams; };
template <> struct ParamsOf<true> { using T = TcParamsFused; };
__device__ __forceinline__ AttnItemDev item_at(const TcParams& p, int32_t i) {
  return p.n_inl ? p.inl[i] : p.items[i];
}

#ifdef S2L_TRACE
// Timing experiment: CTA 0 records (event, tile, step, clock); each writer thread has its own
// region and counter, so a stamp is two fire-and-forget global stores.
__device__ __forceinline__ void trace_ev(const TcParams& p, uint32_t& n, uint32_t writer, uint32_t ev,
                                         uint32_t tile, uint32_t j) {
  if (blockIdx.x != 0 || p.trace == nullptr || n >= 4000) return;
  uint32_t c;
  asm volatile("mov.u32 %0, %%clock;" : "=r"(c));
  uint32_t* e = p.trace + 16 + (writer * 4096 + n) * 2;
  e[0] = (ev << 24) | (tile << 16) | (j & 0xffff);
  e[1] = c;
  ++n;
  p.trace[writer] = n;
}
#define TRACE(ev, tile, j) trace_ev(p, tr_n, tr_w, ev, tile, j)
#else
#define TRACE(ev, tile, j)
#endif
#ifdef S2L_CTATRACE
// Timing experiment: every CTA stamps its phases (32 u64 slots per CTA in p.trace): 0/1
// globaltimer at entry / exit, 2.. SM clock at entry, setup done, Q landed (MMA warp), first K/V
// slot full (MMA warp), first S ready / loop end / epilogue done (softmax warp 4), exit; 9 =
// smid << 32 | nT, 10 = unit << 16 | piece << 8 | npieces, 12 = barrier init done (thread 0),
// 13 = TMEM allocated (warp 1), 14 = unit decoded (thread 0), 15 = barriers initialised,
// 16 = O_fin wait done (warp 4).
__device__ __forceinline__ void cta_stamp(uint32_t* tr, int slot, bool global = false) {
  if (tr == nullptr) return;
  uint64_t t;
  if (global) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  else asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  reinterpret_cast<uint64_t*>(tr)[(int64_t)blockIdx.x * 32 + slot] = t;
}
#define CT(slot) cta_stamp(p.trace, slot)
#define CTG(slot) cta_stamp(p.trace, slot, true)
#else
#define CT(slot)
#define CTG(slot)
#endif
// ======================================================================================
// v2: two Q tiles per CTA ping-ponged through the tensor core (the softmax of one tile runs
// while the MMAs of the other execute), P kept in TMEM (TS-MMA: A operand = P from TMEM,
// aliasing the first 64 columns of that tile's S buffer), one unified K/V TMA ring of 5
// 32-KB slots, packed f32x2 FMA / ADD in the softmax, setmaxnreg to give the two softmax
// warpgroups 208 registers.  384 threads: warpgroup 0 = producer (warp 0), MMA issuer and
// TMEM allocator (warp 1), FP8 converters (warps 2-3, FP8 pools); warpgroup 1 = softmax /
// epilogue of Q tile 0; warpgroup 2 = softmax / epilogue of Q tile 1.
// Hand-offs per tile i: MMA commits S_full[i] after S_i(j) (which also covers PV_i(j-1));
// softmax_i writes P_i(j) into TMEM and arrives P_full[i]; MMA issues PV_i(j) then S_i(j+1)
// (in-order tensor pipe: PV_i(j) reads P_i(j) before S_i(j+1) overwrites those columns).
namespace v2 {
constexpr int kThreads = 384;
// setmaxnreg moves registers inside the CTA's launch allocation (384 x 168): the control
// warpgroup releases first, the softmax warpgroups then grow; the sums must fit the pool or
// setmaxnreg.inc waits forever.
#ifndef S2L_REG_CTRL
#define S2L_REG_CTRL 88
#endif
#ifndef S2L_REG_SOFTMAX
#define S2L_REG_SOFTMAX 208
#endif
constexpr int kRegLaunch = 168, kRegCtrl = S2L_REG_CTRL, kRegSoftmax = S2L_REG_SOFTMAX;
static_assert(128 * kRegCtrl + 256 * kRegSoftmax <= kThreads * kRegLaunch, "register pool");
// of every 8 exp2 pairs, this many on the FMA pipe: 2 for bf16 pools; 1 for FP8 pools, whose
// converter warps already load the FMA / ALU pipes of SMSPs 2-3 (A/B in profiles/r02s2)
template <bool kFp8> constexpr int kPolyPairsPer8 = kFp8 ? S2L_POLY_PAIRS_FP8 : S2L_POLY_PAIRS;
// Shared-memory layout (bytes from the 1024-aligned base):
//   K/V ring of NST 32-KB tiles (K-major / MN-major SW128 images; FP8 pools: the converted
//   f16 tiles) | Q tiles 0/1 |
//   FP8 pools only: F8ST 16-KB staging slots for the E4M3 tiles TMA brings in (dense
//   [128 keys][128 d] bytes), converted to the bf16 ring by warps 2-3 | mbarriers | TMEM addr.
template <bool kFp8>
struct Lay {
  static constexpr int NST = kFp8 ? S2L_NST_FP8 : S2L_NST_BF16;
  static constexpr int F8ST = kFp8 ? S2L_F8ST : 0;
  static constexpr uint32_t kF8Tile = 16384;
#ifndef S2L_Q_AFTER_RING
#define S2L_Q_AFTER_RING 1     // bf16 kernels: K/V ring at the base, Q after it (+0.5 % C2 step, +0.6 % C5
#endif                         // over Q first, 6 alternating A/B pairs each, profiles/r02s3/ab_placement.txt)
#ifndef S2L_Q_AFTER_RING_FP8
#define S2L_Q_AFTER_RING_FP8 1 // the FP8-pool kernel too: +2.4 % FP8 step (6 pairs, ab_placement_fp8.txt)
#endif
  static constexpr bool kQLast = kFp8 ? S2L_Q_AFTER_RING_FP8 : S2L_Q_AFTER_RING;
  static constexpr uint32_t OFF_Q0 = kQLast ? NST * kTileBytes : 0, OFF_Q1 = OFF_Q0 + kTileBytes,
                            OFF_RING = kQLast ? 0 : 2 * kTileBytes;
  static constexpr uint32_t OFF_F8 = (2 + NST) * kTileBytes;
  static constexpr uint32_t OFF_BAR = OFF_F8 + F8ST * kF8Tile;
  // barriers: Q_full, ring_full[NST], ring_empty[NST], S_full[2], P_full[2] (keys 0-63),
  // P_half[2] (keys 64-127), O_fin[2], fp8 staging full[F8ST] / empty[F8ST], fp8: Q in f16
  static constexpr uint32_t B_QF = 0, B_RF = 1, B_RE = 1 + NST, B_SF = 1 + 2 * NST, B_PF = B_SF + 2,
                            B_PH = B_PF + 2, B_OF = B_PH + 2, B_8F = B_OF + 2, B_8E = B_8F + F8ST,
                            B_QC = B_8E + F8ST, NBARS = B_QC + (kFp8 ? 1 : 0);
  static constexpr uint32_t OFF_TMEM = OFF_BAR + NBARS * 8;
  static constexpr uint32_t SMEM = OFF_TMEM + 16 + 1024;
  static_assert(SMEM <= 232448, "shared memory");
};
}  // namespace v2

// two E4M3 codes (low byte first) -> f16x2, exactly (every E4M3 value, 2^-9 .. 448, is an f16)
__device__ __forceinline__ uint32_t e4m3x2_to_f16x2(uint16_t v) {
  uint32_t h2;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(v));
  return h2;
}
// bf16x2 -> f16x2: exact for |x| in [2^-14, 65504] (f16 has the wider mantissa); beyond, the
// nearest f16 (saturating at +-65504, subnormal / zero below) -- reading Z20 in DESIGN.md
__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t x) {
  uint32_t r;
  asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(__uint_as_float(x & 0xffff0000u)),
      "f"(__uint_as_float(x << 16)));
  return r;
}

// kFuse: the fused-append instantiation (NEXT-2); kFp8: K/V pool in FP8 E4M3 (kv_dtype 1).
template <bool kFuse, bool kFp8>
__global__ void __launch_bounds__(v2::kThreads, 1)
    attn_tc2_kernel(const __grid_constant__ CUtensorMap tmap_q,
                    const __grid_constant__ CUtensorMap tmap_kv,
                    const __grid_constant__ CUtensorMap tmap_kv4,
                    const __grid_constant__ CUtensorMap tmap_o,
                    const __grid_constant__ typename ParamsOf<kFuse>::T p) {
  using namespace v2;
  using L = Lay<kFp8>;
  constexpr int WNST = L::NST;
  constexpr uint32_t WOFF_Q0 = L::OFF_Q0, WOFF_Q1 = L::OFF_Q1, WOFF_RING = L::OFF_RING, WOFF_BAR = L::OFF_BAR,
                     WOFF_TMEM = L::OFF_TMEM;
  constexpr uint32_t WB_QF = L::B_QF, WB_RF = L::B_RF, WB_RE = L::B_RE, WB_SF = L::B_SF, WB_PF = L::B_PF,
                     WB_PH = L::B_PH, WB_OF = L::B_OF;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](uint32_t i) { return sb + WOFF_BAR + 8u * i; };
  uint32_t* tmem_holder = (uint32_t*)(smem + WOFF_TMEM);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef S2L_TRACE
  uint32_t tr_n = 0;
  const uint32_t tr_w = warp == 1 ? 0u : (warp == 4 ? 1u : (warp == 8 ? 2u : 3u));
#endif

  if (threadIdx.x == 0) { CTG(0); CT(2); }
  // ---- work unit: (item, kv head, pair of Q tiles), longest first
  int32_t unit = blockIdx.x, piece = 0, npieces = 1;
  if (unit >= p.split_begin) {
    const int32_t b = unit - p.split_begin;
    unit = p.split_begin + b / p.split_s;
    piece = b % p.split_s;
    npieces = p.split_s;
  }
  int32_t lo = 0, hi = p.n_items - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (item_at(p, mid).unit_begin <= unit) lo = mid; else hi = mid - 1;
  }
  const AttnItemDev it = item_at(p, lo);
  const int32_t local = unit - it.unit_begin;
  const int32_t pairs = (it.tiles + 1) >> 1;
#if S2L_HEAD_MAJOR
  // the pairs of one (item, kv head) are adjacent units: they stream the same K/V tiles at
  // about the same time, so L2 serves the repeats
  const int32_t pair = pairs - 1 - local % pairs;
  const int32_t kvh = local / pairs;
#else
  const int32_t pair = pairs - 1 - local / p.h_kv;
  const int32_t kvh = local % p.h_kv;
#endif
  // 32-bit arithmetic (key positions < 2^31: s2l_create checks max_blocks_per_request *
  // block_size); G and k are powers of two (G divides 128, k checked by s2l_create), so the
  // divisions by them are shifts -- the 64-bit divisions this replaces cost ~1000 cycles per CTA
  const int32_t G = p.group;
  const int32_t toks = kBM >> (__ffs(G) - 1);
  const int32_t tok0 = pair * 2 * toks;               // first token of tile 0; tile 1 at +toks
  const int32_t tok_last = min(tok0 + 2 * toks, it.n_q) - 1;
  const int32_t qpos = (int32_t)it.q_pos;
  const int32_t key_last = qpos + tok_last;
  const int32_t nT_all = key_last / kBN + 1;
  const int32_t jb = nT_all * piece / npieces;        // this CTA's KV tiles
  const int32_t nT = nT_all * (piece + 1) / npieces - jb;
  const int32_t kv_len = qpos + it.n_q;
  const int32_t nblk_valid = (kv_len + p.kb - 1) >> (__ffs(p.kb) - 1);

  if (threadIdx.x == 0) {
    CT(14);
    mbar_init(bar(WB_QF), 1);
    for (int s = 0; s < WNST; ++s) {
      mbar_init(bar(WB_RF + s), kFp8 ? 2 : 1);   // fp8: one arrival per converter warp
      mbar_init(bar(WB_RE + s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(WB_SF + i), 1);
      mbar_init(bar(WB_PF + i), 128);
      mbar_init(bar(WB_PH + i), 128);
      mbar_init(bar(WB_OF + i), 1);
    }
    for (int s = 0; s < L::F8ST; ++s) {
      mbar_init(bar(L::B_8F + s), 1);
      mbar_init(bar(L::B_8E + s), 2);
    }
    if (kFp8) mbar_init(bar(L::B_QC), 2);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    CT(15);
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_kv) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_kv4) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_o) : "memory");
#if !S2L_PDL
    // the two Q tiles start loading before the TMEM allocation and the CTA barrier (with PDL
    // the load has to follow griddepcontrol.wait: Q may come from the previous kernel)
    mbar_expect_tx(bar(WB_QF), 2 * kTileBytes);
    const int32_t z = (int32_t)(it.q_row + tok0);
    tma_load_3d(sb + WOFF_Q0, &tmap_q, bar(WB_QF), 0, kvh * G, z);
    tma_load_3d(sb + WOFF_Q0 + kAtom, &tmap_q, bar(WB_QF), 64, kvh * G, z);
    tma_load_3d(sb + WOFF_Q1, &tmap_q, bar(WB_QF), 0, kvh * G, z + toks);
    tma_load_3d(sb + WOFF_Q1 + kAtom, &tmap_q, bar(WB_QF), 64, kvh * G, z + toks);
#endif
    CT(12);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (lane == 0) CT(13);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
#ifdef S2L_CTATRACE
  if (threadIdx.x == 0 && p.trace) {
    CT(3);
    int32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    reinterpret_cast<uint64_t*>(p.trace)[(int64_t)blockIdx.x * 32 + 9] = ((uint64_t)smid << 32) | (uint32_t)nT;
    reinterpret_cast<uint64_t*>(p.trace)[(int64_t)blockIdx.x * 32 + 10] =
        ((uint64_t)unit << 16) | ((uint64_t)piece << 8) | (uint64_t)npieces;
  }
#endif
  pdl_prologue();   // the item descriptors above come from the parameters or the staging ring

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtrl));
    if (warp == 0) {
      // ================= TMA producer =================
      if (S2L_PDL && lane == 0) {
        mbar_expect_tx(bar(WB_QF), 2 * kTileBytes);
        const int32_t z = (int32_t)(it.q_row + tok0);
        tma_load_3d(sb + WOFF_Q0, &tmap_q, bar(WB_QF), 0, kvh * G, z);
        tma_load_3d(sb + WOFF_Q0 + kAtom, &tmap_q, bar(WB_QF), 64, kvh * G, z);
        tma_load_3d(sb + WOFF_Q1, &tmap_q, bar(WB_QF), 0, kvh * G, z + toks);
        tma_load_3d(sb + WOFF_Q1 + kAtom, &tmap_q, bar(WB_QF), 64, kvh * G, z + toks);
      }
      const int32_t nb_tile = kBN / p.kb;               // 1..8 blocks per 128-key tile
      const int32_t* trow = p.table + (int64_t)it.slot * p.max_blocks;
      const int32_t rows_per_block = p.L * 2 * p.h_kv * p.kb;
      const int32_t row_kv[2] = {((p.layer * 2 + 0) * p.h_kv + kvh) * p.kb,
                                 ((p.layer * 2 + 1) * p.h_kv + kvh) * p.kb};
      const int32_t lkh[2] = {(p.layer * 2 + 0) * p.h_kv + kvh, (p.layer * 2 + 1) * p.h_kv + kvh};
      auto load_id = [&](int32_t jt) {                  // lane b < nb_tile: block b of tile jt
        const int32_t b = (jb + jt) * nb_tile + lane;
        return __ldg(trow + (b < nblk_valid ? b : 0));
      };
      int32_t next_id = (lane < nb_tile) ? load_id(0) : 0;
      if constexpr (kFp8) {
        // FP8 pool: E4M3 tiles (dense [128 keys][128 d] bytes) into the staging slots; warps
        // 2-3 convert them into the bf16 ring the MMAs read
        uint32_t r8 = 0;
        for (int32_t j = 0; j < nT; ++j) {
          const int32_t cur_id = next_id;
          if (j + 1 < nT && lane < nb_tile) next_id = load_id(j + 1);
          int32_t ids[8];
#pragma unroll
          for (int b = 0; b < 8; ++b) ids[b] = __shfl_sync(0xffffffffu, cur_id, b);
          bool run = (jb + j + 1) * nb_tile <= nblk_valid;
#pragma unroll
          for (int b = 1; b < 8; ++b)
            if (b < nb_tile) run = run && (ids[b] == ids[0] + b);
#pragma unroll
          for (int kind = 0; kind < 2; ++kind, ++r8) {
            const uint32_t s = r8 % L::F8ST, ph = (r8 / L::F8ST) & 1;
            mbar_wait(bar(L::B_8E + s), ph ^ 1);
            if (lane == 0) {
              mbar_expect_tx(bar(L::B_8F + s), L::kF8Tile);
              const uint32_t dst = sb + L::OFF_F8 + s * L::kF8Tile;
              if (run) {
                tma_load_4d(dst, &tmap_kv4, bar(L::B_8F + s), 0, 0, lkh[kind], ids[0]);
              } else {
#pragma unroll
                for (int b = 0; b < 8; ++b)
                  if (b < nb_tile)
                    tma_load_2d(dst + b * p.kb * 128, &tmap_kv, bar(L::B_8F + s), 0,
                                ids[b] * rows_per_block + row_kv[kind]);
              }
            }
            __syncwarp();
          }
        }
      } else {
      uint32_t rp = 0;
      // fused append: blocks starting at or after q_pos come from the caller's rows; this unit
      // writes the blocks whose first position lies in its token range [wr_lo, wr_hi)
      bool fuse = false;
      if constexpr (kFuse) fuse = p.fuse != 0 && (lo >= 64 || ((p.fuse_mask >> lo) & 1ull));
      const int64_t wr_lo = it.q_pos + tok0, wr_hi = it.q_pos + min(tok0 + 2 * toks, it.n_q);
      bool st_pending = false;                          // lane 0 has TMA stores in flight
      if constexpr (kFuse) {
        // the chunk's K/V rows this unit will read from the caller's input (its last KV
        // tiles) are prefetched into L2 now, so the diagonal tiles do not wait on DRAM (the
        // plain path reads them from L2, where the append kernel just wrote them)
        if (fuse && lane < 2) {
          const CUtensorMap* tin = lane ? &p.tmap_vin_t : &p.tmap_kin_t;
          for (int64_t tpos = (int64_t)jb * kBN; tpos < (int64_t)(jb + nT) * kBN; tpos += kBN) {
            if (tpos < it.q_pos) continue;
            const int32_t z = (int32_t)(it.q_row + (tpos - it.q_pos));
            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(tin), "r"(0),
                         "r"(kvh), "r"(z) : "memory");
            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(tin), "r"(64),
                         "r"(kvh), "r"(z) : "memory");
          }
        }
      }
      for (int32_t j = 0; j < nT; ++j) {
        const int32_t cur_id = next_id;
        if (j + 1 < nT && lane < nb_tile) next_id = load_id(j + 1);   // prefetch the next ids
        int32_t ids[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) ids[b] = __shfl_sync(0xffffffffu, cur_id, b);
        const int64_t tpos = (int64_t)(jb + j) * kBN;     // first key position of the tile
        const bool fresh = fuse && tpos + kBN > it.q_pos; // tile holds chunk blocks
        bool run = !fresh && (jb + j + 1) * nb_tile <= nblk_valid;   // whole tile inside the table
#pragma unroll
        for (int b = 1; b < 8; ++b)
          if (b < nb_tile) run = run && (ids[b] == ids[0] + b);
        uint32_t slot[2];
#pragma unroll
        for (int kind = 0; kind < 2; ++kind, ++rp) {
          const uint32_t s = rp % WNST, ph = (rp / WNST) & 1;
          slot[kind] = s;
          if (st_pending) {                             // the stores still read a ring slot
            if (lane == 0) bulk_wait_read();
            st_pending = false;
          }
          mbar_wait(bar(WB_RE + s), ph ^ 1);
          if (lane == 0 && run) {
            // consecutive block ids: two 4-D boxes (d halves) cover the whole 128-key tile
            mbar_expect_tx(bar(WB_RF + s), kTileBytes);
            const uint32_t dst = sb + WOFF_RING + s * kTileBytes;
            tma_load_4d(dst, &tmap_kv4, bar(WB_RF + s), 0, 0, lkh[kind], ids[0]);
            tma_load_4d(dst + kAtom, &tmap_kv4, bar(WB_RF + s), 64, 0, lkh[kind], ids[0]);
          } else if (kFuse && lane == 0 && fresh && tpos >= it.q_pos) {
            if constexpr (kFuse) {
              // tile wholly inside the chunk: two boxes {64, 1, 128} of the caller's rows
              mbar_expect_tx(bar(WB_RF + s), kTileBytes);
              const uint32_t dst = sb + WOFF_RING + s * kTileBytes;
              const CUtensorMap* tin = kind ? &p.tmap_vin_t : &p.tmap_kin_t;
              const int32_t z = (int32_t)(it.q_row + (tpos - it.q_pos));
              tma_load_3d(dst, tin, bar(WB_RF + s), 0, kvh, z);
              tma_load_3d(dst + kAtom, tin, bar(WB_RF + s), 64, kvh, z);
            }
          } else if (lane == 0) {
            // one lane issues the whole tile: 2 boxes {64, k} (d halves) per block
            mbar_expect_tx(bar(WB_RF + s), kTileBytes);
            const uint32_t dst = sb + WOFF_RING + s * kTileBytes;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
              if (b < nb_tile) {
                const int64_t pos0 = tpos + b * p.kb;
                if (fresh && pos0 >= it.q_pos) {
                  if constexpr (kFuse) {
                    // chunk block: rows q_row + (pos0 - q_pos) .. of this layer's K or V input
                    const CUtensorMap* tin = kind ? &p.tmap_vin : &p.tmap_kin;
                    const int32_t z = (int32_t)(it.q_row + (pos0 - it.q_pos));
                    tma_load_3d(dst + b * p.kb * 128, tin, bar(WB_RF + s), 0, kvh, z);
                    tma_load_3d(dst + kAtom + b * p.kb * 128, tin, bar(WB_RF + s), 64, kvh, z);
                  }
                } else {
                  const int32_t y = ids[b] * rows_per_block + row_kv[kind];
                  tma_load_2d(dst + b * p.kb * 128, &tmap_kv, bar(WB_RF + s), 0, y);
                  tma_load_2d(dst + kAtom + b * p.kb * 128, &tmap_kv, bar(WB_RF + s), 64, y);
                }
              }
            }
          }
          __syncwarp();
        }
        if (fresh && tpos + kBN > wr_lo && tpos < wr_hi) {
          // write this unit's chunk blocks of the tile (K and V) from the ring to the pool
#pragma unroll
          for (int kind = 0; kind < 2; ++kind) {
            const uint32_t s = slot[kind], ph = ((rp - 2 + kind) / WNST) & 1;
            mbar_wait(bar(WB_RF + s), ph);
#pragma unroll
            for (int b = 0; b < 8; ++b) {
              const int64_t pos0 = tpos + b * p.kb;
              if (b >= nb_tile || pos0 < wr_lo || pos0 >= wr_hi) continue;
              const uint32_t src = sb + WOFF_RING + s * kTileBytes + b * p.kb * 128;
              const int32_t y = ids[b] * rows_per_block + row_kv[kind];
              const int64_t valid = min((int64_t)p.kb, it.q_pos + it.n_q - pos0);
              if (valid == p.kb) {
                if (lane == 0) {
                  tma_store_2d(&tmap_kv, src, 0, y);
                  tma_store_2d(&tmap_kv, src + kAtom, 64, y);
                  bulk_commit();
                }
                st_pending = true;
              } else {
                // partial last block: the valid rows by plain 16-byte copies (SW128 un-swizzle)
                for (int32_t e = lane; e < (int32_t)valid * 16; e += 32) {
                  const int32_t r = e >> 4, h = (e >> 3) & 1, c = e & 7;
                  uint4 val;
                  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                               : "=r"(val.x), "=r"(val.y), "=r"(val.z), "=r"(val.w)
                               : "r"(src + h * kAtom + r * 128 + ((c ^ (r & 7)) << 4)));
                  *reinterpret_cast<uint4*>(p.pool + ((int64_t)y + r) * kD + h * 64 + c * 8) = val;
                }
              }
            }
          }
          __syncwarp();
        }
      }
      if (kFuse && lane == 0) bulk_wait_all();
      }
    } else if (kFp8 && warp >= 2) {
      // ================= FP8 -> f16 converters (warps 2-3) =================
      // The FP8 kernel's MMAs run on f16 operands: E4M3 -> f16 is one exact conversion per two
      // values (E4M3 -> bf16 would need three more).  First the two Q tiles are converted
      // bf16 -> f16 in place (elementwise, so the SW128 image is unchanged); then each E4M3
      // tile (TMA, dense [key][128 B]) becomes the f16 K-major SW128 image the MMAs read:
      // key r, d-half h, 16-byte chunk c at h*16 KB + r*128 + ((c ^ (r & 7)) << 4).
      const int ct = threadIdx.x - 64;                    // 0..63
      mbar_wait(bar(WB_QF), 0);
#pragma unroll 4
      for (int i = ct; i < 2 * (int)kTileBytes / 16; i += 64) {
        const uint32_t a = sb + WOFF_Q0 + 16u * (uint32_t)i;   // Q0 and Q1 are contiguous
        uint32_t f[4];
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(f[0]), "=r"(f[1]), "=r"(f[2]), "=r"(f[3]) : "r"(a));
        st_shared_v4(a, bf16x2_to_f16x2(f[0]), bf16x2_to_f16x2(f[1]), bf16x2_to_f16x2(f[2]),
                     bf16x2_to_f16x2(f[3]));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(L::B_QC));
      uint32_t r8 = 0, rp = 0;
      for (int32_t j = 0; j < nT; ++j) {
#pragma unroll 1
        for (int kind = 0; kind < 2; ++kind, ++r8, ++rp) {
          const uint32_t s8 = r8 % L::F8ST, s = rp % WNST;
          mbar_wait(bar(L::B_8F + s8), (r8 / L::F8ST) & 1);
          mbar_wait(bar(WB_RE + s), ((rp / WNST) & 1) ^ 1);
          const uint32_t src = sb + L::OFF_F8 + s8 * L::kF8Tile;
          const uint32_t dst = sb + WOFF_RING + s * kTileBytes;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const uint32_t r = (uint32_t)(ct + 64 * i);
#pragma unroll
            for (uint32_t jj = 0; jj < 8; ++jj) {
              const uint32_t jc = (jj + r) & 7;             // staggered: rows spread over banks
              uint32_t f[4];
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(f[0]), "=r"(f[1]), "=r"(f[2]), "=r"(f[3])
                           : "r"(src + r * 128 + jc * 16));
              uint32_t o[8];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                o[2 * e] = e4m3x2_to_f16x2((uint16_t)(f[e] & 0xffffu));
                o[2 * e + 1] = e4m3x2_to_f16x2((uint16_t)(f[e] >> 16));
              }
              const uint32_t h = jc >> 2, c = (jc & 3) * 2;  // d = 16 jc .. 16 jc + 15
              const uint32_t row = dst + h * kAtom + r * 128;
              st_shared_v4(row + ((c ^ (r & 7)) << 4), o[0], o[1], o[2], o[3]);
              st_shared_v4(row + (((c + 1) ^ (r & 7)) << 4), o[4], o[5], o[6], o[7]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // visible to tcgen05
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(bar(WB_RF + s));
            mbar_arrive(bar(L::B_8E + s8));
          }
        }
      }
    } else if (warp == 1) {
      // ================= MMA issuer (whole warp, one elected lane issues) =================
      constexpr uint32_t idesc_s = idesc_bf16(kBM, kBN, 0, 0, kFp8);   // fp8 pools: f16 operands
      constexpr uint32_t idesc_o = idesc_bf16(kBM, kD, 0, 1, kFp8);
      // descriptors of the buffer bases; the start-address field (bits 0-13, 16-byte units)
      // is advanced by adding (byte offset >> 4) — smem addresses stay below 256 KB
      const uint64_t dq[2] = {sdesc(sb + WOFF_Q0, 16, 1024), sdesc(sb + WOFF_Q1, 16, 1024)};
      const uint64_t dk0 = sdesc(sb + WOFF_RING, 16, 1024);
      const uint64_t dv0 = sdesc(sb + WOFF_RING, kAtom, 1024);
      uint32_t rp = 0;
      auto next_full = [&]() {
        const uint32_t s = rp % WNST, ph = (rp / WNST) & 1;
        ++rp;
        mbar_wait(bar(WB_RF + s), ph);
        tc_fence_after();
        return s;
      };
      auto issue_s = [&](int i, uint32_t kslot) {
        if (lane == 0) TRACE(13, i, 0);
        const uint64_t kd = dk0 + ((kslot * kTileBytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * kAtom + (kk & 3) * 32) >> 4;
          mma_ss_elect(tmem + tm_s(i), dq[i] + off, kd + off, idesc_s, kk > 0);
        }
        mma_commit_elect(bar(WB_SF + i));
        if (lane == 0) TRACE(14, i, 0);
      };
      auto issue_pv = [&](int i, uint32_t vslot, int32_t j) {
        const uint64_t vd = dv0 + ((vslot * kTileBytes) >> 4);
        if (lane == 0) TRACE(10, i, j);
        mbar_wait(bar(WB_PF + i), j & 1);               // P keys 0-63 in TMEM
        tc_fence_after();
        if (lane == 0) TRACE(11, i, j);
#pragma unroll
        for (int kk = 0; kk < kBN / 32; ++kk)
          mma_ts_elect(tmem + tm_o(i), tmem + tm_s(i) + kk * 8, vd + ((kk * 16 * 128) >> 4),
                       idesc_o, (j > 0 || kk > 0));
        mbar_wait(bar(WB_PH + i), j & 1);               // P keys 64-127
        tc_fence_after();
        if (lane == 0) TRACE(12, i, j);
#pragma unroll
        for (int kk = kBN / 32; kk < kBN / 16; ++kk)
          mma_ts_elect(tmem + tm_o(i), tmem + tm_s(i) + kk * 8, vd + ((kk * 16 * 128) >> 4),
                       idesc_o, 1);
      };
      mbar_wait(bar(kFp8 ? L::B_QC : WB_QF), 0);
      tc_fence_after();
      if (lane == 0) CT(4);
      uint32_t kslot = next_full();
      if (lane == 0) CT(5);
      issue_s(0, kslot);
      issue_s(1, kslot);
      mma_commit_elect(bar(WB_RE + kslot));
      for (int32_t j = 0; j < nT; ++j) {
        const uint32_t vslot = next_full();
        issue_pv(0, vslot, j);
        const bool more = j + 1 < nT;
        if (more) {
          kslot = next_full();
          issue_s(0, kslot);
        } else {
          mma_commit_elect(bar(WB_OF + 0));
        }
        issue_pv(1, vslot, j);
        mma_commit_elect(bar(WB_RE + vslot));
        if (more) {
          issue_s(1, kslot);
          mma_commit_elect(bar(WB_RE + kslot));
        } else {
          mma_commit_elect(bar(WB_OF + 1));
        }
      }
      __syncwarp();
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    // ================= softmax / correction / epilogue of Q tile i =================
    const int i = (warp - 4) >> 2;                   // 0: warps 4-7, 1: warps 8-11
    const int r = (warp & 3) * 32 + lane;            // tile row == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_off + tm_s(i);
    const uint32_t tO = tmem + lane_off + tm_o(i);
    const int32_t tok = tok0 + i * toks + r / G;
    const int32_t hq = kvh * G + r % G;
    const bool valid = tok < it.n_q;
    const int64_t limit = it.q_pos + (valid ? tok : tok_last);
    const float sl2 = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    for (int32_t j = 0; j < nT; ++j) {
      const bool tr = (warp & 3) == 0 && lane == 0;
      if (tr) TRACE(20, i, j);
      mbar_wait(bar(WB_SF + i), j & 1);
      tc_fence_after();
      if (tr) TRACE(21, i, j);
      if (j == 0 && warp == 4 && lane == 0) CT(6);
      const int64_t key0 = (int64_t)(jb + j) * kBN;
      const int64_t vis64 = limit - key0;                 // keys c <= vis of this tile visible
      const int32_t vis = (int32_t)(vis64 < -1 ? -1 : (vis64 > kBN ? kBN : vis64));
      const bool masked_tile = __any_sync(0xffffffffu, vis < kBN - 1);
      uint32_t sv[128];
      float mt[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) mt[q] = -INFINITY;
      // Steady state (stale-max fast path): a tile after the first one of this CTA, with no
      // masked key and a finite running max in every row, is exponentiated against the running
      // max m_run straight away, chunk by chunk as its scores arrive from TMEM (p <= 2^8 as long
      // as the tile max stays within kRescaleThresh of m_run, the same bound the lazy rescale
      // keeps).  P of keys 0-63 is released to the PV MMAs only once the whole tile's max is
      // known to be within that bound; otherwise (rare) the tile falls through to the exact
      // path below, which rescales O and recomputes P with the new max (S is still in sv).
      const bool fast = j > 0 && !masked_tile && __all_sync(0xffffffffu, m_run != -INFINITY);
      bool loaded = false;
      if (fast) {
        const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m_run, -m_run);
        uint32_t pk[16];
        tmem_ld32(tS, sv);
        tmem_wait_ld();
        tmem_ld32(tS + 32, sv + 32);
        tmem_ld32(tS + 64, sv + 64);
        tmem_ld32(tS + 96, sv + 96);
        float2 acc = chunk_p32<kPolyPairsPer8<kFp8>, kFp8>(sv, make_float2(0.f, 0.f), sc2, nm2, pk);
        tmem_st16(tS, pk);
        tmem_wait_ld();
        acc = chunk_p32<kPolyPairsPer8<kFp8>, kFp8>(sv + 32, acc, sc2, nm2, pk);
        tmem_st16(tS + 16, pk);
        max32<false>(sv, 0, 0, mt);
        max32<false>(sv + 32, 0, 32, mt);
        max32<false>(sv + 64, 0, 64, mt);
        max32<false>(sv + 96, 0, 96, mt);
        const float mxf = fmaxf(fmaxf(fmaxf(mt[0], mt[1]), fmaxf(mt[2], mt[3])),
                                fmaxf(fmaxf(mt[4], mt[5]), fmaxf(mt[6], mt[7]))) * sl2;
        if (!__any_sync(0xffffffffu, mxf > m_run + kRescaleThresh)) {
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bar(WB_PF + i));                  // P keys 0-63
          if (tr) TRACE(23, i, j);
          acc = chunk_p32<kPolyPairsPer8<kFp8>, kFp8>(sv + 64, acc, sc2, nm2, pk);
          tmem_st16(tS + 32, pk);
          acc = chunk_p32<kPolyPairsPer8<kFp8>, kFp8>(sv + 96, acc, sc2, nm2, pk);
          tmem_st16(tS + 48, pk);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bar(WB_PH + i));                  // P keys 64-127
          if (tr) TRACE(24, i, j);
          l_run += acc.x + acc.y;
          continue;
        }
        tmem_wait_st();                                 // speculative P lands before the rewrite
        loaded = true;
      }
      if (!loaded) {
        tmem_ld32(tS, sv);
        tmem_ld32(tS + 32, sv + 32);
        tmem_wait_ld();
        tmem_ld32(tS + 64, sv + 64);                    // in flight during the first max half
        tmem_ld32(tS + 96, sv + 96);
        if (masked_tile) { max32<true>(sv, vis, 0, mt); max32<true>(sv + 32, vis, 32, mt); }
        else { max32<false>(sv, vis, 0, mt); max32<false>(sv + 32, vis, 32, mt); }
        tmem_wait_ld();
        if (masked_tile) { max32<true>(sv + 64, vis, 64, mt); max32<true>(sv + 96, vis, 96, mt); }
        else { max32<false>(sv + 64, vis, 64, mt); max32<false>(sv + 96, vis, 96, mt); }
      }
      float mx = fmaxf(fmaxf(fmaxf(mt[0], mt[1]), fmaxf(mt[2], mt[3])), fmaxf(fmaxf(mt[4], mt[5]), fmaxf(mt[6], mt[7])));
      mx *= sl2;
      if (tr) TRACE(22, i, j);
      const float m_new = (mx > m_run + kRescaleThresh) ? mx : m_run;
      if (j > 0) {
        const bool resc = m_new != m_run;
        if (__any_sync(0xffffffffu, resc)) {
          const float alpha = resc ? fast_exp2(m_run - m_new) : 1.f;
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
          l_run *= alpha;
        }
      }
      m_run = m_new;
      // a row with no visible key yet (possible in a split piece) keeps m = -inf and p = 0
      const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
      const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m_use, -m_use);
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t pk[32];
        acc = masked_tile ? chunk_p64<true, 0, kFp8>(sv + 64 * hh, acc, vis, 64 * hh, sc2, nm2, pk)
                          : chunk_p64<false, kPolyPairsPer8<kFp8>, kFp8>(sv + 64 * hh, acc, vis, 64 * hh, sc2, nm2, pk);
        tmem_st16(tS + 32 * hh, pk);
        tmem_st16(tS + 32 * hh + 16, pk + 16);
        tmem_wait_st();                // keys 64hh .. 64hh+63 of P are in TMEM
        tc_fence_before();
        mbar_arrive(bar((hh == 0 ? WB_PF : WB_PH) + i));
        if (tr) TRACE(hh == 0 ? 23 : 24, i, j);
      }
      l_run += acc.x + acc.y;
    }
    // epilogue
    if (warp == 4 && lane == 0) CT(7);
    mbar_wait(bar(WB_OF + i), 0);
    tc_fence_after();
    if (warp == 4 && lane == 0) CT(16);
    __nv_bfloat16* orow = p.o + ((it.q_row + tok) * p.h_q + hq) * (int64_t)kD;
    // Output tile: when all 128 rows of tile i are valid, the bf16 rows go into the tile's Q
    // buffer (free: O_fin covers every S MMA) in the SW128 image the Q TMA loaded, and one
    // thread stores them with two TMA boxes (d halves) -- per-thread row stores are 16-byte
    // pieces 256 B apart and took ~5000 cycles per CTA; a ragged tile stores its valid rows.
    const bool tile_full = tok0 + (i + 1) * toks <= it.n_q;
    const uint32_t ob = sb + (i ? WOFF_Q1 : WOFF_Q0);
    auto put16 = [&](int c, const uint32_t (&w)[8]) {   // bf16 output columns 16c .. 16c+15
      if (tile_full) {
        const uint32_t row = ob + (uint32_t)(c >> 2) * kAtom + (uint32_t)r * 128;
        const uint32_t cc = (uint32_t)(c & 3) * 2;
        st_shared_v4(row + ((cc ^ (r & 7)) << 4), w[0], w[1], w[2], w[3]);
        st_shared_v4(row + (((cc + 1) ^ (r & 7)) << 4), w[4], w[5], w[6], w[7]);
      } else if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 16);
        dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
        dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    };
    auto flush = [&]() {
      if (!tile_full) return;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // st.shared -> TMA
      asm volatile("bar.sync %0, 128;" ::"r"(2 + i) : "memory");
      if ((warp & 3) == 0 && lane == 0) {
        const int32_t z = (int32_t)(it.q_row + tok0 + i * toks);
        tma_store_3d(&tmap_o, ob, 0, kvh * G, z);
        tma_store_3d(&tmap_o, ob + kAtom, 64, kvh * G, z);
        bulk_commit();
#if S2L_OUT_WAIT_READ
        bulk_wait_read();   // shared memory may be released; the global writes complete on their own
#else
        bulk_wait_all();
#endif
      }
    };
    if (npieces == 1) {
      const float inv = 1.f / l_run;
      uint32_t sv[128];
      tmem_ld32(tO, sv);                               // the whole O row in one wait
      tmem_ld32(tO + 32, sv + 32);
      tmem_ld32(tO + 64, sv + 64);
      tmem_ld32(tO + 96, sv + 96);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t w[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          w[e] = pack_bf16(__uint_as_float(sv[16 * c + 2 * e]) * inv, __uint_as_float(sv[16 * c + 2 * e + 1]) * inv);
        put16(c, w);
      }
      flush();
      if (valid && p.lse)
        p.lse[(it.q_row + tok) * p.h_q + hq] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
    } else {
      // Split piece: (unnormalised O, m, l) of this KV range.  The piece that finds every other
      // piece already published merges straight from its own TMEM O; otherwise it publishes its
      // partial (workspace, float4 [column quad][row] per (piece, tile): a warp's stores and
      // loads are 512 contiguous bytes) and the last piece to publish merges from the workspace.
      //   O = sum_k 2^(m_k - M) O_k / sum_k 2^(m_k - M) l_k,  M = max_k m_k.
      const int32_t su = unit - p.split_begin;                 // split-unit index
      float4* ws4 = reinterpret_cast<float4*>(p.ws);
      auto wsi = [&](int32_t k) { return (((int64_t)su * npieces + k) * 2 + i) * 32 * 128 + r; };
      auto mli = [&](int32_t k) { return ((((int64_t)su * npieces + k) * 2 + i) * 128 + r) * 2; };
      volatile uint32_t* flag = (volatile uint32_t*)(smem + WOFF_TMEM + 8);
      if (threadIdx.x == 128) {
        int32_t done;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(done) : "l"(p.ws_cnt + su) : "memory");
        const uint32_t direct = (p.split_direct && done == npieces - 1) ? 1u : 0u;
        if (direct) p.ws_cnt[su] = 0;                         // ready for the next launch
        *flag = direct;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const bool direct = *flag != 0;
      bool merge = direct;
      if (!direct) {
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          uint32_t ov[16];
          tmem_ld16(tO + c * 16, ov);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 4; ++e)
            __stcg(ws4 + wsi(piece) + (int64_t)(4 * c + e) * 128,
                   make_float4(__uint_as_float(ov[4 * e]), __uint_as_float(ov[4 * e + 1]),
                               __uint_as_float(ov[4 * e + 2]), __uint_as_float(ov[4 * e + 3])));
        }
        __stcg(reinterpret_cast<float2*>(p.ws_ml + mli(piece)), make_float2(m_run, l_run));
        __threadfence();
        asm volatile("bar.sync 1, 256;" ::: "memory");       // both softmax warpgroups wrote
        if (threadIdx.x == 128) {
          const int32_t old = atomicAdd(p.ws_cnt + su, 1);
          const uint32_t last = (old == npieces - 1) ? 1u : 0u;
          if (last) p.ws_cnt[su] = 0;                        // ready for the next launch
          *flag = last;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        merge = *flag != 0;
        if (merge) __threadfence();
      }
      if (merge) {
        constexpr int kMaxPieces = 8;
        float mk[kMaxPieces], wk[kMaxPieces];
        float M = direct ? m_run : -INFINITY;
#pragma unroll
        for (int k = 0; k < kMaxPieces; ++k) {
          mk[k] = -INFINITY;
          wk[k] = 0.f;
          if (k < npieces && !(direct && k == piece)) {
            const float2 ml = __ldcg(reinterpret_cast<const float2*>(p.ws_ml + mli(k)));
            mk[k] = ml.x;
            wk[k] = ml.y;                                      // l_k for now
            M = fmaxf(M, ml.x);
          }
        }
        // a row no piece saw a key for keeps M = -inf (weights 0, O = 0; not reached by valid rows)
        const float Mu = (M == -INFINITY) ? 0.f : M;
        float Lsum = 0.f;
#pragma unroll
        for (int k = 0; k < kMaxPieces; ++k) {
          const float l = wk[k];
          wk[k] = (mk[k] == -INFINITY) ? 0.f : fast_exp2(mk[k] - Mu);
          Lsum += wk[k] * l;
        }
        const float wself = (direct && m_run != -INFINITY) ? fast_exp2(m_run - Mu) : 0.f;
        if (direct) Lsum += wself * l_run;
        const float inv = 1.f / Lsum;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          float acc[16];
          if (direct) {
            uint32_t ov[16];
            tmem_ld16(tO + c * 16, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] = wself * __uint_as_float(ov[e]);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) acc[e] = 0.f;
          }
#pragma unroll
          for (int k = 0; k < kMaxPieces; ++k) {
            if (k < npieces && !(direct && k == piece)) {
              const float4* src = ws4 + wsi(k) + (int64_t)(4 * c) * 128;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float4 x = __ldcg(src + e * 128);
                acc[4 * e] += wk[k] * x.x;
                acc[4 * e + 1] += wk[k] * x.y;
                acc[4 * e + 2] += wk[k] * x.z;
                acc[4 * e + 3] += wk[k] * x.w;
              }
            }
          }
          uint32_t w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) w[e] = pack_bf16(acc[2 * e] * inv, acc[2 * e + 1] * inv);
          put16(c, w);
        }
        flush();
        if (valid && p.lse) p.lse[(it.q_row + tok) * p.h_q + hq] = (M + __log2f(Lsum)) * 0.69314718055994531f;
      }
    }
    tc_fence_before();
    if (warp == 4 && lane == 0) CT(8);
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
  if (threadIdx.x == 0) { CT(11); CTG(1); }
}

}  // namespace

bool attn_tc_supported(const Geometry& g) {
  const int32_t G = g.h_q / g.h_kv;
  return g.d == kD && g.k >= 16 && g.k <= 128 && (kBM % G) == 0;
}

bool make_tmap_kv(void* out, const void* pool, int64_t num_blocks, int32_t L, int32_t h_kv,
                  int32_t d, int32_t k, bool fp8, const char** err) {
  auto fn = encode_fn(err);
  if (!fn) return false;
  const int64_t total_rows = num_blocks * L * 2 * h_kv * k;
  if (total_rows >= (1ll << 31)) {
    *err = "pool has >= 2^31 rows";
    return false;
  }
  // bf16 pools: boxes of one d-half (64 values = 128 B) in the SWIZZLE_128B image the MMAs
  // read; FP8 pools: boxes of the whole row (128 values = 128 B), dense, for the converters
  const CUtensorMapDataType dt = fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const CUtensorMapSwizzle sw = fp8 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B;
  const cuuint64_t es = fp8 ? 1 : 2;
  const cuuint32_t bx = fp8 ? 128 : 64;
  // (1) per-block map: the pool as [rows][d], box {bx, k} = one (block, layer, K|V, head) row set
  {
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)total_rows};
    cuuint64_t strides[1] = {(cuuint64_t)d * es};
    cuuint32_t box[2] = {bx, (cuuint32_t)k};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn((CUtensorMap*)out, dt, 2, (void*)pool, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "cuTensorMapEncodeTiled(pool, per block) failed";
      return false;
    }
  }
  // (2) run map: the pool as [block][L*2*h_kv][k][d], box {bx, k, 1, 128/k} = a whole 128-key
  //     tile (bf16: one d-half of it) when the tile's blocks have consecutive ids (the common
  //     case with the lowest-free-id allocator): rows land exactly like 128/k per-block boxes.
  {
    const int32_t R = 128 / k;
    cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)k, (cuuint64_t)L * 2 * h_kv, (cuuint64_t)num_blocks};
    cuuint64_t strides[3] = {(cuuint64_t)d * es, (cuuint64_t)k * d * es, (cuuint64_t)L * 2 * h_kv * k * d * es};
    cuuint32_t box[4] = {bx, (cuuint32_t)k, 1, (cuuint32_t)(R > 0 ? R : 1)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn((CUtensorMap*)((char*)out + 128), dt, 4, (void*)pool, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "cuTensorMapEncodeTiled(pool, block runs) failed";
      return false;
    }
  }
  return true;
}

bool make_tmap_in(void* out, const void* k, const void* v, int64_t rows, int32_t h_kv, int32_t d,
                  int32_t kb, const char** err) {
  auto fn = encode_fn(err);
  if (!fn) return false;
  // one layer's K (out[0,128), out[256,384)) and V (out[128,256), out[384,512)) rows
  // [rows][h_kv][d]; box {64, 1, kb} lands in shared memory exactly like the pool's per-block
  // box {64, kb}, box {64, 1, 128} like a whole-tile block run
  for (int i = 0; i < 4; ++i) {
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)h_kv, (cuuint64_t)rows};
    cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)h_kv * d * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)(i < 2 ? kb : kBN)};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn((CUtensorMap*)((char*)out + 128 * i), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                    (void*)((i & 1) ? v : k), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "cuTensorMapEncodeTiled(k/v input) failed";
      return false;
    }
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

static uint32_t* g_trace = nullptr;
void set_attn_trace(uint32_t* buf) { g_trace = buf; }

// The kernels' dynamic shared-memory limit is a per-device function attribute: set it once per
// device (a context created later on another GPU of the same process gets it too).
static cudaError_t ensure_smem_attr() {
  static std::mutex mu;
  static bool done[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(attn_tc2_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, v2::Lay<false>::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_tc2_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, v2::Lay<false>::SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(attn_tc2_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, v2::Lay<true>::SMEM);
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

cudaError_t launch_attn_tc(const Geometry& g, const AttnItemDev* items, const AttnItemDev* items_host,
                           int32_t n_items,
                           int32_t total_units, int32_t split_begin, int32_t split_s,
                           float* ws, int32_t max_pieces, int32_t* ws_cnt,
                           const int32_t* table, int32_t layer, const void* tmap_q,
                           const void* tmap_kv, const void* tmap_o, void* o, float* lse,
                           int32_t flags, cudaStream_t st, const void* tmap_in, void* pool,
                           uint64_t fuse_mask) {
  const bool fuse = (flags & kAttnFuseAppend) != 0;
  if (fuse && (!tmap_in || !pool)) return cudaErrorInvalidValue;
  cudaError_t e = ensure_smem_attr();
  if (e != cudaSuccess) return e;
  if (total_units <= 0) return cudaSuccess;
  TcParamsFused pf{};
  TcParams plain{};
  TcParams& p = fuse ? static_cast<TcParams&>(pf) : plain;
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
  CUtensorMap tq, tkv, tkv4, to;
  memcpy(&tq, tmap_q, sizeof(CUtensorMap));
  memcpy(&to, tmap_o, sizeof(CUtensorMap));
  memcpy(&tkv, tmap_kv, sizeof(CUtensorMap));
  memcpy(&tkv4, (const char*)tmap_kv + 128, sizeof(CUtensorMap));
  p.split_begin = total_units;
  p.split_s = 1;
  p.split_direct = (flags & kAttnNoDirectMerge) ? 0 : 1;
  int32_t grid = total_units;
  if (split_s > 1 && split_begin < total_units) {
    p.split_begin = split_begin;
    p.split_s = split_s;
    grid = split_begin + (total_units - split_begin) * split_s;
  }
  p.trace = g_trace;
  p.fuse = fuse ? 1 : 0;
  p.pool = (__nv_bfloat16*)pool;
  if (fuse) {
    memcpy(&pf.tmap_kin, tmap_in, sizeof(CUtensorMap));
    memcpy(&pf.tmap_vin, (const char*)tmap_in + 128, sizeof(CUtensorMap));
    memcpy(&pf.tmap_kin_t, (const char*)tmap_in + 256, sizeof(CUtensorMap));
    memcpy(&pf.tmap_vin_t, (const char*)tmap_in + 384, sizeof(CUtensorMap));
    pf.fuse_mask = fuse_mask;
  }
  p.ws = ws;
  p.ws_ml = ws ? ws + (int64_t)max_pieces * 2 * 128 * kD : nullptr;
  p.ws_cnt = ws_cnt;
  if (fuse && g.fp8) return cudaErrorInvalidValue;   // no in-kernel append into an FP8 pool
  if (fuse) return launch_k(attn_tc2_kernel<true, false>, dim3(grid), dim3(v2::kThreads), v2::Lay<false>::SMEM, st, tq, tkv, tkv4, to, pf);
  if (g.fp8) return launch_k(attn_tc2_kernel<false, true>, dim3(grid), dim3(v2::kThreads), v2::Lay<true>::SMEM, st, tq, tkv, tkv4, to, p);
  return launch_k(attn_tc2_kernel<false, false>, dim3(grid), dim3(v2::kThreads), v2::Lay<false>::SMEM, st, tq, tkv, tkv4, to, p);
}

}  // namespace s2l
