// libs2l host runtime: request table, two-tier block allocator, LCP, staging ring, stream /
// event hazards, swap copies, and the extern "C" ABI declared in include/s2l.h.
//
// Every operation follows the paper passage cited at the ABI declaration; the bookkeeping
// is the state machine of SURVEY §8.2 c.2 (and is checked bit-exact against oracle/ by
// tests/test_host_bookkeeping.py).  No attention / K/V arithmetic happens on the host.
#include "s2l.h"
#include "s2l_internal.h"

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace {

thread_local std::string g_err;

s2l_status fail(s2l_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- lowest-free-id allocator (reading Z9) ----------------------------------------------
// A bitset of free ids (bit = 1 -> free) plus a hint to the lowest word that may hold a
// free id.  take_lowest(n) returns the n smallest free ids in ascending order.
class Allocator {
 public:
  void init(int64_t n) {
    n_ = n;
    bits_.assign((size_t)ceil_div(n, 64), ~0ull);
    if (n % 64) bits_.back() = (1ull << (n % 64)) - 1;
    if (n == 0) bits_.clear();
    free_ = n;
    hint_ = 0;
  }
  int64_t free_count() const { return free_; }
  // Caller checks free_count() >= n first.
  void take_lowest(int64_t n, std::vector<int32_t>& out) {
    size_t w = hint_;
    while (n > 0) {
      while (bits_[w] == 0) ++w;
      uint64_t word = bits_[w];
      while (word && n > 0) {
        int b = __builtin_ctzll(word);
        out.push_back((int32_t)(w * 64 + b));
        word &= word - 1;
        --n;
        --free_;
      }
      bits_[w] = word;
    }
    hint_ = w;
  }
  void give_back(const int32_t* ids, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
      size_t w = (size_t)ids[i] >> 6;
      bits_[w] |= 1ull << (ids[i] & 63);
      if (w < hint_) hint_ = w;
    }
    free_ += n;
  }
  void clear() {
    std::fill(bits_.begin(), bits_.end(), 0ull);
    free_ = 0;
    hint_ = 0;
  }
  // Moves every id of this set into `dst` and empties this set.
  void drain_into(Allocator& dst) {
    std::vector<int32_t> ids;
    take_lowest(free_, ids);
    dst.give_back(ids.data(), (int64_t)ids.size());
  }

 private:
  std::vector<uint64_t> bits_;
  int64_t n_ = 0, free_ = 0;
  size_t hint_ = 0;
};

// A tier's free ids (reading Z9): the lowest free id first.  With s2l_config.alloc_cooling
// (opt-in, a performance choice the paper does not make), the GPU ids released by the most
// recent swap-out ("cooling": their D2H may still be reading them) are handed out only after
// every other free id (lowest first among them); all free ids count for capacity.  It keeps
// appends and swap-ins from landing in blocks a D2H is still reading when others are free.
class TierPool {
 public:
  void init(int64_t n) {
    main_.init(n);
    cool_.init(n);
    cool_.clear();
  }
  int64_t free_count() const { return main_.free_count() + cool_.free_count(); }
  void take_lowest(int64_t n, std::vector<int32_t>& out) {
    const int64_t a = std::min(n, main_.free_count());
    main_.take_lowest(a, out);
    cool_.take_lowest(n - a, out);
  }
  void give_back(const int32_t* ids, int64_t n) { main_.give_back(ids, n); }
  // Starts a new cooling set (the previous one becomes ordinary free ids) with `ids`.
  void give_back_cooling(const int32_t* ids, int64_t n) {
    cool_.drain_into(main_);
    cool_.give_back(ids, n);
  }
  // Adds ids to the current cooling set.
  void give_back_cooling_append(const int32_t* ids, int64_t n) { cool_.give_back(ids, n); }

 private:
  Allocator main_, cool_;
};

struct Request {
  int64_t id = 0;
  std::vector<int32_t> input;
  int64_t nc = 0;
  int32_t tier = S2L_TIER_GPU;
  std::vector<int32_t> blocks;
  int64_t tti = 0;
  int32_t slot = -1;
  uint64_t swap_in_seq = 0;   // in-ring record after the H2D that filled its GPU blocks (0: none)
  uint64_t swap_out_seq = 0;  // out-ring record after the D2H that filled its CPU blocks
  uint64_t write_seq = 0;     // compute-ring record after the last append that wrote its blocks
  uint64_t use_seq = 0;       // compute-ring record after the last append / attention using them
};

// Events re-recorded round-robin on ONE stream.  record() returns a sequence number (1, 2,
// ...); a wait on seq uses slot seq % kN.  If that slot has since been re-recorded by a newer
// operation of the same in-order stream, the wait only lasts longer (never too short), and it
// still refers to work enqueued before the wait, so no cycle between streams can form.
struct EventRing {
  static constexpr int kN = 64;
  cudaEvent_t ev[kN] = {};
  uint64_t seq = 0;
  uint64_t done = 0;   // every record <= done is known to have completed
};

// Pinned-host + device staging ring.  Slot s is reused only after its event (recorded after
// the kernels that read it) has completed, which protects both copies.
struct StagingRing {
  static constexpr int kSlots = 16;
  void* host[kSlots] = {};
  void* dev[kSlots] = {};
  size_t cap[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  bool used[kSlots] = {};
  int next = 0;
};

}  // namespace

struct s2l_ctx {
  s2l_config cfg{};
  bool host_only = true;
  int64_t m_block = 0;
  // swap staging (scattered GPU ids): device buffers per direction, grown on demand up to a cap
  void* stage[2] = {nullptr, nullptr};   // [0] swap-out (D2H), [1] swap-in (H2D)
  size_t stage_cap[2] = {0, 0};
  bool swap_stage = true;                // S2L_SWAP_STAGE=0: DMA every run as it is
  void* gpu_pool = nullptr;
  void* cpu_pool = nullptr;
  cudaStream_t compute = nullptr;
  cudaStream_t copy = nullptr;        // swap-out (D2H)
  cudaStream_t copy_in = nullptr;     // swap-in (H2D): a second stream so both directions overlap
  bool own_copy_stream = false, own_copy_in = false;
  int32_t* d_table = nullptr;          // [max_requests][max_blocks] int32
  std::vector<int32_t> h_table;        // host mirror
  std::vector<int32_t> dirty;          // table entries whose host value must reach the device
  std::vector<uint8_t> dirty_flag;
  TierPool alloc[2];
  std::vector<Request> slots;
  std::vector<int32_t> free_slots;     // stack; lowest slot on top
  std::unordered_map<int64_t, int32_t> by_id;
  StagingRing ring;
  s2l_status sticky = S2L_OK;
  int64_t launches = 0;
  int64_t waits[4] = {};              // s2l_wait_counts: inserted cross-stream waits by kind
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> attn_ev, append_ev, ev_pool;
  // Stream hazards (DESIGN.md §5 "Stream hazards"), tracked per request and per block so
  // that swaps overlap the compute work (and the other copy direction) they do not conflict
  // with.  Rings: compute_ring (one record per append / attention launch), out_ring (one per
  // swap-out, on `copy`), in_ring (one per swap-in, on `copy_in`).
  //  * Request: write_seq / use_seq (compute), swap_in_seq (in), swap_out_seq (out);
  //  * free GPU block: freed_use (compute: previous owner's last use), quar_out (a D2H still
  //    reading it), quar_in (an H2D of a since-freed request still writing it);
  //  * free CPU block: cpu_quar_in (an H2D still reading it).
  // All per-block marks are cleared when the block is allocated again.
  EventRing compute_ring, out_ring, in_ring;
  std::vector<uint64_t> freed_use, quar_out, quar_in, cpu_quar_in;
  unsigned char tmap_kv[256] __attribute__((aligned(64)));
  int32_t num_sms = 148;
  float* split_ws = nullptr;          // tail-wave split partials (num_sms pieces)
  int32_t* split_cnt = nullptr;       // per split unit arrival counters (self-resetting)
  bool split_enabled = true;
  bool split_direct = true;
  int64_t stage_min_runs = 4;         // staged swaps need >= this many id runs (S2L_STAGE_MIN_RUNS)
  int64_t stage_run_bytes = 256 << 10; // ... averaging fewer bytes than this (S2L_STAGE_RUN_BYTES)           // S2L_SPLIT_DIRECT=0: the last piece always merges from the workspace (tests)
  uint32_t* trace_buf = nullptr;      // S2L_TRACE=1: device buffer for kernel timelines (experiments)
  int64_t trace_launch = -1, attn_launch_no = 0;  // which attention launch to trace (S2L_TRACE_LAUNCH)
  bool tc_ok = false;
  s2l::Geometry geo{};
};

namespace {

bool cuda_ok(s2l_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  c->sticky = S2L_E_CUDA;
  fail(S2L_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return false;
}
#define CK(call)                                   \
  do {                                             \
    if (!cuda_ok(c, (call), #call)) return S2L_E_CUDA; \
  } while (0)

bool ring_record(s2l_ctx* c, EventRing& R, cudaStream_t st, uint64_t* seq) {
  const uint64_t n = R.seq + 1;
  if (!cuda_ok(c, cudaEventRecord(R.ev[n % EventRing::kN], st), "event ring record")) return false;
  R.seq = n;
  *seq = n;
  return true;
}
// Orders `st` after record `seq` of ring R.  Records known to be complete cost nothing; a
// record whose slot has been reused is represented by the oldest record still held (later on
// the same in-order stream, so waiting for it is sufficient, and it is usually complete too).
bool ring_wait(s2l_ctx* c, EventRing& R, cudaStream_t st, uint64_t seq) {
  if (seq == 0 || seq <= R.done) return true;
  const uint64_t oldest = R.seq >= (uint64_t)EventRing::kN ? R.seq - EventRing::kN + 1 : 1;
  const uint64_t use = std::max(seq, oldest);
  cudaEvent_t ev = R.ev[use % EventRing::kN];
  const cudaError_t q = cudaEventQuery(ev);
  if (q == cudaSuccess) {
    R.done = std::max(R.done, use);
    return true;
  }
  if (q != cudaErrorNotReady) return cuda_ok(c, q, "event ring query");
  const bool on_compute = st == c->compute;
  ++c->waits[on_compute ? (&R == &c->out_ring ? 0 : 1) : (&R == &c->compute_ring ? 2 : 3)];
  return cuda_ok(c, cudaStreamWaitEvent(st, ev, 0), "event ring wait");
}

s2l_status check_config(const s2l_config* cfg) {
  if (!cfg) return fail(S2L_E_INVAL, "config is NULL");
  const s2l_config& g = *cfg;
  if (g.num_layers < 1 || g.num_q_heads < 1 || g.num_kv_heads < 1 ||
      g.num_q_heads % g.num_kv_heads)
    return fail(S2L_E_INVAL, "bad head geometry (L=%d h=%d h_kv=%d)", g.num_layers,
                g.num_q_heads, g.num_kv_heads);
  if (g.head_dim < 8 || g.head_dim > 256 || g.head_dim % 8)
    return fail(S2L_E_INVAL, "head_dim %d must be a multiple of 8 in [8, 256]", g.head_dim);
  if (g.block_size < 1 || g.block_size > 256 || (g.block_size & (g.block_size - 1)))
    return fail(S2L_E_INVAL, "block_size %d must be a power of two <= 256", g.block_size);
  if (g.num_gpu_blocks < 0 || g.num_cpu_blocks < 0 || g.max_requests < 1 ||
      g.max_blocks_per_request < 1)
    return fail(S2L_E_INVAL, "bad pool / table sizes");
  // token positions and table indices are 32-bit on the device
  if ((int64_t)g.max_blocks_per_request * g.block_size >= (1ll << 31) ||
      (int64_t)g.max_requests * g.max_blocks_per_request >= (1ll << 31))
    return fail(S2L_E_INVAL, "max_blocks_per_request * block_size and max_requests * "
                "max_blocks_per_request must be < 2^31");
  if (g.lcp_block_aligned != 0 && g.lcp_block_aligned != 1)
    return fail(S2L_E_INVAL, "lcp_block_aligned must be 0 or 1");
  if (g.alloc_cooling != 0 && g.alloc_cooling != 1)
    return fail(S2L_E_INVAL, "alloc_cooling must be 0 or 1");
  if (g.kv_dtype != 0 && g.kv_dtype != 1)
    return fail(S2L_E_INVAL, "kv_dtype must be 0 (bf16) or 1 (fp8 e4m3)");
  return S2L_OK;
}

s2l_status init_common(s2l_ctx* c, const s2l_config* cfg) {
  c->cfg = *cfg;
  c->m_block = s2l_block_bytes(cfg);
  c->alloc[S2L_TIER_GPU].init(cfg->num_gpu_blocks);
  c->alloc[S2L_TIER_CPU].init(cfg->num_cpu_blocks);
  c->slots.resize(cfg->max_requests);
  c->free_slots.reserve(cfg->max_requests);
  for (int32_t s = cfg->max_requests - 1; s >= 0; --s) c->free_slots.push_back(s);
  c->h_table.assign((size_t)cfg->max_requests * cfg->max_blocks_per_request, -1);
  c->dirty_flag.assign(c->h_table.size(), 0);
  c->geo = s2l::Geometry{cfg->num_layers, cfg->num_q_heads, cfg->num_kv_heads, cfg->head_dim,
                         cfg->block_size, cfg->max_blocks_per_request, cfg->kv_dtype == 1};
  return S2L_OK;
}

Request* find(s2l_ctx* c, int64_t id) {
  auto it = c->by_id.find(id);
  return it == c->by_id.end() ? nullptr : &c->slots[it->second];
}

// Host mirror of the block table; entries that receive a block id are queued as device
// patches.  Freed entries (-1) are updated on the host only: the kernels read a request's
// entries only below its valid block count (attention: nblk_valid = ceil(kv_len / k); append:
// the staged id list), so the device copy of a freed entry is never read, and resetting it
// would make a release / swap-out of a long request a large patch upload.
void set_table(s2l_ctx* c, int32_t slot, int64_t col, int32_t value) {
  size_t idx = (size_t)slot * c->cfg.max_blocks_per_request + (size_t)col;
  c->h_table[idx] = value;
  if (value >= 0 && !c->dirty_flag[idx]) {
    c->dirty_flag[idx] = 1;
    c->dirty.push_back((int32_t)idx);
  }
}

// Frees blocks [keep, end) of the request on its tier and resets those table entries.
void free_tail(s2l_ctx* c, Request* r, size_t keep) {
  if (keep >= r->blocks.size()) return;
  if (r->tier == S2L_TIER_GPU && r->swap_in_seq && !c->host_only) {
    // blocks possibly still being filled by a swap-in: an append reusing them waits for it
    for (size_t j = keep; j < r->blocks.size(); ++j)
      c->quar_in[(size_t)r->blocks[j]] = std::max(c->quar_in[(size_t)r->blocks[j]], r->swap_in_seq);
    if (keep == 0) r->swap_in_seq = 0;
  }
  c->alloc[r->tier].give_back(r->blocks.data() + keep, (int64_t)(r->blocks.size() - keep));
  if (r->tier == S2L_TIER_GPU)
    for (size_t j = keep; j < r->blocks.size(); ++j) {
      set_table(c, r->slot, (int64_t)j, -1);
      // kernels of this request enqueued so far may still use the block: an H2D reusing it
      // waits for them (an append reusing it is ordered on the compute stream anyway)
      if (!c->host_only) c->freed_use[(size_t)r->blocks[j]] = r->use_seq;
    }
  r->blocks.resize(keep);
}

// ---- staging ring --------------------------------------------------------------------------
// Returns slot index with at least `bytes` of host+device space, or -1 on CUDA error.
int staging_acquire(s2l_ctx* c, size_t bytes) {
  StagingRing& R = c->ring;
  int s = R.next;
  R.next = (R.next + 1) % StagingRing::kSlots;
  if (R.used[s]) {
    if (!cuda_ok(c, cudaEventSynchronize(R.ev[s]), "staging event sync")) return -1;
    R.used[s] = false;
  }
  if (R.cap[s] < bytes) {
    size_t cap = std::max<size_t>(bytes, 64 << 10);
    cap = (cap + 4095) & ~size_t(4095);
    if (R.host[s]) cudaFreeHost(R.host[s]);
    if (R.dev[s]) cudaFree(R.dev[s]);
    R.host[s] = R.dev[s] = nullptr;
    R.cap[s] = 0;
    if (!cuda_ok(c, cudaHostAlloc(&R.host[s], cap, cudaHostAllocDefault), "cudaHostAlloc staging"))
      return -1;
    if (!cuda_ok(c, cudaMalloc(&R.dev[s], cap), "cudaMalloc staging")) return -1;
    R.cap[s] = cap;
  }
  return s;
}

bool staging_upload_and_mark(s2l_ctx* c, int s, size_t bytes) {
  StagingRing& R = c->ring;
  if (bytes && !cuda_ok(c, cudaMemcpyAsync(R.dev[s], R.host[s], bytes, cudaMemcpyHostToDevice,
                                           c->compute), "staging H2D"))
    return false;
  return true;
}

bool staging_release(s2l_ctx* c, int s) {
  StagingRing& R = c->ring;
  if (!cuda_ok(c, cudaEventRecord(R.ev[s], c->compute), "staging event record")) return false;
  R.used[s] = true;
  return true;
}

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Packs the dirty table entries into dst (as TablePatch) and clears the dirty set.
int32_t take_patches(s2l_ctx* c, s2l::TablePatch* dst) {
  int32_t n = 0;
  for (int32_t idx : c->dirty) {
    dst[n++] = s2l::TablePatch{idx, c->h_table[idx]};
    c->dirty_flag[idx] = 0;
  }
  c->dirty.clear();
  return n;
}

// Event pairs for per-kernel timing.
std::pair<cudaEvent_t, cudaEvent_t> timing_pair(s2l_ctx* c) {
  if (!c->ev_pool.empty()) {
    auto p = c->ev_pool.back();
    c->ev_pool.pop_back();
    return p;
  }
  std::pair<cudaEvent_t, cudaEvent_t> p{nullptr, nullptr};
  cudaEventCreate(&p.first);
  cudaEventCreate(&p.second);
  return p;
}


// Flush pending table patches with a standalone patch kernel (used before attention when no
// append kernel carried them).
s2l_status flush_patches(s2l_ctx* c) {
  if (c->dirty.empty()) return S2L_OK;
  if ((int64_t)c->dirty.size() <= s2l::kInlinePatches) {   // by value: no copy-engine upload
    std::vector<s2l::TablePatch> ps(c->dirty.size());
    int32_t n = take_patches(c, ps.data());
    CK(s2l::launch_table_patch_inline(ps.data(), n, c->d_table, c->compute));
    c->launches++;
    return S2L_OK;
  }
  size_t bytes = c->dirty.size() * sizeof(s2l::TablePatch);
  int s = staging_acquire(c, bytes);
  if (s < 0) return S2L_E_CUDA;
  int32_t n = take_patches(c, (s2l::TablePatch*)c->ring.host[s]);
  if (!staging_upload_and_mark(c, s, bytes)) return S2L_E_CUDA;
  CK(s2l::launch_table_patch((const s2l::TablePatch*)c->ring.dev[s], n, c->d_table, c->compute));
  c->launches++;
  if (!staging_release(c, s)) return S2L_E_CUDA;
  return S2L_OK;
}

s2l_status swap_impl(s2l_ctx* c, int32_t n_reqs, const int64_t* ids, int64_t* bytes_out,
                     int32_t src, int32_t dst) {
  if (bytes_out) *bytes_out = 0;
  if (n_reqs < 0 || (n_reqs > 0 && !ids)) return fail(S2L_E_INVAL, "bad request list");
  std::unordered_set<int64_t> seen;
  int64_t need = 0;
  for (int32_t i = 0; i < n_reqs; ++i) {
    Request* r = find(c, ids[i]);
    if (!r) return fail(S2L_E_NO_REQUEST, "unknown request %lld", (long long)ids[i]);
    if (!seen.insert(ids[i]).second) return fail(S2L_E_INVAL, "request %lld repeated", (long long)ids[i]);
    if (r->tier != src) return fail(S2L_E_STATE, "request %lld is not on the %s tier",
                                    (long long)ids[i], src == S2L_TIER_GPU ? "GPU" : "CPU");
    need += (int64_t)r->blocks.size();
  }
  if (need > c->alloc[dst].free_count())
    return fail(dst == S2L_TIER_CPU ? S2L_E_NO_CPU_BLOCKS : S2L_E_NO_GPU_BLOCKS,
                "swap needs %lld blocks, %lld free", (long long)need,
                (long long)c->alloc[dst].free_count());
  if (c->sticky) return fail(c->sticky, "context has a sticky CUDA error");

  // ---- bookkeeping (identical in host-only contexts) ----
  std::vector<std::pair<int32_t, int32_t>> moves;  // (src id, dst id) in request/block order
  moves.reserve((size_t)need);
  std::vector<Request*> touched;
  for (int32_t i = 0; i < n_reqs; ++i) {
    Request* r = find(c, ids[i]);
    std::vector<int32_t> nid;
    nid.reserve(r->blocks.size());
    c->alloc[dst].take_lowest((int64_t)r->blocks.size(), nid);
    for (size_t j = 0; j < nid.size(); ++j) moves.emplace_back(r->blocks[j], nid[j]);
    if (src == S2L_TIER_GPU && !c->host_only)
      for (int32_t b : r->blocks) c->freed_use[(size_t)b] = r->use_seq;
    if (src == S2L_TIER_GPU && c->cfg.alloc_cooling) {   // opt-in: ids cool until the next swap-out
      if (i == 0) c->alloc[src].give_back_cooling(nullptr, 0);
      c->alloc[src].give_back_cooling_append(r->blocks.data(), (int64_t)r->blocks.size());
    } else {
      c->alloc[src].give_back(r->blocks.data(), (int64_t)r->blocks.size());
    }
    for (size_t j = 0; j < nid.size(); ++j)
      set_table(c, r->slot, (int64_t)j, dst == S2L_TIER_GPU ? nid[j] : -1);
    r->blocks.swap(nid);
    r->tier = dst;
    touched.push_back(r);
  }
  if (bytes_out) *bytes_out = need * c->m_block;
  if (c->host_only || need == 0) return S2L_OK;

  // ---- copies on the copy stream: order only against the compute work they conflict with --
  cudaStream_t st = (src == S2L_TIER_GPU) ? c->copy : c->copy_in;
  uint64_t wc = 0, wo = 0, wi = 0;   // waits on the compute / out / in rings
  if (src == S2L_TIER_GPU) {
    // D2H reads GPU blocks written by the requests' appends (compute) or swap-ins (in), and
    // writes CPU blocks an earlier H2D may still be reading (cpu_quar_in).
    for (Request* r : touched) {
      wc = std::max(wc, r->write_seq);
      wi = std::max(wi, r->swap_in_seq);
    }
    for (const auto& m : moves) {
      wi = std::max(wi, c->cpu_quar_in[(size_t)m.second]);
      c->cpu_quar_in[(size_t)m.second] = 0;
    }
  } else {
    // H2D reads CPU blocks written by the requests' swap-outs (out) and overwrites free GPU
    // blocks that kernels of their previous owner (freed_use), a D2H (quar_out) or an
    // earlier H2D on this stream (quar_in, ordered) may still touch.
    for (Request* r : touched) wo = std::max(wo, r->swap_out_seq);
    for (const auto& m : moves) {
      const size_t b = (size_t)m.second;
      wc = std::max(wc, c->freed_use[b]);
      wo = std::max(wo, c->quar_out[b]);
      c->freed_use[b] = c->quar_out[b] = c->quar_in[b] = 0;
    }
  }
  if (!ring_wait(c, c->compute_ring, st, wc) || !ring_wait(c, c->out_ring, st, wo) ||
      !ring_wait(c, c->in_ring, st, wi))
    return S2L_E_CUDA;
  // Coalesce runs where both source and destination ids are consecutive (the lowest-free
  // allocator makes these long when the pools are not fragmented).
  char* gbase = (char*)c->gpu_pool;
  char* hbase = (char*)c->cpu_pool;
  const cudaMemcpyKind kind = dst == S2L_TIER_GPU ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  // One cudaMemcpyAsync per coalesced run (the batched-copy entry points are not used: they
  // are closed on the GPU pool this build runs on); many short runs take the staged path below.
  auto dma = [&](std::vector<void*>& dsts, std::vector<void*>& srcs, std::vector<size_t>& sizes) -> bool {
    for (size_t i = 0; i < sizes.size(); ++i)
      if (!cuda_ok(c, cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], kind, st), "swap copy")) return false;
    return true;
  };
  size_t runs = 0;
  for (size_t i = 0; i < moves.size(); ++i)
    if (i == 0 || moves[i].first != moves[i - 1].first + 1 || moves[i].second != moves[i - 1].second + 1) ++runs;
  // Scattered GPU ids (short runs): stage through device memory so that every run of
  // consecutive HOST ids is one DMA -- swap-out gathers the GPU blocks into a contiguous
  // staging buffer (one kernel, HBM -> HBM) and copies it out; swap-in copies in and scatters.
  // Measured (profiles/r02/c4_swap_grid.jsonl, profiles/r02s2/swap_stage_*.jsonl): with one DMA per
  // run, 64 KiB random ids reach 0.31 / 0.42 of the link at 16 / 32 blocks; staged from 4 runs on,
  // 0.58 / 0.73; 512 KiB blocks in ~1 MiB runs: 0.82 -> 0.92-0.94 staged at 64 / 512 blocks, but
  // 0.80 -> 0.62 at 8 blocks (4 MiB); 2 MiB blocks stream at 0.94 unstaged and lose staged.  Below
  // ~8 x 64 KiB the fixed per-transfer latency bounds either way (a contiguous 512 KiB copy
  // reaches 0.52-0.55 of the link).
  // Staged when there are enough runs and they are short: avg < stage_run_bytes (256 KiB), or
  // avg < 2 MiB for a transfer of >= 16 MiB (the gather / scatter of a small transfer costs
  // more than the per-DMA latency it saves; large runs stream at the link rate anyway).
  const int64_t tot_bytes = (int64_t)moves.size() * c->m_block;
  const bool staged = c->swap_stage && (int64_t)runs >= c->stage_min_runs && c->m_block % 16 == 0 &&
                      (tot_bytes < c->stage_run_bytes * (int64_t)runs ||
                       (tot_bytes >= (16ll << 20) && tot_bytes < (2ll << 20) * (int64_t)runs));
  if (staged) {
    const int dir = dst == S2L_TIER_GPU ? 1 : 0;
    const size_t cap_bytes = std::max<size_t>((size_t)c->m_block, (size_t)64 << 20);
    const size_t per = std::min<size_t>({(size_t)s2l::kSwapIdsPerLaunch, cap_bytes / (size_t)c->m_block,
                                         moves.size()});
    const size_t want = per * (size_t)c->m_block;
    if (c->stage_cap[dir] < want) {
      if (c->stage[dir] && !cuda_ok(c, cudaStreamSynchronize(st), "staging resize sync")) return S2L_E_CUDA;
      if (c->stage[dir]) cudaFree(c->stage[dir]);
      c->stage[dir] = nullptr;
      c->stage_cap[dir] = 0;
      CK(cudaMalloc(&c->stage[dir], want));
      c->stage_cap[dir] = want;
    }
    char* sbase = (char*)c->stage[dir];
    std::vector<int32_t> gids;
    for (size_t c0 = 0; c0 < moves.size(); c0 += per) {
      const size_t n = std::min(per, moves.size() - c0);
      gids.clear();
      std::vector<void*> dsts, srcs;
      std::vector<size_t> sizes;
      for (size_t i = 0; i < n;) {                          // runs of consecutive host ids
        const auto& m0 = moves[c0 + i];
        const int32_t h0 = dir ? m0.first : m0.second;
        size_t j = i + 1;
        while (j < n && (dir ? moves[c0 + j].first : moves[c0 + j].second) == h0 + (int32_t)(j - i)) ++j;
        char* hp = hbase + (size_t)h0 * c->m_block;
        char* sp = sbase + i * (size_t)c->m_block;
        dsts.push_back(dir ? (void*)sp : (void*)hp);
        srcs.push_back(dir ? (void*)hp : (void*)sp);
        sizes.push_back((j - i) * (size_t)c->m_block);
        i = j;
      }
      for (size_t i = 0; i < n; ++i) gids.push_back(dir ? moves[c0 + i].second : moves[c0 + i].first);
      if (!dir) {
        CK(s2l::launch_swap_stage(gids.data(), (int32_t)n, c->gpu_pool, sbase, c->m_block, true, st));
        c->launches++;
      }
      if (!dma(dsts, srcs, sizes)) return S2L_E_CUDA;
      if (dir) {
        CK(s2l::launch_swap_stage(gids.data(), (int32_t)n, c->gpu_pool, sbase, c->m_block, false, st));
        c->launches++;
      }
    }
  } else {
    std::vector<void*> dsts, srcs;
    std::vector<size_t> sizes;
    for (size_t i = 0; i < moves.size();) {
      size_t j = i + 1;
      while (j < moves.size() && moves[j].first == moves[j - 1].first + 1 &&
             moves[j].second == moves[j - 1].second + 1)
        ++j;
      size_t nb = j - i;
      char* s_ptr = (src == S2L_TIER_GPU ? gbase : hbase) + (size_t)moves[i].first * c->m_block;
      char* d_ptr = (dst == S2L_TIER_GPU ? gbase : hbase) + (size_t)moves[i].second * c->m_block;
      srcs.push_back(s_ptr);
      dsts.push_back(d_ptr);
      sizes.push_back(nb * (size_t)c->m_block);
      i = j;
    }
    if (!dma(dsts, srcs, sizes)) return S2L_E_CUDA;
  }
  uint64_t seq = 0;
  if (src == S2L_TIER_GPU) {
    if (!ring_record(c, c->out_ring, st, &seq)) return S2L_E_CUDA;
    for (const auto& m : moves) c->quar_out[(size_t)m.first] = seq;   // freed GPU ids
    for (Request* r : touched) r->swap_out_seq = seq;
  } else {
    if (!ring_record(c, c->in_ring, st, &seq)) return S2L_E_CUDA;
    for (const auto& m : moves) c->cpu_quar_in[(size_t)m.first] = seq;   // freed CPU ids
    for (Request* r : touched) r->swap_in_seq = seq;
  }
  return S2L_OK;
}

}  // namespace

// =========================================================================================
extern "C" {

int64_t s2l_block_bytes(const s2l_config* cfg) {
  if (!cfg || cfg->num_layers < 1 || cfg->num_kv_heads < 1 || cfg->head_dim < 1 ||
      cfg->block_size < 1)
    return -1;
  return 2ll * cfg->num_layers * cfg->block_size * cfg->num_kv_heads * cfg->head_dim * (cfg->kv_dtype == 1 ? 1ll : 2ll);
}

s2l_status s2l_create_host_only(const s2l_config* cfg, s2l_ctx** out) {
  if (!out) return fail(S2L_E_INVAL, "out is NULL");
  *out = nullptr;
  s2l_status st = check_config(cfg);
  if (st) return st;
  auto* c = new s2l_ctx();
  c->host_only = true;
  init_common(c, cfg);
  *out = c;
  return S2L_OK;
}

s2l_status s2l_create(const s2l_config* cfg, void* gpu_pool, void* cpu_pool_pinned,
                      void* compute_stream, void* copy_stream, s2l_ctx** out) {
  if (!out) return fail(S2L_E_INVAL, "out is NULL");
  *out = nullptr;
  s2l_status st = check_config(cfg);
  if (st) return st;
  if (!gpu_pool && cfg->num_gpu_blocks > 0) return fail(S2L_E_INVAL, "gpu_pool is NULL");
  if (!cpu_pool_pinned && cfg->num_cpu_blocks > 0) return fail(S2L_E_INVAL, "cpu_pool is NULL");
  if (((uintptr_t)gpu_pool) & 255) return fail(S2L_E_INVAL, "gpu_pool must be 256-byte aligned");
  std::unique_ptr<s2l_ctx> holder(new s2l_ctx());
  s2l_ctx* c = holder.get();
  c->host_only = false;
  init_common(c, cfg);
  c->gpu_pool = gpu_pool;
  c->cpu_pool = cpu_pool_pinned;
  c->compute = (cudaStream_t)compute_stream;
  c->copy = (cudaStream_t)copy_stream;
  if (!c->copy) {
    CK(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
    c->own_copy_stream = true;
  }
  CK(cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking));
  c->own_copy_in = true;
  CK(cudaMalloc(&c->d_table, c->h_table.size() * sizeof(int32_t)));
  CK(cudaMemsetAsync(c->d_table, 0xFF, c->h_table.size() * sizeof(int32_t), c->compute));
  size_t gbytes = (size_t)cfg->num_gpu_blocks * (size_t)c->m_block;
  if (gbytes) CK(cudaMemsetAsync(gpu_pool, 0, gbytes, c->compute));
  size_t hbytes = (size_t)cfg->num_cpu_blocks * (size_t)c->m_block;
  if (hbytes) memset(cpu_pool_pinned, 0, hbytes);
  for (int s = 0; s < StagingRing::kSlots; ++s)
    CK(cudaEventCreateWithFlags(&c->ring.ev[s], cudaEventDisableTiming));
  for (EventRing* R : {&c->compute_ring, &c->out_ring, &c->in_ring})
    for (int i = 0; i < EventRing::kN; ++i) CK(cudaEventCreateWithFlags(&R->ev[i], cudaEventDisableTiming));
  c->freed_use.assign((size_t)cfg->num_gpu_blocks, 0);
  c->quar_out.assign((size_t)cfg->num_gpu_blocks, 0);
  c->quar_in.assign((size_t)cfg->num_gpu_blocks, 0);
  c->cpu_quar_in.assign((size_t)cfg->num_cpu_blocks, 0);
  {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  c->tc_ok = s2l::attn_tc_supported(c->geo);
  if (c->tc_ok && cfg->num_gpu_blocks > 0) {
    const char* err = nullptr;
    if (!s2l::make_tmap_kv(c->tmap_kv, gpu_pool, cfg->num_gpu_blocks, cfg->num_layers,
                           cfg->num_kv_heads, cfg->head_dim, cfg->block_size, c->geo.fp8, &err))
      return fail(S2L_E_CUDA, "tensor map (pool): %s", err ? err : "?");
  } else {
    c->tc_ok = false;
  }
  if (c->tc_ok) {
    CK(cudaMalloc(&c->split_ws, (size_t)c->num_sms * s2l::kSplitPieceFloats * sizeof(float)));
    CK(cudaMalloc(&c->split_cnt, (size_t)c->num_sms * sizeof(int32_t)));
    CK(cudaMemsetAsync(c->split_cnt, 0, (size_t)c->num_sms * sizeof(int32_t), c->compute));
    const char* e = getenv("S2L_NO_SPLIT");
    c->split_enabled = !(e && e[0] == '1');
    e = getenv("S2L_SPLIT_DIRECT");
    c->split_direct = !(e && e[0] == '0');
    e = getenv("S2L_SWAP_STAGE");
    c->swap_stage = !(e && e[0] == '0');
    e = getenv("S2L_STAGE_MIN_RUNS");
    if (e && atoll(e) > 0) c->stage_min_runs = atoll(e);
    e = getenv("S2L_STAGE_RUN_BYTES");
    if (e && atoll(e) > 0) c->stage_run_bytes = atoll(e);

    e = getenv("S2L_TRACE");
    if (e && e[0] == '1') {
      CK(cudaMalloc(&c->trace_buf, ((size_t)1 << 20)));
      CK(cudaMemsetAsync(c->trace_buf, 0, ((size_t)1 << 20), c->compute));
      const char* tl = getenv("S2L_TRACE_LAUNCH");
      c->trace_launch = tl ? atoll(tl) : 0;
    }
  }
  CK(cudaStreamSynchronize(c->compute));
  *out = holder.release();
  return S2L_OK;
}

void s2l_destroy(s2l_ctx* c) {
  if (!c) return;
  if (!c->host_only) {
    cudaStreamSynchronize(c->compute);
    cudaStreamSynchronize(c->copy);
    if (c->copy_in) cudaStreamSynchronize(c->copy_in);
    for (int s = 0; s < StagingRing::kSlots; ++s) {
      if (c->ring.host[s]) cudaFreeHost(c->ring.host[s]);
      if (c->ring.dev[s]) cudaFree(c->ring.dev[s]);
      if (c->ring.ev[s]) cudaEventDestroy(c->ring.ev[s]);
    }
    for (EventRing* R : {&c->compute_ring, &c->out_ring, &c->in_ring})
      for (int i = 0; i < EventRing::kN; ++i)
        if (R->ev[i]) cudaEventDestroy(R->ev[i]);
    for (auto* v : {&c->attn_ev, &c->append_ev, &c->ev_pool})
      for (auto& p : *v) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
      }
    if (c->trace_buf) {   // experiments: dump the recorded timeline
      std::vector<uint32_t> h(((size_t)1 << 20) / sizeof(uint32_t));
      cudaMemcpy(h.data(), c->trace_buf, h.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost);
      const char* path = getenv("S2L_TRACE_FILE");
      if (FILE* f = fopen(path ? path : "s2l_trace.bin", "wb")) {
        fwrite(h.data(), sizeof(uint32_t), h.size(), f);
        fclose(f);
      }
      cudaFree(c->trace_buf);
    }
    if (c->split_ws) cudaFree(c->split_ws);
    for (void* sp : c->stage)
      if (sp) cudaFree(sp);
    if (c->split_cnt) cudaFree(c->split_cnt);
    if (c->d_table) cudaFree(c->d_table);
    if (c->own_copy_stream) cudaStreamDestroy(c->copy);
    if (c->own_copy_in && c->copy_in) cudaStreamDestroy(c->copy_in);
  }
  delete c;
}

s2l_status s2l_new_request(s2l_ctx* c, int64_t id, const int32_t* tokens, int64_t n) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  if (n < 0 || (n > 0 && !tokens)) return fail(S2L_E_INVAL, "bad token array");
  if (c->by_id.count(id)) return fail(S2L_E_STATE, "request %lld already exists", (long long)id);
  if (c->free_slots.empty()) return fail(S2L_E_CAPACITY, "request table full");
  int32_t slot = c->free_slots.back();
  c->free_slots.pop_back();
  Request& r = c->slots[slot];
  r = Request();
  r.id = id;
  r.slot = slot;
  r.input.assign(tokens, tokens + n);
  c->by_id[id] = slot;
  return S2L_OK;
}

s2l_status s2l_release_request(s2l_ctx* c, int64_t id) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  Request* r = find(c, id);
  if (!r) return fail(S2L_E_NO_REQUEST, "unknown request %lld", (long long)id);
  free_tail(c, r, 0);
  r->swap_in_seq = 0;
  c->by_id.erase(id);
  c->free_slots.push_back(r->slot);
  return S2L_OK;
}

s2l_status s2l_preempt_recompute(s2l_ctx* c, int64_t id) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  Request* r = find(c, id);
  if (!r) return fail(S2L_E_NO_REQUEST, "unknown request %lld", (long long)id);
  free_tail(c, r, 0);
  r->nc = 0;
  r->tier = S2L_TIER_GPU;
  r->swap_in_seq = 0;
  return S2L_OK;
}

s2l_status s2l_append_chunk(s2l_ctx* c, int32_t n_items, const s2l_append_item* items,
                            const void* k, const void* v, int64_t kv_rows) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  if (n_items < 0 || (n_items > 0 && !items)) return fail(S2L_E_INVAL, "bad item array");
  const int64_t kb = c->cfg.block_size;
  std::unordered_set<int64_t> seen;
  int64_t need = 0, total_rows = 0, total_ids = 0;
  for (int32_t i = 0; i < n_items; ++i) {
    const s2l_append_item& it = items[i];
    Request* r = find(c, it.req_id);
    if (!r) return fail(S2L_E_NO_REQUEST, "item %d: unknown request %lld", i, (long long)it.req_id);
    if (!seen.insert(it.req_id).second)
      return fail(S2L_E_INVAL, "item %d: request %lld repeated", i, (long long)it.req_id);
    // reading Z19: tokens may arrive while a request is swapped out (a preempted
    // request keeps receiving input); writing K/V needs the GPU tier
    if (r->tier != S2L_TIER_GPU && it.n_kv != 0)
      return fail(S2L_E_STATE, "item %d: request %lld is swapped out", i, (long long)it.req_id);
    if (it.n_tokens < 0 || it.n_kv < 0 || it.kv_row < 0 || (it.n_tokens > 0 && !it.tokens))
      return fail(S2L_E_INVAL, "item %d: negative sizes or NULL tokens", i);
    if (it.n_kv > 0 && it.kv_row + it.n_kv > kv_rows)
      return fail(S2L_E_INVAL, "item %d: rows [%lld,%lld) beyond kv_rows %lld", i,
                  (long long)it.kv_row, (long long)(it.kv_row + it.n_kv), (long long)kv_rows);
    if (it.n_kv > (int64_t)r->input.size() + it.n_tokens - r->nc)
      return fail(S2L_E_INVAL, "item %d: n_kv %lld exceeds pending tokens", i, (long long)it.n_kv);
    int64_t nb = ceil_div(r->nc + it.n_kv, kb);
    if (nb > c->cfg.max_blocks_per_request)
      return fail(S2L_E_INVAL, "item %d: %lld blocks exceed max_blocks_per_request", i, (long long)nb);
    need += nb - (int64_t)r->blocks.size();
    total_rows += it.n_kv;
    if (it.n_kv) total_ids += nb - r->nc / kb;
  }
  if (need > c->alloc[S2L_TIER_GPU].free_count())
    return fail(S2L_E_NO_GPU_BLOCKS, "append needs %lld blocks, %lld free", (long long)need,
                (long long)c->alloc[S2L_TIER_GPU].free_count());
  // k = v = NULL on a device context: reserve (NEXT-2) -- allocate and advance nc, the K/V of
  // each layer is written later by s2l_prefill_append
  if (!c->host_only && (!k) != (!v)) return fail(S2L_E_INVAL, "exactly one of k/v is NULL");
  const bool reserve = !k;
  if (c->host_only && (k || v)) return fail(S2L_E_STATE, "host-only context cannot write K/V");
  if (c->sticky) return fail(c->sticky, "context has a sticky CUDA error");

  // Staging layout: [AppendItemDev x n_items][int32 ids x total_ids][TablePatch x patches]
  std::vector<s2l::AppendItemDev> dev_items;
  std::vector<int32_t> ids;
  std::vector<Request*> wait_in, written;
  uint64_t quar_wait = 0, quar_wait_in = 0;   // newest D2H / H2D still touching a block reallocated here
  dev_items.reserve(n_items);
  ids.reserve((size_t)total_ids);
  int64_t row_begin = 0;
  for (int32_t i = 0; i < n_items; ++i) {
    const s2l_append_item& it = items[i];
    Request* r = find(c, it.req_id);
    if (it.n_tokens) r->input.insert(r->input.end(), it.tokens, it.tokens + it.n_tokens);
    int64_t nb = ceil_div(r->nc + it.n_kv, kb);
    size_t held = r->blocks.size();
    c->alloc[S2L_TIER_GPU].take_lowest(nb - (int64_t)held, r->blocks);
    for (size_t j = held; j < r->blocks.size(); ++j) set_table(c, r->slot, (int64_t)j, r->blocks[j]);
    if (!c->host_only)
      for (size_t j = held; j < r->blocks.size(); ++j) {
        const size_t b = (size_t)r->blocks[j];
        quar_wait = std::max(quar_wait, c->quar_out[b]);
        quar_wait_in = std::max(quar_wait_in, c->quar_in[b]);
        c->quar_out[b] = c->quar_in[b] = c->freed_use[b] = 0;
      }
    if (it.n_kv) {
      s2l::AppendItemDev d{};
      d.nc = r->nc;
      d.n_kv = it.n_kv;
      d.kv_row = it.kv_row;
      d.row_begin = row_begin;
      d.id_off = (int32_t)ids.size();
      for (int64_t b = r->nc / kb; b < nb; ++b) ids.push_back(r->blocks[(size_t)b]);
      dev_items.push_back(d);
      row_begin += it.n_kv;
      if (r->swap_in_seq) wait_in.push_back(r);
      written.push_back(r);
    }
    r->nc += it.n_kv;
  }
  if (c->host_only) return S2L_OK;
  if (total_rows == 0 || reserve) {
    if (!ring_wait(c, c->out_ring, c->compute, quar_wait) || !ring_wait(c, c->in_ring, c->compute, quar_wait_in))
      return S2L_E_CUDA;
    // reserve: the new entries stay pending; a fused s2l_prefill_append writes them in-kernel,
    // any other launch reading the table flushes them first
    return reserve ? S2L_OK : flush_patches(c);
  }

  size_t off_ids = align16(dev_items.size() * sizeof(s2l::AppendItemDev));
  size_t off_patch = align16(off_ids + ids.size() * sizeof(int32_t));
  size_t bytes = off_patch + c->dirty.size() * sizeof(s2l::TablePatch);
  // Small calls pass their descriptors by value in the kernel parameters; a staged upload
  // would queue on the copy engine behind bulk H2D traffic and stall the compute stream.
  const bool inl = bytes <= (size_t)s2l::kInlineBytes;
  int s = -1;
  char* h = nullptr;
  std::unique_ptr<s2l::InlineBlob> blob;
  if (inl) {
    blob.reset(new s2l::InlineBlob());
    h = (char*)blob->b;
  } else {
    s = staging_acquire(c, bytes);
    if (s < 0) return S2L_E_CUDA;
    h = (char*)c->ring.host[s];
  }
  memcpy(h, dev_items.data(), dev_items.size() * sizeof(s2l::AppendItemDev));
  memcpy(h + off_ids, ids.data(), ids.size() * sizeof(int32_t));
  int32_t n_patch = take_patches(c, (s2l::TablePatch*)(h + off_patch));
  if (!inl && !staging_upload_and_mark(c, s, bytes)) return S2L_E_CUDA;
  if (!ring_wait(c, c->out_ring, c->compute, quar_wait) || !ring_wait(c, c->in_ring, c->compute, quar_wait_in))
    return S2L_E_CUDA;
  for (Request* r : wait_in) {
    if (!ring_wait(c, c->in_ring, c->compute, r->swap_in_seq)) return S2L_E_CUDA;
  }
  std::pair<cudaEvent_t, cudaEvent_t> tp{};
  if (c->timing) {
    tp = timing_pair(c);
    CK(cudaEventRecord(tp.first, c->compute));
  }
  if (inl) {
    CK(s2l::launch_append_inline(c->geo, *blob, (int32_t)dev_items.size(), total_rows,
                                 (int32_t)off_ids, (int32_t)ids.size(), (int32_t)off_patch, n_patch,
                                 c->d_table, k, v, kv_rows, c->gpu_pool, c->compute));
  } else {
    char* dv = (char*)c->ring.dev[s];
    CK(s2l::launch_append(c->geo, (const s2l::AppendItemDev*)dv, (int32_t)dev_items.size(),
                          total_rows, (const int32_t*)(dv + off_ids), (int32_t)ids.size(),
                          (const s2l::TablePatch*)(dv + off_patch), n_patch, c->d_table, k, v,
                          kv_rows, c->gpu_pool, c->compute));
  }
  c->launches++;
  if (c->timing) {
    CK(cudaEventRecord(tp.second, c->compute));
    c->append_ev.push_back(tp);
  }
  uint64_t wseq = 0;
  if (!ring_record(c, c->compute_ring, c->compute, &wseq)) return S2L_E_CUDA;
  for (Request* r : written) r->write_seq = r->use_seq = wseq;
  if (!inl && !staging_release(c, s)) return S2L_E_CUDA;
  return S2L_OK;
}

s2l_status s2l_invalidate_lcp(s2l_ctx* c, int64_t id, const int32_t* new_tokens, int64_t new_len,
                              int64_t* lcp_out, int64_t* inval_out) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  if (new_len < 0 || (new_len > 0 && !new_tokens)) return fail(S2L_E_INVAL, "bad token array");
  Request* r = find(c, id);
  if (!r) return fail(S2L_E_NO_REQUEST, "unknown request %lld", (long long)id);
  // a1: LCP by a word-wise compare (8 tokens per 32-byte step), then the exact tail.
  const int32_t* a = r->input.data();
  int64_t n = std::min<int64_t>((int64_t)r->input.size(), new_len);
  int64_t p = 0;
  while (p + 8 <= n && memcmp(a + p, new_tokens + p, 32) == 0) p += 8;
  while (p < n && a[p] == new_tokens[p]) ++p;
  // a2: invalidate beyond b = min(p, nc) (Z5), keep ceil(b/k) blocks (Z4 / S:L191 variant).
  const int64_t kb = c->cfg.block_size;
  int64_t b = std::min(p, r->nc);
  if (c->cfg.lcp_block_aligned) b = (b / kb) * kb;
  size_t keep = (size_t)ceil_div(b, kb);
  free_tail(c, r, keep);
  int64_t inval = r->nc - b;
  r->nc = b;
  r->tti += inval;
  r->input.assign(new_tokens, new_tokens + new_len);
  if (r->tier == S2L_TIER_CPU && keep == 0) r->tier = S2L_TIER_GPU;
  if (lcp_out) *lcp_out = p;
  if (inval_out) *inval_out = inval;
  return S2L_OK;
}

// One layer's append of the chunk rows [q_pos, q_pos+n_q) of each item from k/v rows
// [q_row, q_row+n_q) ([q_rows][h_kv][d]) by the append kernel (fallback of the fused path).
static s2l_status layer_append(s2l_ctx* c, int32_t layer, int32_t n_items,
                               const s2l_prefill_item* items, const void* k, const void* v,
                               int64_t q_rows) {
  const int64_t kb = c->cfg.block_size;
  std::vector<s2l::AppendItemDev> dev_items;
  std::vector<int32_t> ids;
  int64_t row_begin = 0;
  for (int32_t i = 0; i < n_items; ++i) {
    const s2l_prefill_item& it = items[i];
    Request* r = find(c, it.req_id);
    s2l::AppendItemDev d{};
    d.nc = it.q_pos;
    d.n_kv = it.n_q;
    d.kv_row = it.q_row;
    d.row_begin = row_begin;
    d.id_off = (int32_t)ids.size();
    for (int64_t b = it.q_pos / kb; b < ceil_div(it.q_pos + it.n_q, kb); ++b) ids.push_back(r->blocks[(size_t)b]);
    dev_items.push_back(d);
    row_begin += it.n_q;
  }
  size_t off_ids = align16(dev_items.size() * sizeof(s2l::AppendItemDev));
  size_t bytes = align16(off_ids + ids.size() * sizeof(int32_t));
  if (bytes <= (size_t)s2l::kInlineBytes) {
    std::unique_ptr<s2l::InlineBlob> blob(new s2l::InlineBlob());
    memcpy(blob->b, dev_items.data(), dev_items.size() * sizeof(s2l::AppendItemDev));
    memcpy(blob->b + off_ids, ids.data(), ids.size() * sizeof(int32_t));
    CK(s2l::launch_append_inline(c->geo, *blob, n_items, row_begin, (int32_t)off_ids,
                                 (int32_t)ids.size(), (int32_t)bytes, 0, c->d_table, k, v, q_rows,
                                 c->gpu_pool, c->compute, layer, 1));
  } else {
    int s = staging_acquire(c, bytes);
    if (s < 0) return S2L_E_CUDA;
    char* h = (char*)c->ring.host[s];
    memcpy(h, dev_items.data(), dev_items.size() * sizeof(s2l::AppendItemDev));
    memcpy(h + off_ids, ids.data(), ids.size() * sizeof(int32_t));
    if (!staging_upload_and_mark(c, s, bytes)) return S2L_E_CUDA;
    char* dv = (char*)c->ring.dev[s];
    CK(s2l::launch_append(c->geo, (const s2l::AppendItemDev*)dv, n_items, row_begin,
                          (const int32_t*)(dv + off_ids), (int32_t)ids.size(), nullptr, 0,
                          c->d_table, k, v, q_rows, c->gpu_pool, c->compute, layer, 1));
    if (!staging_release(c, s)) return S2L_E_CUDA;
  }
  c->launches++;
  return S2L_OK;
}

// s2l_prefill_batch, and with k/v != NULL s2l_prefill_append (NEXT-2: the chunk's K/V of this
// layer are written to the pool by the attention kernel itself when every q_pos is
// block-aligned, else by a one-layer append launch before it).
static s2l_status prefill_impl(s2l_ctx* c, int32_t layer, int32_t n_items,
                               const s2l_prefill_item* items, const void* q, const void* k,
                               const void* v, void* o, float* lse, int64_t q_rows) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  if (c->host_only) return fail(S2L_E_STATE, "host-only context has no device");
  if (n_items < 0 || (n_items > 0 && !items)) return fail(S2L_E_INVAL, "bad item array");
  if (layer < 0 || layer >= c->cfg.num_layers) return fail(S2L_E_INVAL, "layer %d out of range", layer);
  for (int32_t i = 0; i < n_items; ++i) {
    const s2l_prefill_item& it = items[i];
    Request* r = find(c, it.req_id);
    if (!r) return fail(S2L_E_NO_REQUEST, "item %d: unknown request %lld", i, (long long)it.req_id);
    if (r->tier != S2L_TIER_GPU)
      return fail(S2L_E_STATE, "item %d: request %lld is swapped out", i, (long long)it.req_id);
    if (it.n_q < 1 || it.q_pos < 0 || it.q_row < 0 || it.q_pos + it.n_q > r->nc ||
        it.q_row + it.n_q > q_rows || it.n_q > (1ll << 30))
      return fail(S2L_E_INVAL, "item %d: bad q range (q_pos %lld n_q %lld nc %lld)", i,
                  (long long)it.q_pos, (long long)it.n_q, (long long)r->nc);
  }
  if (n_items > 0 && (!q || !o)) return fail(S2L_E_INVAL, "q/o is NULL");
  const bool append = k != nullptr;
  bool fused = false;                    // the attention launch fuses (some of) the appends
  std::vector<uint8_t> in_kernel(n_items > 0 ? n_items : 1, 0);   // item's append inside it
  std::vector<s2l_prefill_item> separate;                         // items appended by a launch
  if (append) {
    if (!v) return fail(S2L_E_INVAL, "k/v is NULL");
    std::unordered_set<int64_t> seen;
    const bool kern = c->tc_ok && !c->geo.fp8;   // no in-kernel append into an FP8 pool
    int32_t aligned = 0;
    for (int32_t i = 0; i < n_items; ++i) {
      if (!seen.insert(items[i].req_id).second)
        return fail(S2L_E_INVAL, "item %d: request %lld repeated", i, (long long)items[i].req_id);
      aligned += items[i].q_pos % c->cfg.block_size == 0;
    }
    // per item when the items travel inline (the kernel gets a mask), else all or nothing
    const bool per_item = n_items <= s2l::kInlineAttnItems;
    fused = kern && aligned > 0 && (aligned == n_items || per_item);
    for (int32_t i = 0; i < n_items; ++i) {
      in_kernel[i] = fused && items[i].q_pos % c->cfg.block_size == 0;
      if (!in_kernel[i]) separate.push_back(items[i]);
    }
  }
  if (c->sticky) return fail(c->sticky, "context has a sticky CUDA error");
  if (n_items == 0) return S2L_OK;
  s2l_status st = flush_patches(c);
  if (st) return st;
  for (int32_t i = 0; i < n_items; ++i) {
    Request* r = find(c, items[i].req_id);
    if (r->swap_in_seq) {
      if (!ring_wait(c, c->in_ring, c->compute, r->swap_in_seq)) return S2L_E_CUDA;
    }
  }
  if (!separate.empty()) {
    st = layer_append(c, layer, (int32_t)separate.size(), separate.data(), k, v, q_rows);
    if (st) return st;
  }
  const int32_t G = c->cfg.num_q_heads / c->cfg.num_kv_heads;
  // Items ordered by descending KV length (q_pos + n_q) so that the longest Q tiles start
  // first (longest-processing-time order for the hardware block scheduler).
  std::vector<int32_t> order(n_items);
  for (int32_t i = 0; i < n_items; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
    return items[x].q_pos + items[x].n_q > items[y].q_pos + items[y].n_q;
  });
  std::vector<s2l::AttnItemDev> dev(n_items);
  uint64_t fuse_mask = ~0ull;            // bit i: item i (kernel order) appended in-kernel
  if (fused && n_items <= s2l::kInlineAttnItems) {
    fuse_mask = 0;
    for (int32_t i = 0; i < n_items; ++i)
      if (in_kernel[order[i]]) fuse_mask |= 1ull << i;
  }
  const int64_t tiles_per_cta = c->tc_ok ? 2 : 1;   // tensor-core kernel: a pair of Q tiles per CTA
  int64_t units = 0, total_q = 0;
  for (int32_t i = 0; i < n_items; ++i) {
    const s2l_prefill_item& it = items[order[i]];
    Request* r = find(c, it.req_id);
    s2l::AttnItemDev& d = dev[i];
    d.q_pos = it.q_pos;
    d.q_row = it.q_row;
    d.n_q = (int32_t)it.n_q;
    d.slot = r->slot;
    d.tiles = (int32_t)ceil_div(it.n_q * G, 128);
    d.unit_begin = (int32_t)units;
    units += ceil_div(d.tiles, tiles_per_cta) * c->cfg.num_kv_heads;
    total_q += it.n_q;
  }
  if (units >= (1ll << 31)) return fail(S2L_E_INVAL, "batch too large");
  size_t bytes = dev.size() * sizeof(s2l::AttnItemDev);
  // tensor-core kernel: up to kInlineAttnItems items travel in the kernel parameters
  const bool inl = c->tc_ok && n_items <= s2l::kInlineAttnItems;
  int s = -1;
  const s2l::AttnItemDev* dv = nullptr;
  if (!inl) {
    s = staging_acquire(c, bytes);
    if (s < 0) return S2L_E_CUDA;
    memcpy(c->ring.host[s], dev.data(), bytes);
    if (!staging_upload_and_mark(c, s, bytes)) return S2L_E_CUDA;
    dv = (const s2l::AttnItemDev*)c->ring.dev[s];
  }
  std::pair<cudaEvent_t, cudaEvent_t> tp{};
  if (c->timing) {
    tp = timing_pair(c);
    CK(cudaEventRecord(tp.first, c->compute));
  }
  if (c->tc_ok) {
    alignas(64) unsigned char tq[128];
    const char* err = nullptr;
    if (!s2l::make_tmap_q(tq, q, q_rows, c->cfg.num_q_heads, c->cfg.head_dim, G, &err))
      return fail(S2L_E_CUDA, "tensor map (q): %s", err ? err : "?");
    alignas(64) unsigned char to[128];                // O has Q's shape: the same box
    if (!s2l::make_tmap_q(to, o, q_rows, c->cfg.num_q_heads, c->cfg.head_dim, G, &err))
      return fail(S2L_E_CUDA, "tensor map (o): %s", err ? err : "?");
    // Tail-wave split (hybrid stream-K): whole units fill the full waves; the units of the
    // last partial wave are cut into s contiguous KV ranges so that wave is ~full as well.
    const int64_t P = c->num_sms;
    const int64_t rem = units % P;
    int32_t split_begin = (int32_t)units, split_s = 1;
    if (c->split_enabled && rem > 0 && rem * 2 <= P) {
      int64_t s_want = std::min<int64_t>(P / rem, 8);
      // no piece may be empty: s <= the smallest KV-tile count among the split units
      const int64_t first = units - rem;
      for (int32_t i = n_items - 1; i >= 0 && s_want > 1; --i) {
        const s2l::AttnItemDev& d = dev[i];
        const int64_t pairs = ceil_div(d.tiles, 2);
        const int64_t u0 = d.unit_begin, u1 = u0 + pairs * c->cfg.num_kv_heads;
        if (u1 <= first) break;
        for (int64_t pr = 0; pr < pairs; ++pr) {       // pair index; its units are >= first?
          const int64_t local0 = (pairs - 1 - pr) * c->cfg.num_kv_heads;
          // head-major order: a pair's units are spread over the item; count every pair
          if (!S2L_HEAD_MAJOR && u0 + local0 + c->cfg.num_kv_heads <= first) continue;
          const int64_t toks = 128 / G;
          const int64_t tok_last = std::min<int64_t>((pr * 2 + 2) * toks, d.n_q) - 1;
          const int64_t nT = (d.q_pos + tok_last) / 128 + 1;
          s_want = std::min(s_want, nT);
        }
      }
      if (s_want > 1) {
        split_begin = (int32_t)(units - rem);
        split_s = (int32_t)s_want;
      }
    }
    alignas(64) unsigned char tin[512];
    if (fused && !s2l::make_tmap_in(tin, k, v, q_rows, c->cfg.num_kv_heads, c->cfg.head_dim,
                                    (int32_t)c->cfg.block_size, &err))
      return fail(S2L_E_CUDA, "tensor map (k/v input): %s", err ? err : "?");
    s2l::set_attn_trace(c->attn_launch_no++ == c->trace_launch ? c->trace_buf : nullptr);
    CK(s2l::launch_attn_tc(c->geo, dv, inl ? dev.data() : nullptr, n_items, (int32_t)units,
                           split_begin, split_s,
                           c->split_ws, c->num_sms, c->split_cnt, c->d_table, layer, tq,
                           c->tmap_kv, to, o, lse,
                           (fused ? s2l::kAttnFuseAppend : 0) | (c->split_direct ? 0 : s2l::kAttnNoDirectMerge),
                           c->compute, fused ? tin : nullptr, c->gpu_pool, fuse_mask));
  } else {
    CK(s2l::launch_attn_generic(c->geo, dv, n_items, total_q, c->d_table, layer, q, o, lse,
                                c->gpu_pool, c->compute));
  }
  c->launches++;
  if (c->timing) {
    CK(cudaEventRecord(tp.second, c->compute));
    c->attn_ev.push_back(tp);
  }
  uint64_t useq = 0;
  if (!ring_record(c, c->compute_ring, c->compute, &useq)) return S2L_E_CUDA;
  for (int32_t i = 0; i < n_items; ++i) {
    Request* r = find(c, items[i].req_id);
    r->use_seq = useq;
    if (append) r->write_seq = useq;
  }
  if (!inl && !staging_release(c, s)) return S2L_E_CUDA;
  return S2L_OK;
}

s2l_status s2l_prefill_batch(s2l_ctx* c, int32_t layer, int32_t n_items,
                             const s2l_prefill_item* items, const void* q, void* o, float* lse,
                             int64_t q_rows) {
  return prefill_impl(c, layer, n_items, items, q, nullptr, nullptr, o, lse, q_rows);
}

s2l_status s2l_prefill_append(s2l_ctx* c, int32_t layer, int32_t n_items,
                              const s2l_prefill_item* items, const void* q, const void* k,
                              const void* v, void* o, float* lse, int64_t q_rows) {
  if (c && (!k || !v) && n_items > 0) return fail(S2L_E_INVAL, "k/v is NULL");
  return prefill_impl(c, layer, n_items, items, q, k ? k : v, v, o, lse, q_rows);
}

s2l_status s2l_swap_out(s2l_ctx* c, int32_t n, const int64_t* ids, int64_t* bytes_out) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  return swap_impl(c, n, ids, bytes_out, S2L_TIER_GPU, S2L_TIER_CPU);
}

s2l_status s2l_swap_in(s2l_ctx* c, int32_t n, const int64_t* ids, int64_t* bytes_out) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  return swap_impl(c, n, ids, bytes_out, S2L_TIER_CPU, S2L_TIER_GPU);
}

s2l_status s2l_query(s2l_ctx* c, int64_t id, s2l_req_info* out) {
  if (!c || !out) return fail(S2L_E_INVAL, "NULL argument");
  Request* r = find(c, id);
  if (!r) return fail(S2L_E_NO_REQUEST, "unknown request %lld", (long long)id);
  out->num_tokens = (int64_t)r->input.size();
  out->num_computed = r->nc;
  out->total_tokens_invalidated = r->tti;
  out->tier = r->tier;
  out->num_blocks = (int32_t)r->blocks.size();
  return S2L_OK;
}

s2l_status s2l_block_table(s2l_ctx* c, int64_t id, int32_t* ids_out, int64_t cap, int64_t* n_out) {
  if (!c || cap < 0 || (cap > 0 && !ids_out)) return fail(S2L_E_INVAL, "bad arguments");
  Request* r = find(c, id);
  if (!r) return fail(S2L_E_NO_REQUEST, "unknown request %lld", (long long)id);
  int64_t n = (int64_t)r->blocks.size();
  if (n_out) *n_out = n;
  if (n > 0 && cap > 0) memcpy(ids_out, r->blocks.data(), (size_t)std::min(n, cap) * sizeof(int32_t));
  return S2L_OK;
}

s2l_status s2l_free_blocks(s2l_ctx* c, int64_t* gpu_free, int64_t* cpu_free) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  if (gpu_free) *gpu_free = c->alloc[S2L_TIER_GPU].free_count();
  if (cpu_free) *cpu_free = c->alloc[S2L_TIER_CPU].free_count();
  return S2L_OK;
}

s2l_status s2l_set_swap_in_stream(s2l_ctx* c, void* stream) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  if (c->host_only) return fail(S2L_E_STATE, "host-only context has no device");
  if (!stream) return fail(S2L_E_INVAL, "stream is NULL");
  CK(cudaStreamSynchronize(c->copy_in));
  if (c->own_copy_in) cudaStreamDestroy(c->copy_in);
  c->copy_in = (cudaStream_t)stream;
  c->own_copy_in = false;
  return S2L_OK;
}

s2l_status s2l_sync(s2l_ctx* c) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  if (c->host_only) return S2L_OK;
  CK(cudaStreamSynchronize(c->compute));
  CK(cudaStreamSynchronize(c->copy));
  CK(cudaStreamSynchronize(c->copy_in));
  return c->sticky;
}

int64_t s2l_kernel_launches(s2l_ctx* c) { return c ? c->launches : -1; }

s2l_status s2l_wait_counts(s2l_ctx* c, int64_t* waits) {
  if (!c || !waits) return fail(S2L_E_INVAL, "ctx or waits is NULL");
  for (int i = 0; i < 4; ++i) waits[i] = c->waits[i];
  return S2L_OK;
}

s2l_status s2l_set_timing(s2l_ctx* c, int32_t enable) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  if (c->host_only) return fail(S2L_E_STATE, "host-only context has no device");
  CK(cudaStreamSynchronize(c->compute));
  for (auto* v : {&c->attn_ev, &c->append_ev}) {
    for (auto& p : *v) c->ev_pool.push_back(p);
    v->clear();
  }
  c->timing = enable != 0;
  return S2L_OK;
}

s2l_status s2l_timing_read(s2l_ctx* c, double* attn_ms, int64_t* attn_n, double* app_ms,
                           int64_t* app_n) {
  if (!c) return fail(S2L_E_INVAL, "ctx is NULL");
  if (c->host_only) return fail(S2L_E_STATE, "host-only context has no device");
  CK(cudaStreamSynchronize(c->compute));
  double t[2] = {0, 0};
  int i = 0;
  for (auto* v : {&c->attn_ev, &c->append_ev}) {
    for (auto& p : *v) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, p.first, p.second));
      t[i] += ms;
    }
    ++i;
  }
  if (attn_ms) *attn_ms = t[0];
  if (attn_n) *attn_n = (int64_t)c->attn_ev.size();
  if (app_ms) *app_ms = t[1];
  if (app_n) *app_n = (int64_t)c->append_ev.size();
  return S2L_OK;
}

const char* s2l_last_error(void) { return g_err.c_str(); }

const char* s2l_version(void) { return "libs2l 0.1 sm_100a (tcgen05/TMEM/TMA attention)"; }

}  // extern "C"
