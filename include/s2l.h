/*
 * s2l.h — C ABI of libs2l, the B200 (sm_100a) streaming-prefill KV / attention library
 * for STREAM2LLM (arXiv 2604.16395).  Citations: P:Lnnn = /root/reference/PAPER.md line,
 * S:Lnnn = SPEC.md line, Zn = a reading recorded in DESIGN.md §Readings.
 *
 * What the library holds ("GPU and CPU block pools"):
 *   - a GPU block pool (caller-owned device memory) and a CPU block pool (caller-owned
 *     PINNED host memory), both laid out as
 *         pool[block][layer][2 (0=K,1=V)][kv_head][slot (0..k-1)][head_dim]   bf16
 *     so one block is contiguous across layers and occupies
 *         M_block = 2 * L * k * h_kv * d * b bytes   (= P:L73 with d_model*h_kv/h = h_kv*d;
 *                                                     b = 2 for bf16, 1 for kv_dtype FP8);
 *   - a request table: per request its input tokens, num_computed_tokens (nc), tier
 *     (GPU or CPU), ordered block ids on that tier, total_tokens_invalidated;
 *   - a device block table [max_requests][max_blocks_per_request] int32 (library-owned)
 *     read by the kernels; block j of a request holds positions [j*k, j*k+k).
 *
 * Allocation (Z9; the paper only says "free block pool"): every allocation takes the
 * LOWEST free ids of the tier, ascending, independent of the order in which ids were freed
 * (SURVEY.md §8.2 c.4 Z9); requests/items of one call are served in call order.  Opt-in
 * (s2l_config.alloc_cooling = 1, a performance choice, not the paper's): the GPU ids released
 * by the most recent swap-out ("cooling": their D2H copy may still be reading them) come after
 * every other free GPU id, so appends and swap-ins rarely wait for a D2H.  Every call that can fail is
 * all-or-nothing: arguments and capacity are validated before any state changes.
 *
 * Streams: `compute_stream` runs append/patch/attention kernels; `copy_stream` runs swap-out
 * copies and a second stream (library-created, or s2l_set_swap_in_stream) runs swap-in copies
 * (cudaStream_t handles passed as void*; NULL = legacy default stream).  The library inserts
 * only the event waits real conflicts need (per request and per block, DESIGN.md §5 stream
 * hazards), so swaps overlap unrelated compute.  Per-call descriptors of small calls travel in
 * the kernel parameters, larger ones through a pinned staging ring.  Pointer arguments to
 * device/pinned buffers must stay valid until the work enqueued by the call has completed on
 * its stream (stream-ordered semantics).  Host token arrays and item arrays are copied before
 * the call returns.
 *
 * Errors: every function returns an s2l_status.  State/argument errors are detected before
 * any mutation.  A CUDA error is reported as S2L_E_CUDA and is sticky for the context.
 * s2l_last_error() returns a thread-local message for the most recent failure.
 * No C++ exception crosses the ABI.  One host thread per context at a time.
 */
#ifndef S2L_H_
#define S2L_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct s2l_ctx s2l_ctx;
typedef int32_t s2l_status;

enum {
  S2L_OK = 0,
  S2L_E_INVAL = -1,          /* bad argument / geometry / duplicate request in one call    */
  S2L_E_NO_GPU_BLOCKS = -2,  /* GPU pool cannot satisfy the whole call    */
  S2L_E_NO_CPU_BLOCKS = -3,  /* CPU pool cannot satisfy the whole swap-out        */
  S2L_E_NO_REQUEST = -4,     /* unknown request id                                          */
  S2L_E_STATE = -5,          /* wrong tier for the call / request already exists            */
  S2L_E_CUDA = -6,           /* CUDA runtime / driver failure (sticky)                      */
  S2L_E_CAPACITY = -7        /* request table full (max_requests)                           */
};

enum { S2L_TIER_GPU = 0, S2L_TIER_CPU = 1 };

/* Bookkeeping is identical in every context; the attention kernel variant is chosen per
 * call: the tcgen05/TMEM/TMA tensor-core kernel when head_dim == 128 and 16 <= block_size
 * <= 128, otherwise a CUDA-core kernel (e.g. C1: head_dim 16, block 4).  Both are sm_100a
 * code in this library; there is no CPU path. */
typedef struct s2l_config {
  int32_t num_layers;             /* L: layers held by the pools                            */
  int32_t num_q_heads;            /* h                                            */
  int32_t num_kv_heads;           /* h_kv; must divide num_q_heads (GQA, Z2)         */
  int32_t head_dim;               /* d_h = d/h; multiple of 8, <= 256                       */
  int32_t block_size;             /* k tokens per block; power of two, 1..256       */
  int32_t num_gpu_blocks;         /* blocks in the GPU pool                                 */
  int32_t num_cpu_blocks;         /* blocks in the CPU pool (may be 0: no swapping)         */
  int32_t max_requests;           /* live requests at once                                  */
  int32_t max_blocks_per_request; /* columns of the device block table; max_requests * this
                                     and this * block_size must be < 2^31 (E_INVAL)         */
  int32_t lcp_block_aligned;      /* 0 = token-granular LCP (default, Z4);
                                     1 = round the kept prefix down to a block     */
  int32_t alloc_cooling;          /* 0 = plain lowest-free-id order (Z9, default);
                                     1 = GPU ids freed by the latest swap-out go last       */
  int32_t kv_dtype;               /* 0 = bf16 K/V (b = 2 bytes per value; default);
                                     1 = FP8 E4M3 K/V cache (b = 1, not the
                                     paper's): s2l_append_chunk stores each bf16 value as the
                                     nearest E4M3 code (RNE, saturating to +-448, reading
                                     Z20), attention dequantizes it exactly to bf16 before
                                     its MMAs; s2l_prefill_append then appends with a
                                     separate launch (no in-kernel append)                  */
} s2l_config;

/* One request of an s2l_append_chunk call. */
typedef struct s2l_append_item {
  int64_t req_id;
  const int32_t* tokens;  /* host; n_tokens ids appended to the input first (Append event,
                             LCP = old length); NULL when n_tokens == 0             */
  int64_t n_tokens;
  int64_t n_kv;           /* K/V rows written for positions [nc, nc+n_kv); 0..pending     */
  int64_t kv_row;         /* first row of this item in the k/v token dimension            */
} s2l_append_item;

/* One request of an s2l_prefill_batch call. */
typedef struct s2l_prefill_item {
  int64_t req_id;
  int64_t q_pos;          /* absolute position of the first query row (normally nc - n_q) */
  int64_t n_q;            /* >= 1 query rows; q_pos + n_q <= nc                            */
  int64_t q_row;          /* first row of this item in q / o / lse                         */
} s2l_prefill_item;

typedef struct s2l_req_info {
  int64_t num_tokens;               /* len(input)                                         */
  int64_t num_computed;             /* nc = num_computed_tokens                  */
  int64_t total_tokens_invalidated;
  int32_t tier;                     /* S2L_TIER_GPU / S2L_TIER_CPU                        */
  int32_t num_blocks;               /* blocks held on that tier = ceil(nc / k)            */
} s2l_req_info;

/* M_block = 2*L*k*h_kv*d*2 bytes.  Returns -1 for an invalid config. */
int64_t s2l_block_bytes(const s2l_config* cfg);

/* Create a context bound to the current CUDA device.
 *   gpu_pool        device pointer, num_gpu_blocks*M_block bytes, 256-B aligned
 *   cpu_pool_pinned page-locked host pointer, num_cpu_blocks*M_block bytes (NULL iff
 *                   num_cpu_blocks == 0)
 *   compute_stream, copy_stream: cudaStream_t as void*.
 * Both pools are zero-filled (device: cudaMemsetAsync on compute_stream; host: memset) so
 * never-written slots are finite.  The library allocates its own device block table and a
 * small pinned + device staging ring.  Ownership of the pools stays with the caller and
 * they must outlive the context.  The library orders its own kernels and copies (stream
 * hazards); swaps run on their own streams, so a caller that reads or writes
 * pool memory directly must call s2l_sync first.  Errors: S2L_E_INVAL (geometry), S2L_E_CUDA. */
s2l_status s2l_create(const s2l_config* cfg, void* gpu_pool, void* cpu_pool_pinned,
                      void* compute_stream, void* copy_stream, s2l_ctx** out);

/* Bookkeeping-only context for host-logic tests (no device, no pools).  Every call runs its
 * validation and state machine exactly as in a device context; calls that would move data
 * require their data pointers to be NULL (append: k = v = NULL) and s2l_prefill_batch returns
 * S2L_E_STATE.  It never computes attention or moves bytes. */
s2l_status s2l_create_host_only(const s2l_config* cfg, s2l_ctx** out);

/* Synchronises both streams, frees library-owned memory.  NULL is a no-op. */
void s2l_destroy(s2l_ctx* ctx);

/* NewStream: input := tokens (copied), nc := 0, GPU tier, no blocks.
 * S2L_E_STATE if req_id is live, S2L_E_CAPACITY if max_requests are live. */
s2l_status s2l_new_request(s2l_ctx* ctx, int64_t req_id, const int32_t* tokens, int64_t n);

/* Request finished: frees its blocks on its tier and forgets the id. */
s2l_status s2l_release_request(s2l_ctx* ctx, int64_t req_id);

/* Recomputation preemption: frees all its blocks on its tier, nc := 0,
 * tier := GPU; the input is kept.  total_tokens_invalidated is unchanged. */
s2l_status s2l_preempt_recompute(s2l_ctx* ctx, int64_t req_id);

/* Append (a3): for each item, append its tokens to the input, allocate
 * ceil((nc+n_kv)/k) - held blocks (lowest free ids, P:L69 on-demand from the free pool),
 * write K/V of positions [nc, nc+n_kv) into slot (table[pos/k], pos%k) of every layer,
 * nc += n_kv.
 *   k, v: device, [num_layers][kv_rows][h_kv][d] bf16, item i's rows at
 *         [kv_row_i, kv_row_i + n_kv_i); kv_rows = token rows per layer.
 * Validation (first failing item in call order wins; capacity checked last):
 *   unknown id -> E_NO_REQUEST; id repeated in the call -> E_INVAL; CPU tier with
 *   n_kv != 0 -> E_STATE (a token-only item, n_kv = 0, is valid on either tier: input keeps
 *   arriving while a request is swapped out, reading Z19);
 *   n_tokens/n_kv/kv_row < 0, kv_row+n_kv > kv_rows, n_kv > len(input)+n_tokens-nc, or
 *   ceil((nc+n_kv)/k) > max_blocks_per_request -> E_INVAL;
 *   total new blocks > free GPU blocks -> E_NO_GPU_BLOCKS.
 * Reserve (NEXT-2): k = v = NULL on a device context does all of the above except the data
 * write; the K/V of each layer are then written by s2l_prefill_append (until then the rows are
 * undefined).  Exactly one of k / v NULL -> E_INVAL.
 * On any error nothing changes (all-or-nothing). */
s2l_status s2l_append_chunk(s2l_ctx* ctx, int32_t n_items, const s2l_append_item* items,
                            const void* k, const void* v, int64_t kv_rows);

/* Update event (a1 + a2).  p = LCP(input, new_tokens); b = min(p, nc)
 * (Z5; lcp_block_aligned: b = floor(b/k)*k); keep ceil(b/k) blocks (Z4) and
 * return the rest to the pool of the tier holding them (GPU, or CPU when swapped);
 * nc := b; input := new_tokens; invalidated = nc_old - b is added to
 * total_tokens_invalidated.  A swapped request left with no blocks becomes a
 * GPU-tier request.  Host-only: the freed entries of the block table are reset on the
 * host mirror; the device copy of an entry is only read below a request's valid block count, so
 * it is updated when the entry receives a block id again (patch on the next kernel launch).
 * lcp_out / tokens_invalidated_out may be NULL. */
s2l_status s2l_invalidate_lcp(s2l_ctx* ctx, int64_t req_id, const int32_t* new_tokens,
                              int64_t new_len, int64_t* lcp_out, int64_t* tokens_invalidated_out);

/* Chunked-prefill attention (a4): for item i, query row t (0 <= t < n_q) at
 * absolute position q_pos+t and q head h,
 *   o[q_row+t][h] = softmax_j( q·K_j / sqrt(d) ) · V   over keys j = 0 .. q_pos+t of kv head
 *   g(h) = floor(h / (h/h_kv)) (Z2), K/V read from layer `layer` of the GPU pool through the
 *   request's block table.  lse (optional) = natural-log log-sum-exp of the scaled scores.
 *   q, o: device [q_rows][h][d] bf16; lse: device [q_rows][h] fp32 or NULL.
 * Requirements: GPU tier, n_q >= 1, q_pos >= 0, q_pos + n_q <= nc, q_row + n_q <= q_rows,
 * 0 <= layer < L (else E_INVAL / E_STATE / E_NO_REQUEST).  Read-only on the request state;
 * waits for any swap-in of the listed requests.  fp32 accumulation, bf16 P, bf16 output. */
s2l_status s2l_prefill_batch(s2l_ctx* ctx, int32_t layer, int32_t n_items,
                             const s2l_prefill_item* items, const void* q, void* o, float* lse,
                             int64_t q_rows);

/* Fused append + attention for one layer (a3 + a4, P:L59 / P:L67 / P:L69): for
 * each item, first the K/V rows of positions [q_pos, q_pos+n_q) of layer `layer` are taken from
 * k / v rows [q_row, q_row+n_q) and stored in the pool (as s2l_append_chunk stores them), then
 * the attention of s2l_prefill_batch is computed over the prefix plus those rows.  The blocks
 * must already be held (s2l_append_chunk, normally in reserve mode with k = v = NULL).
 *   k, v: device [q_rows][h_kv][d] bf16 of this layer (same row indexing as q).
 For items whose q_pos is a multiple of k (tensor-core kernel) one kernel does both: it reads
 * the chunk's K/V tiles from k / v and each work unit writes the blocks starting in its own token
 * range to the pool; the other items (or all, when more than 64 items are passed and one is
 * unaligned) are appended by a one-layer append launch before the attention.
 * Errors: those of s2l_prefill_batch; k or v NULL, or a request repeated in the call -> E_INVAL. */
s2l_status s2l_prefill_append(s2l_ctx* ctx, int32_t layer, int32_t n_items,
                              const s2l_prefill_item* items, const void* q, const void* k,
                              const void* v, void* o, float* lse, int64_t q_rows);

/* Swap-out (a5): all-or-nothing over the listed requests (all GPU tier, no
 * duplicates): allocate |blocks| CPU ids per request (lowest free), copy every block GPU ->
 * CPU in order on copy_stream (whole blocks, Z12), free the GPU ids, tier := CPU, nc kept.
 * The copies wait only for the work they conflict with (the requests' appends / swap-ins, an
 * H2D still reading the destination CPU blocks); later appends that reuse the freed GPU ids
 * wait for them (DESIGN.md §5 stream hazards).
 * bytes_out = total blocks * M_block.  E_NO_CPU_BLOCKS if the CPU pool is short. */
s2l_status s2l_swap_out(s2l_ctx* ctx, int32_t n_reqs, const int64_t* req_ids, int64_t* bytes_out);

/* Swap-in (a6, "symmetric", P:L184 prefix only after an update): mirror of
 * s2l_swap_out CPU -> GPU, on the swap-in stream (s2l_set_swap_in_stream).  The H2D waits for
 * the requests' swap-outs and for any kernel / D2H still using the destination GPU blocks;
 * appends / attention of the requests wait for it.  E_NO_GPU_BLOCKS if the GPU pool is short. */
s2l_status s2l_swap_in(s2l_ctx* ctx, int32_t n_reqs, const int64_t* req_ids, int64_t* bytes_out);

s2l_status s2l_query(s2l_ctx* ctx, int64_t req_id, s2l_req_info* out);

/* Copies the request's block ids (on its current tier) into ids_out[0..cap); *n_out = count
 * (may exceed cap; then only cap ids are written). */
s2l_status s2l_block_table(s2l_ctx* ctx, int64_t req_id, int32_t* ids_out, int64_t cap,
                           int64_t* n_out);

/* Free block counts of both tiers. */
s2l_status s2l_free_blocks(s2l_ctx* ctx, int64_t* gpu_free, int64_t* cpu_free);

/* Swap-ins (H2D) run on a second copy stream so that they overlap swap-outs (D2H, on
 * copy_stream) as well as compute; by default the library creates it.  This call replaces it
 * with a caller-owned cudaStream_t (e.g. to record timing events on it); the previous stream
 * is drained first.  Errors: S2L_E_INVAL (NULL), S2L_E_STATE (host-only context). */
s2l_status s2l_set_swap_in_stream(s2l_ctx* ctx, void* stream);

/* Blocks until all work enqueued by this context on its streams (compute, swap-out,
 * swap-in) has completed. */
s2l_status s2l_sync(s2l_ctx* ctx);

/* Number of kernels this context has launched since creation (evidence counter). */
int64_t s2l_kernel_launches(s2l_ctx* ctx);

/* Evidence counters since creation: cross-stream waits the runtime inserted because the work
 * they order after was still pending when the call was issued (orderings against finished work
 * cost nothing and are not counted).  waits[0]: the compute stream after a swap-out D2H (an
 * append reusing a block the D2H still reads); waits[1]: compute after a swap-in H2D (the
 * request's K/V, or a reused block, still arriving); waits[2]: a copy stream after compute
 * (blocks kernels may still use); waits[3]: a copy stream after the other copy stream.
 * waits: caller-owned array of 4.  Errors: S2L_E_INVAL (NULL ctx or array). */
s2l_status s2l_wait_counts(s2l_ctx* ctx, int64_t* waits);

/* Per-kernel device timing (for the roofline in bench.py).  s2l_set_timing(ctx, 1) clears
 * and starts a window: every attention / append kernel launch is then bracketed by CUDA
 * events on compute_stream.  s2l_timing_read synchronises compute_stream and returns the
 * summed event durations (ms) and launch counts of the window.  Timing off by default. */
s2l_status s2l_set_timing(s2l_ctx* ctx, int32_t enable);
s2l_status s2l_timing_read(s2l_ctx* ctx, double* attn_ms, int64_t* attn_launches,
                           double* append_ms, int64_t* append_launches);

/* Thread-local description of the most recent error ("" if none). */
const char* s2l_last_error(void);

/* Library build string (arch, version). */
const char* s2l_version(void);

#ifdef __cplusplus
}
#endif

#endif /* S2L_H_ */
