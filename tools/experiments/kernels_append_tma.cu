// Paged KV append (a3) by TMA bulk-tensor copies: global -> shared -> global, no registers.
//
// a3, P:L59 / P:L67: the K/V rows of positions [nc, nc+n_kv) of each request are stored in
// block table[pos / k] at slot pos % k of every layer.  Pool layout (include/s2l.h):
//   pool[block][layer][2][kv_head][slot][d]  bf16,
// caller rows: k, v = [L'][kv_rows][h_kv][d] (L' = the layers of this call).
//
// Work unit = (touched block, layer, K|V).  A block filled by the append from slot 0 to k-1 is
// ONE TMA load of the caller's k consecutive rows (box {d, h_kv, k, 1} over [L'][rows][h_kv][d],
// smem order [slot][head][d]) and ONE TMA store through a pool map whose dimensions are ordered
// (d, head, slot, layer*2+kind, block) -- strides 2, k*d*2, d*2, ... -- so the same smem order
// lands as [head][slot][d] in the pool.  A partially filled block (the append starts or ends
// inside it) moves row by row (box {d, h_kv, 1, ...}): only the appended slots are written, as
// with the register kernel (the stale tail of a block is never touched).
// One thread per CTA issues everything; a ring of NBUF shared-memory slots keeps NBUF-1 units
// loading while the oldest one is stored.  Persistent grid: one CTA per SM.
#include "tc_common.cuh"

#include <cstring>
#include <mutex>

namespace s2l {
namespace {

constexpr int kTmaThreads = 32;
constexpr int NBUF = 6;
constexpr uint32_t kSlotBytes = 32768;            // h_kv * k * d * 2 <= 32 KB (Llama-3: 8*16*128*2)
constexpr uint32_t OFF_BARS = NBUF * kSlotBytes;
constexpr uint32_t APPEND_SMEM = OFF_BARS + NBUF * 8 + 1024;

struct AppendTmaMaps {
  CUtensorMap in_blk[2];    // K, V input: box {d, h_kv, k, 1}
  CUtensorMap in_row[2];    // K, V input: box {d, h_kv, 1, 1}
  CUtensorMap pool_blk;     // pool (d, head, slot, layer*2+kind, block): box {d, h_kv, k, 1, 1}
  CUtensorMap pool_row;     // same dims: box {d, h_kv, 1, 1, 1}
};

__device__ __forceinline__ void tma_load_4d_tx(uint32_t dst, const void* tmap, uint32_t bar, int32_t x, int32_t y,
                                               int32_t z, int32_t w) {
  tma_load_4d(dst, tmap, bar, x, y, z, w);
}
__device__ __forceinline__ void tma_store_5d(const void* tmap, uint32_t src, int32_t x, int32_t y, int32_t z,
                                             int32_t w, int32_t v) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(tmap),
      "r"(x), "r"(y), "r"(z), "r"(w), "r"(v), "r"(src)
      : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read_n() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(kTmaThreads, 1) append_tma_kernel(
    const __grid_constant__ AppendTmaMaps m, const AppendItemDev* __restrict__ items_p, int32_t n_items,
    const int32_t* __restrict__ ids_p, int32_t n_ids, const TablePatch* __restrict__ patches_p, int32_t n_patches,
    int32_t* __restrict__ table, const __grid_constant__ InlineBlob blob, int32_t blob_mode, int32_t off_ids,
    int32_t off_patch, int32_t layer0, int32_t nl, int32_t kb, uint32_t row_bytes, uint32_t row_stride) {
  pdl_prologue();
  const AppendItemDev* items = blob_mode ? reinterpret_cast<const AppendItemDev*>(blob.b) : items_p;
  const int32_t* ids = blob_mode ? reinterpret_cast<const int32_t*>(blob.b + off_ids) : ids_p;
  const TablePatch* patches = blob_mode ? reinterpret_cast<const TablePatch*>(blob.b + off_patch) : patches_p;
  if (blockIdx.x == 0)
    for (int32_t i = threadIdx.x; i < n_patches; i += blockDim.x) table[patches[i].idx] = patches[i].value;
  if (threadIdx.x != 0) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int i) { return sb + OFF_BARS + 8u * (uint32_t)i; };
  for (int i = 0; i < NBUF; ++i) mbar_init(bar(i), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

  const int32_t lk_n = nl * 2;
  const int32_t units = n_ids * lk_n;
  // unit -> (block index bu in the id list, layer-kind lk); bu -> item (last id_off <= bu)
  struct U {
    int32_t blk, slot0, cnt, lk;
    int64_t src;
  };
  auto decode = [&](int32_t u) {
    const int32_t bu = u / lk_n, lk = u - bu * lk_n;
    int32_t lo = 0, hi = n_items - 1;
    while (lo < hi) {
      const int32_t mid = (lo + hi + 1) >> 1;
      if (items[mid].id_off <= bu) lo = mid; else hi = mid - 1;
    }
    const AppendItemDev it = items[lo];
    const int64_t start = (it.nc / kb + (bu - it.id_off)) * (int64_t)kb;   // first position of the block
    const int64_t p0 = it.nc > start ? it.nc : start;
    const int64_t e = it.nc + it.n_kv, p1 = e < start + kb ? e : start + kb;
    U r;
    r.blk = ids[bu];
    r.slot0 = (int32_t)(p0 - start);
    r.cnt = (int32_t)(p1 - p0);
    r.lk = lk;
    r.src = it.kv_row + (p0 - it.nc);
    return r;
  };
  auto issue_load = [&](const U& w, int slot) {
    const uint32_t dst = sb + (uint32_t)slot * kSlotBytes;
    const int kind = w.lk & 1, li = w.lk >> 1;
    mbar_expect_tx(bar(slot), (uint32_t)w.cnt * row_bytes);
    if (w.cnt == kb) {
      tma_load_4d_tx(dst, &m.in_blk[kind], bar(slot), 0, 0, (int32_t)w.src, li);
    } else {
      for (int32_t r = 0; r < w.cnt; ++r)
        tma_load_4d_tx(dst + (uint32_t)r * row_stride, &m.in_row[kind], bar(slot), 0, 0, (int32_t)(w.src + r), li);
    }
  };
  auto issue_store = [&](const U& w, int slot) {
    const uint32_t src = sb + (uint32_t)slot * kSlotBytes;
    const int32_t plane = (layer0 + (w.lk >> 1)) * 2 + (w.lk & 1);
    if (w.cnt == kb) {
      tma_store_5d(&m.pool_blk, src, 0, 0, 0, plane, w.blk);
    } else {
      for (int32_t r = 0; r < w.cnt; ++r)
        tma_store_5d(&m.pool_row, src + (uint32_t)r * row_stride, 0, 0, w.slot0 + r, plane, w.blk);
    }
    bulk_commit();
  };
  // this CTA's units: u = blockIdx.x + t * gridDim.x
  const int32_t T = units > (int32_t)blockIdx.x ? (units - 1 - (int32_t)blockIdx.x) / (int32_t)gridDim.x + 1 : 0;
  U w[NBUF];
  for (int32_t t = 0; t < T && t < NBUF - 1; ++t) {
    w[t] = decode((int32_t)blockIdx.x + t * (int32_t)gridDim.x);
    issue_load(w[t], t);
  }
  for (int32_t t = 0; t < T; ++t) {
    const int slot = t % NBUF;
    mbar_wait(bar(slot), (uint32_t)(t / NBUF) & 1);
    issue_store(w[slot], slot);
    const int32_t tn = t + NBUF - 1;
    if (tn < T) {
      const int sn = tn % NBUF;                         // = (t - 1) % NBUF: the previous store's slot
      bulk_wait_read_n<1>();                            // every store but this one has read its slot
      w[sn] = decode((int32_t)blockIdx.x + tn * (int32_t)gridDim.x);
      issue_load(w[sn], sn);
    }
  }
  bulk_wait_all();
}

cudaError_t ensure_append_attr() {
  static std::mutex mu;
  static bool done[kMaxDevices] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(append_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, APPEND_SMEM);
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

}  // namespace

bool append_tma_supported(const Geometry& g) {
  // a row-by-row copy puts each row at a 128-byte aligned shared-memory address (TMA)
  const int64_t row = (int64_t)g.h_kv * g.d * 2, row_al = (row + 127) / 128 * 128;
  return g.d % 8 == 0 && g.d <= 256 && g.h_kv <= 256 && g.k <= 256 && row % 16 == 0 &&
         (int64_t)g.k * row_al <= (int64_t)kSlotBytes;
}

bool make_tmap_pool_append(void* out256, const void* pool, int64_t num_blocks, const Geometry& g, const char** err) {
  auto fn = encode_fn(err);
  if (!fn) return false;
  const cuuint64_t d = (cuuint64_t)g.d, h = (cuuint64_t)g.h_kv, k = (cuuint64_t)g.k;
  // (d, head, slot, layer*2+kind, block): strides 2, k*d*2, d*2, h*k*d*2, L*2*h*k*d*2
  cuuint64_t dims[5] = {d, h, k, (cuuint64_t)g.L * 2, (cuuint64_t)num_blocks};
  cuuint64_t strides[4] = {k * d * 2, d * 2, h * k * d * 2, (cuuint64_t)g.L * 2 * h * k * d * 2};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 2; ++i) {
    cuuint32_t box[5] = {(cuuint32_t)d, (cuuint32_t)h, i == 0 ? (cuuint32_t)k : 1u, 1, 1};
    CUresult r = fn((CUtensorMap*)((char*)out256 + 128 * i), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, (void*)pool, dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      *err = "cuTensorMapEncodeTiled(pool, append) failed";
      return false;
    }
  }
  return true;
}

cudaError_t launch_append_tma(const Geometry& g, const void* pool_maps, const AppendItemDev* items, int32_t n_items,
                              const int32_t* ids, int32_t n_ids, const TablePatch* patches, int32_t n_patches,
                              int32_t* table, const InlineBlob* blob, int32_t off_ids, int32_t off_patch,
                              const void* k, const void* v, int64_t kv_rows, int32_t layer0, int32_t nl,
                              int32_t num_sms, cudaStream_t st) {
  cudaError_t e = ensure_append_attr();
  if (e != cudaSuccess) return e;
  if (nl <= 0) nl = g.L;
  const char* err = nullptr;
  auto fn = encode_fn(&err);
  if (!fn) return cudaErrorNotSupported;
  AppendTmaMaps m;
  const cuuint64_t d = (cuuint64_t)g.d, h = (cuuint64_t)g.h_kv;
  cuuint64_t dims[4] = {d, h, (cuuint64_t)kv_rows, (cuuint64_t)nl};
  cuuint64_t strides[3] = {d * 2, h * d * 2, (cuuint64_t)kv_rows * h * d * 2};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  for (int kind = 0; kind < 2; ++kind)
    for (int i = 0; i < 2; ++i) {
      cuuint32_t box[4] = {(cuuint32_t)d, (cuuint32_t)h, i == 0 ? (cuuint32_t)g.k : 1u, 1};
      CUresult r = fn(i == 0 ? &m.in_blk[kind] : &m.in_row[kind], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                      (void*)(kind ? v : k), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return cudaErrorNotSupported;
    }
  memcpy(&m.pool_blk, pool_maps, sizeof(CUtensorMap));
  memcpy(&m.pool_row, (const char*)pool_maps + 128, sizeof(CUtensorMap));
  const int64_t units = (int64_t)n_ids * nl * 2;
  if (units <= 0 && n_patches <= 0) return cudaSuccess;
  int32_t grid = (int32_t)(units < num_sms ? (units > 0 ? units : 1) : num_sms);
  static InlineBlob empty;
  const uint32_t row_bytes = (uint32_t)(h * d * 2), row_stride = (row_bytes + 127) / 128 * 128;
  return launch_k(append_tma_kernel, dim3(grid), dim3(kTmaThreads), APPEND_SMEM, st, m, items, n_items, ids, n_ids,
                  patches, n_patches, table, blob ? *blob : empty, blob ? 1 : 0, off_ids, off_patch, layer0, nl,
                  g.k, row_bytes, row_stride);
}

}  // namespace s2l
