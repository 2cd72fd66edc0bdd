// K10: historical-cache admission / eviction / ring scatter-update for one
// layer, bit-exact with histgnn/cache.py:131-204 (oracle: oracle/histcache.py).
//
//   U1  keys (norm fp64 bits, node id) for the live nodes; one device sort
//       (merge sort, or 96-bit LSD radix at large n) ranks them "norm
//       ascending, ties by id" (cache.py:191); ids are unique, so the order is
//       total and independent of the algorithm
//   U2  rank j >= k (k = floor(p_grad * n)): gradient eviction of cached nodes;
//       rank j < k: admitted; admitted & computed -> write flag
//   U3  compaction of write flags in rank order -> write list, n_write
//   U4  release the rows the written nodes held (cache.py:159 / :148)
//   U5  ring scan: rows (header + w) % cap lose their old owner, counted as a
//       forced eviction when age < t_stale (all when t_stale = inf), else as a
//       late staleness eviction (cache.py:175-186); the n_write >= cap branch
//       drops every live row (cache.py:145-157)
//   U6  scatter the embeddings + row_owner / row_of / admit_iter
//   U7  header update; U8 optional refresh of retained timestamps
// Norms are non-negative, so their IEEE bit patterns order like the values.
#include "hgb200.h"
#include <cub/device/device_merge_sort.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cstdlib>
#include <cstring>

#include "hg_scan.cuh"
#include "hg_state.h"

namespace hg {
namespace {

struct NormKey {
  unsigned long long norm;
  unsigned id;
};

struct NormKeyLess {
  __device__ bool operator()(const NormKey& a, const NormKey& b) const {
    return a.norm < b.norm || (a.norm == b.norm && a.id < b.id);
  }
};

// rank sort: CUB merge sort (block sort + merge-path passes) up to kMergeMaxN
// live nodes, CUB 96-bit LSD radix sort above (12 onesweep passes, better at
// large n). HG_CACHE_SORT=radix|merge overrides (A/B measurements).
constexpr long long kMergeMaxN = 1 << 20;
enum SortMode { kSortMerge = 1, kSortRadix = 2 };
inline int sort_mode(long long n_max) {
  static int v = -2;
  if (v == -2) {
    const char* e = std::getenv("HG_CACHE_SORT");
    v = !e ? -1 : (std::strcmp(e, "radix") == 0 ? kSortRadix : (std::strcmp(e, "merge") == 0 ? kSortMerge : -1));
  }
  if (v >= 0) return v;
  return n_max <= kMergeMaxN ? kSortMerge : kSortRadix;
}

struct NormKeyDecomposer {
  __host__ __device__ ::cuda::std::tuple<unsigned long long&, unsigned&> operator()(NormKey& k) const {
    return {k.norm, k.id};
  }
};

// keys for i < n; the tail up to n_max gets sentinels that sort last
__global__ void k_norm_keys(const int32_t* n_dev, int n_max, double p_grad, const int32_t* __restrict__ live,
                            const int32_t* __restrict__ src_nodes, const double* __restrict__ norms,
                            NormKey* __restrict__ keys, int32_t* __restrict__ vals, long long* ctr) {
  pdl_wait();
  const int n = *n_dev;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr[kCtrK] = (long long)floor(p_grad * (double)n);  // cache.py:190
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_max; i += gridDim.x * blockDim.x) {
    if (i < n) {
      keys[i] = NormKey{(unsigned long long)__double_as_longlong(norms[i]), (unsigned)src_nodes[live[i]]};
    } else {
      keys[i] = NormKey{~0ull, ~0u};
    }
    vals[i] = i;
  }
}

__global__ void k_rank_admit(const int32_t* n_dev, const NormKey* __restrict__ skeys,
                             const int32_t* __restrict__ svals, const int32_t* __restrict__ live,
                             const uint8_t* __restrict__ computed_flag, int32_t* __restrict__ row_of,
                             int32_t* __restrict__ row_owner, uint8_t* __restrict__ wflag,
                             uint8_t* __restrict__ retained, long long* ctr) {
  pdl_wait();
  unsigned long long* c = reinterpret_cast<unsigned long long*>(ctr);
  const int n = *n_dev;
  const long long k = ctr[kCtrK];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int id = (int)skeys[j].id;
    const int i = svals[j];
    const bool admitted = j < k;
    const bool computed = computed_flag[live[i]] != 0;
    bool evicted = false;
    if (!admitted) {
      const int r = row_of[id];
      if (r >= 0) {
        row_owner[r] = -1;
        row_of[id] = -1;
        evicted = true;
      }
    }
    wflag[j] = admitted && computed;
    retained[j] = admitted && !computed;
    warp_count_add(c + kCtrGradientEvictions, evicted);
    if (evicted) atomicAdd(c + kCtrValid, (unsigned long long)-1ll);
  }
}

struct StoreNWrite {
  long long* ctr;
  __device__ void operator()(int t) const { ctr[kCtrNWrite] = t; }
};

__global__ void k_release_writes(const int32_t* __restrict__ wlist, const NormKey* __restrict__ skeys, int cap,
                                 int32_t* __restrict__ row_of, int32_t* __restrict__ row_owner, long long* ctr) {
  pdl_wait();
  cap = (int)ctr[kCtrCapacity];  // logical ring size lives on the device (grows at sweeps)
  const long long nw = ctr[kCtrNWrite];
  const long long w0 = nw >= cap ? nw - cap : 0;
  const long long neff = nw - w0;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < neff; w += (long long)gridDim.x * blockDim.x) {
    const int id = (int)skeys[wlist[w0 + w]].id;
    const int r = row_of[id];
    if (r >= 0) {
      row_owner[r] = -1;
      row_of[id] = -1;
      atomicAdd(reinterpret_cast<unsigned long long*>(ctr) + kCtrValid, (unsigned long long)-1ll);
    }
  }
}

__global__ void k_ring_scan(int cap, const int32_t* it_dev, double t_stale, int t_inf, int32_t* __restrict__ row_of,
                            int32_t* __restrict__ row_owner, const int32_t* __restrict__ admit_iter, long long* ctr) {
  pdl_wait();
  cap = (int)ctr[kCtrCapacity];  // logical ring size lives on the device (grows at sweeps)
  const int it = *it_dev;
  const long long nw = ctr[kCtrNWrite];
  const long long header = ctr[kCtrHeader];
  const bool wrap_all = nw >= cap;
  const long long n = wrap_all ? cap : nw;
  unsigned long long* c = reinterpret_cast<unsigned long long*>(ctr);
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < n; w += (long long)gridDim.x * blockDim.x) {
    const int row = wrap_all ? (int)w : (int)((header + w) % cap);
    const int old = row_owner[row];
    bool forced = false, late = false;
    if (old >= 0) {
      const int age = it - admit_iter[old];
      forced = t_inf || (double)age < t_stale;
      late = !forced;
      row_of[old] = -1;
      if (wrap_all) row_owner[row] = -1;
    }
    warp_count_add(c + kCtrForcedEvictions, forced);
    warp_count_add(c + kCtrWindowForced, forced);
    warp_count_add(c + kCtrStalenessEvictions, late);
    if (forced || late) atomicAdd(c + kCtrValid, (unsigned long long)-1ll);
  }
}

// one warp per written row
__global__ void k_write_rows(const int32_t* __restrict__ wlist, const NormKey* __restrict__ skeys,
                             const int32_t* __restrict__ svals, const int32_t* __restrict__ live,
                             const float* __restrict__ emb, int H, int cap, const int32_t* it_dev,
                             float* __restrict__ table,
                             int32_t* __restrict__ row_of, int32_t* __restrict__ row_owner,
                             int32_t* __restrict__ admit_iter, long long* ctr) {
  pdl_wait();
  cap = (int)ctr[kCtrCapacity];  // logical ring size lives on the device (grows at sweeps)
  const long long nw = ctr[kCtrNWrite];
  const long long header = ctr[kCtrHeader];
  const bool wrap_all = nw >= cap;
  const long long w0 = wrap_all ? nw - cap : 0;
  const long long neff = nw - w0;
  const int lane = threadIdx.x & 31;
  const int it = *it_dev;
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < neff; w += warps) {
    const int j = wlist[w0 + w];
    const int id = (int)skeys[j].id;
    const int i = svals[j];
    const int row = wrap_all ? (int)w : (int)((header + w) % cap);
    const float* src = emb + (long long)live[i] * H;
    float* dst = table + (long long)row * H;
    if ((H & 3) == 0) {
      for (int v = lane; v < (H >> 2); v += 32)
        reinterpret_cast<float4*>(dst)[v] = reinterpret_cast<const float4*>(src)[v];
    } else {
      for (int v = lane; v < H; v += 32) dst[v] = src[v];
    }
    if (lane == 0) {
      row_owner[row] = id;
      row_of[id] = row;
      admit_iter[id] = it;
    }
  }
}

__global__ void k_commit(int cap, long long* ctr) {
  pdl_wait();
  cap = (int)ctr[kCtrCapacity];  // logical ring size lives on the device (grows at sweeps)
  const long long nw = ctr[kCtrNWrite];
  const bool wrap_all = nw >= cap;
  const long long neff = wrap_all ? cap : nw;
  if (nw == 0) return;
  ctr[kCtrHeader] = wrap_all ? neff % cap : (ctr[kCtrHeader] + nw) % cap;
  ctr[kCtrAdmissions] += neff;
  ctr[kCtrWindowAdmissions] += neff;
  ctr[kCtrValid] += neff;
}

__global__ void k_refresh(const long long* ctr, const uint8_t* __restrict__ retained,
                          const NormKey* __restrict__ skeys, const int32_t* __restrict__ row_of,
                          int32_t* __restrict__ admit_iter, const int32_t* it_dev) {
  pdl_wait();
  const long long k = ctr[kCtrK];
  const int it = *it_dev;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    if (!retained[j]) continue;
    const int id = (int)skeys[j].id;
    if (row_of[id] >= 0) admit_iter[id] = it;
  }
}

__global__ void k_iota_deg(long long n, const int64_t* __restrict__ start, const int64_t* __restrict__ end,
                           long long* __restrict__ deg, int32_t* __restrict__ ids) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    deg[i] = end[i] - start[i];
    ids[i] = (int32_t)i;
  }
}
__global__ void k_region_rows(long long k, const int32_t* __restrict__ sorted_ids, int32_t* __restrict__ chosen,
                              int32_t* __restrict__ feature_row_of) {
  pdl_wait();
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < k; p += (long long)gridDim.x * blockDim.x) {
    const int id = sorted_ids[p];
    const int row = (int)(k - 1 - p);  // max-degree node last (cache.py:348)
    chosen[row] = id;
    feature_row_of[id] = row;
  }
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

long long hg_cache_update_scratch_bytes(long long n_max) {
  size_t tmp = 0, tmp2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const NormKey*)nullptr, (NormKey*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)(n_max > 0 ? n_max : 1), NormKeyDecomposer{});
  cub::DeviceMergeSort::SortPairs(nullptr, tmp2, (NormKey*)nullptr, (int32_t*)nullptr, (int)(n_max > 0 ? n_max : 1),
                                  NormKeyLess{});
  if (tmp2 > tmp) tmp = tmp2;
  const long long n = n_max + 16;
  // keys_in, keys_out (16 B), vals_in, vals_out, wlist (4 B), wflag, retained (1 B), scan partials
  return n * 16 * 2 + n * 4 * 3 + n * 2 + (scan_tiles(n_max) + 1) * 4 + (long long)tmp + 2048;
}

// Stage 1 (U1-U3): rank and evict; leaves the write list + n_write on device.
// n (live nodes) is read from n_dev; n_max sizes the sort (sentinel padding),
// k = floor(p_grad * n) is computed on the device (cache.py:190).
// The caller allocates the ring table on first use after reading n_write.
int hg_cache_rank(const int32_t* n_dev, int n_max, double p_grad, const int32_t* live, const int32_t* src_nodes,
                  const double* norms, const uint8_t* computed_flag, int32_t* row_of, int32_t* row_owner,
                  long long* layer_ctr, void* scratch, long long scratch_bytes, cudaStream_t stream) {
  const char* W = "hg_cache_rank";
  if (scratch_bytes < hg_cache_update_scratch_bytes(n_max)) return fail(W, kBadArg, "scratch too small");
  if (n_max <= 0) return kOk;
  const long long nn = n_max + 16;
  char* p = reinterpret_cast<char*>(scratch);
  NormKey* keys_in = reinterpret_cast<NormKey*>(p);
  NormKey* keys_out = keys_in + nn;
  int32_t* vals_in = reinterpret_cast<int32_t*>(keys_out + nn);
  int32_t* vals_out = vals_in + nn;
  int32_t* wlist = vals_out + nn;
  uint8_t* wflag = reinterpret_cast<uint8_t*>(wlist + nn);
  uint8_t* retained = wflag + nn;
  int* part = reinterpret_cast<int*>(retained + nn + 16 - ((uintptr_t)(retained + nn) & 15));
  void* tmp = part + scan_tiles(n_max) + 4;
  size_t tmp_bytes = (size_t)(scratch_bytes - ((char*)tmp - p));
  const bool radix = sort_mode(n_max) == kSortRadix;
  // the merge sort is in place: keys go straight to keys_out / vals_out
  { const cudaError_t _pe = hg::launch_pdl(k_norm_keys, dim3(grid_for(n_max, 256)), dim3(256), 0, stream, n_dev, n_max, p_grad, live, src_nodes, norms,
                                                        radix ? keys_in : keys_out, radix ? vals_in : vals_out,
                                                        layer_ctr); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  cudaError_t e = radix ? cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, vals_in, vals_out, n_max,
                                                          NormKeyDecomposer{}, stream)
                        : cub::DeviceMergeSort::SortPairs(tmp, tmp_bytes, keys_out, vals_out, n_max, NormKeyLess{},
                                                          stream);
  if (e != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(e));
  { const cudaError_t _pe = hg::launch_pdl(k_rank_admit, dim3(grid_for(n_max, 256)), dim3(256), 0, stream, n_dev, keys_out, vals_out, live, computed_flag, row_of,
                                                         row_owner, wflag, retained, layer_ctr); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return scan_launch<int>(W, FlagU8{wflag}, DevCount{n_dev}, n_max, part, EmitCompact{wlist}, StoreNWrite{layer_ctr},
                          stream);
}

// Stage 2 (U4-U8): ring write into a table of `cap` rows of H floats.
int hg_cache_write(int n_max, int cap, int H, const int32_t* it_dev, double t_stale, int refresh_retained,
                   const int32_t* live, const float* emb, float* table, int32_t* row_of, int32_t* row_owner,
                   int32_t* admit_iter, long long* layer_ctr, void* scratch, long long scratch_bytes,
                   cudaStream_t stream) {
  const char* W = "hg_cache_write";
  if (n_max <= 0) return kOk;
  if (cap < 1) return fail(W, kBadArg, "capacity must be >= 1");
  const long long nn = n_max + 16;
  char* p = reinterpret_cast<char*>(scratch);
  NormKey* keys_out = reinterpret_cast<NormKey*>(p) + nn;
  int32_t* vals_out = reinterpret_cast<int32_t*>(keys_out + nn) + nn;
  int32_t* wlist = vals_out + nn;
  uint8_t* wflag = reinterpret_cast<uint8_t*>(wlist + nn);
  uint8_t* retained = wflag + nn;
  const int t_inf = isinf(t_stale) ? 1 : 0;
  const long long nmax = n_max;  // rows touched per update <= n_write <= n_max (a wrap needs n_write >= capacity)
  { const cudaError_t _pe = hg::launch_pdl(k_release_writes, dim3(grid_for(n_max, 256)), dim3(256), 0, stream, wlist, keys_out, cap, row_of, row_owner, layer_ctr); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  { const cudaError_t _pe = hg::launch_pdl(k_ring_scan, dim3(grid_for(nmax, 256)), dim3(256), 0, stream, cap, it_dev, t_stale, t_inf, row_of, row_owner, admit_iter,
                                                       layer_ctr); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  { const cudaError_t _pe = hg::launch_pdl(k_write_rows, dim3(grid_for((long long)n_max * 32, 256, 148 * 16)), dim3(256), 0, stream, 
      wlist, keys_out, vals_out, live, emb, H, cap, it_dev, table, row_of, row_owner, admit_iter, layer_ctr); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  { const cudaError_t _pe = hg::launch_pdl(k_commit, dim3(1), dim3(1), 0, stream, cap, layer_ctr); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  if (refresh_retained) {
    { const cudaError_t _pe = hg::launch_pdl(k_refresh, dim3(grid_for(n_max, 256)), dim3(256), 0, stream, layer_ctr, retained, keys_out, row_of, admit_iter, it_dev); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
    HG_LAUNCHED(W);
  }
  return kOk;
}

long long hg_degree_order_scratch_bytes(long long n) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, (const long long*)nullptr, (long long*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, (int)(n > 0 ? n : 1));
  return (n + 16) * (8 * 2 + 4 * 2) + (long long)tmp + 256;
}


// Static layer-0 region (cache.py:338-351): top-k in-degree nodes, ties to the
// lower id, stored ascending by degree. feature_row_of must be -1 filled.
int hg_feature_region(const int64_t* g_start, const int64_t* g_end, long long n, long long k, int32_t* chosen,
                      int32_t* feature_row_of, void* scratch, long long scratch_bytes, cudaStream_t stream) {
  const char* W = "hg_feature_region";
  if (scratch_bytes < hg_degree_order_scratch_bytes(n)) return fail(W, kBadArg, "scratch too small");
  if (k <= 0 || n <= 0) return kOk;
  char* p = reinterpret_cast<char*>(scratch);
  long long* deg = reinterpret_cast<long long*>(p);
  long long* deg_out = deg + n + 16;
  int32_t* ids = reinterpret_cast<int32_t*>(deg_out + n + 16);
  int32_t* ids_out = ids + n + 16;
  void* tmp = ids_out + n + 16;
  size_t tmp_bytes = (size_t)(scratch_bytes - ((char*)tmp - p));
  { const cudaError_t _pe = hg::launch_pdl(k_iota_deg, dim3(grid_for(n, 256)), dim3(256), 0, stream, n, g_start, g_end, deg, ids); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  cudaError_t e =
      cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, deg, deg_out, ids, ids_out, (int)n, 0, 64, stream);
  if (e != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(e));
  { const cudaError_t _pe = hg::launch_pdl(k_region_rows, dim3(grid_for(k, 256)), dim3(256), 0, stream, k, ids_out, chosen, feature_row_of); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

}  // extern "C"
