// K3 + K4: cache-aware prune of one sampled block and the historical-cache
// lookup over the surviving frontier, bit-exact with histgnn/trainer.py:166-207
// and histgnn/cache.py:103-129 (oracle: oracle/step.py prune_with_cache,
// oracle/histcache.py _Ring.lookup).
//
// Block b (outer -> inner walk driven by the host):
//   keep[r]   = live_dst[r] && !inj_dst[r]           (live from block b+1's
//               frontier, inj = cache hits of layer b+1 over the same rows)
//   !keep[r]  -> end[r] = start[r]   (CSR2 O(1) row cut, counted as a prune write)
//   need_src  = keep rows (dst is a prefix of src) + sources of surviving rows
//   compute_rows = compact(keep), layer_live[b] = compact(need_src) (both sorted)
// then for b >= 1 the layer-b cache is probed for src_nodes[layer_live[b]]:
//   fresh <=> row_of >= 0 && (t_stale = inf || it - admit_iter <= t_stale)
//   expired entries are invalidated on the spot (staleness eviction).
// Hits become inj flags / cache rows for block b-1's dst rows.
#include "hgb200.h"
#include "hg_scan.cuh"
#include "hg_state.h"

namespace hg {
namespace {

__global__ void k_prune_rows(const int32_t* n_dst_dev, const uint8_t* __restrict__ live_dst,
                             const uint8_t* __restrict__ inj_dst, const int32_t* __restrict__ start,
                             int32_t* __restrict__ end, const int32_t* __restrict__ col,
                             uint8_t* __restrict__ keep, uint8_t* __restrict__ src_mask,
                             unsigned long long* prune_writes) {
  pdl_wait();
  const int n = *n_dst_dev;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const bool k = (!live_dst || live_dst[r]) && !(inj_dst && inj_dst[r]);
    keep[r] = k;
    if (!k) {
      end[r] = start[r];
    } else {
      src_mask[r] = 1;
      const int e1 = end[r];
      for (int e = start[r]; e < e1; ++e) src_mask[col[e]] = 1;
    }
    warp_count_add(prune_writes, !k);
  }
}

// both compactions of a block in one scan: (keep[i] for i < n_dst, src_mask[i])
struct KeepSrcFlags {
  const uint8_t* keep;
  const uint8_t* src_mask;
  const int32_t* n_dst_dev;
  __device__ I64x2 operator()(long long i) const {
    return {(i < *n_dst_dev && keep[i]) ? 1ll : 0ll, src_mask[i] ? 1ll : 0ll};
  }
};
struct EmitKeepSrc {
  int32_t* compute_rows;
  int32_t* pos_of;
  int32_t* live_src;
  const int32_t* n_dst_dev;
  __device__ void operator()(long long i, I64x2 excl, I64x2 v) const {
    if (i < *n_dst_dev) {
      if (v.a) compute_rows[excl.a] = (int32_t)i;
      pos_of[i] = v.a ? (int32_t)excl.a : -1;
    }
    if (v.b) live_src[excl.b] = (int32_t)i;
  }
};
struct StoreKeepSrcTotals {
  int32_t* counts;
  __device__ void operator()(I64x2 t) const {
    counts[0] = (int32_t)t.a;
    counts[1] = (int32_t)t.b;
  }
};

__global__ void k_lookup(const int32_t* n_live_dev, const int32_t* __restrict__ live,
                         const int32_t* __restrict__ src_nodes, int32_t* __restrict__ row_of,
                         const int32_t* __restrict__ admit_iter, int32_t* __restrict__ row_owner, const int* it_dev,
                         double t_stale, int t_inf, uint8_t* __restrict__ hit_flag, int32_t* __restrict__ hit_row,
                         long long* ctr) {
  pdl_wait();
  const int n = *n_live_dev;
  const int it = *it_dev;
  unsigned long long* c = reinterpret_cast<unsigned long long*>(ctr);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int loc = live[i];
    const int v = src_nodes[loc];
    const int r = row_of[v];
    bool fresh = r >= 0;
    bool expired = false;
    if (fresh && !t_inf) {
      const double age = (double)(it - admit_iter[v]);
      if (!(age <= t_stale)) {
        fresh = false;
        expired = true;
        row_owner[r] = -1;
        row_of[v] = -1;
      }
    }
    hit_flag[loc] = fresh;
    hit_row[loc] = fresh ? r : -1;
    warp_count_add(c + kCtrHits, fresh);
    warp_count_add(c + kCtrMisses, !fresh);
    warp_count_add(c + kCtrStalenessEvictions, expired);
    if (expired) atomicAdd(c + kCtrValid, (unsigned long long)-1ll);
  }
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

long long hg_prune_scratch_bytes(long long n_src_max) { return (scan_tiles(n_src_max) + 1) * 16 + 256; }

// Prune block b and (optionally) probe the layer-b cache. See hgb200.h.
int hg_prune_block(const int32_t* n_dst_dev, long long n_dst_max, const int32_t* n_src_dev, long long n_src_max,
                   const uint8_t* live_dst, const uint8_t* inj_dst, const int32_t* start, int32_t* end,
                   const int32_t* col, uint8_t* keep, int32_t* compute_rows, int32_t* pos_of, uint8_t* src_mask,
                   int32_t* live_src, int32_t* counts_dev, long long* global_ctr, void* scratch,
                   long long scratch_bytes, cudaStream_t stream) {
  const char* W = "hg_prune_block";
  if (scratch_bytes < hg_prune_scratch_bytes(n_src_max > n_dst_max ? n_src_max : n_dst_max))
    return fail(W, kBadArg, "scratch too small");
  HG_CHECK_CUDA(W, cudaMemsetAsync(src_mask, 0, (size_t)n_src_max, stream));
  { const cudaError_t _pe = hg::launch_pdl(k_prune_rows, dim3(grid_for(n_dst_max, 256)), dim3(256), 0, stream, 
      n_dst_dev, live_dst, inj_dst, start, end, col, keep, src_mask,
      reinterpret_cast<unsigned long long*>(global_ctr + kGCtrPruneWrites)); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  // compute rows (compact keep) and layer_live (compact src_mask) in one pass
  // over the block's sources (dst rows are a prefix of them)
  I64x2* part = reinterpret_cast<I64x2*>(scratch);
  return scan_launch<I64x2>(W, KeepSrcFlags{keep, src_mask, n_dst_dev}, DevCount{n_src_dev}, n_src_max, part,
                            EmitKeepSrc{compute_rows, pos_of, live_src, n_dst_dev}, StoreKeepSrcTotals{counts_dev},
                            stream);
}

int hg_cache_lookup(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const int32_t* src_nodes,
                    long long n_src_max, int32_t* row_of, const int32_t* admit_iter, int32_t* row_owner,
                    const int32_t* it_dev, double t_stale, uint8_t* hit_flag, int32_t* hit_row, long long* layer_ctr,
                    cudaStream_t stream) {
  const char* W = "hg_cache_lookup";
  HG_CHECK_CUDA(W, cudaMemsetAsync(hit_flag, 0, (size_t)n_src_max, stream));
  const int t_inf = isinf(t_stale) ? 1 : 0;
  { const cudaError_t _pe = hg::launch_pdl(k_lookup, dim3(grid_for(n_live_max, 256)), dim3(256), 0, stream, n_live_dev, live, src_nodes, row_of, admit_iter,
                                                          row_owner, it_dev, t_stale, t_inf, hit_flag, hit_row,
                                                          layer_ctr); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

}  // extern "C"
