// K5: layer-0 input load (histgnn/trainer.py:326-343 + cache.py:274-284).
//
// For every live layer-0 frontier row: if the node sits in the static
// feature region (top in-degree nodes, HBM resident) its row is copied from
// the region table (a feature hit, no fetch), else from the feature source
// (HBM, a peer GPU's HBM or host memory mapped through UVA — any pointer the
// device can dereference). Rows are converted to fp32 into the block-0 input
// matrix at their local frontier position. Non-live rows are not touched
// (no kernel ever reads them).
//
// Persistent warps copy batches of 32 rows as a flat stream of 128-bit
// vectors (see k_load_rows); the bulk-copy (TMA engine) variant is opt-in.
#include "hgb200.h"
#include <cuda_fp16.h>
#include <cstdlib>
#include <cstring>

#include "hg_common.cuh"
#include "hg_state.h"

namespace hg {
namespace {

__device__ KTimer* g_kt = nullptr;
}  // namespace
int set_timers_gather(void* p) {
  cudaError_t e = cudaMemcpyToSymbol(g_kt, &p, sizeof(p));
  return e == cudaSuccess ? kOk : fail("set_timers_gather", kCuda, cudaGetErrorString(e));
}
namespace {

constexpr int kWarps = 8;       // warps per CTA (256 threads)

// Persistent warps; a warp owns batches of 32 live rows (lane r resolves row
// r's index chain live -> node id -> region row, 3 dependent loads). The rows
// of a batch are copied as one flat stream of (row, 16-byte vector) pairs
// spread over all 32 lanes, kU independent 128-bit loads per lane in flight
// (8 for fp32, 6 for fp16 whose conversion needs registers),
// so narrow rows (e.g. 100 fp32 = 25 vectors) keep every lane busy. The next
// batch's index chain advances one dependent step per chunk of the current
// batch, hiding its latency behind the row loads.
// Sharded source: the miss rows live in P owner shards, shard o
// holding nodes [bounds[o], bounds[o+1]) (histgnn/comms.py:329-337 contiguous
// partition); shard pointers may be peer-GPU memory mapped over NVLink (CUDA
// IPC), so a miss is a one-sided P2P read by the loading GPU.
struct Shards {
  const void* const* ptr;     // device array [P]
  const long long* bounds;    // device array [P + 1]
  int P;
  int local;                  // index of this GPU's own shard (remote-row accounting)
  unsigned long long* owner_rows;   // [P] rows read per owner shard (NULL = not counted)
};
constexpr int kMaxShards = 16;

template <typename TIn, int kU, bool kShard>
__global__ void __launch_bounds__(kWarps * 32, 4) k_load_rows(const int32_t* n_live_dev, const int32_t* __restrict__ live,
                                                           const int32_t* __restrict__ src_nodes,
                                                           const int32_t* __restrict__ feature_row_of,
                                                           const TIn* __restrict__ region,
                                                           const TIn* __restrict__ feats, int dim,
                                                           float* __restrict__ out,
                                                           unsigned long long* __restrict__ gctr, Shards sh) {
  pdl_wait();
  constexpr int kPerVec = 16 / sizeof(TIn);  // elements per 16-byte vector
  __shared__ const TIn* s_row[kWarps][32];
  __shared__ int s_loc[kWarps][32];
  __shared__ const TIn* s_shard[kMaxShards];
  __shared__ long long s_bound[kMaxShards + 1];
  if (kShard) {
    if (threadIdx.x < sh.P) s_shard[threadIdx.x] = static_cast<const TIn*>(sh.ptr[threadIdx.x]);
    if (threadIdx.x <= sh.P) s_bound[threadIdx.x] = sh.bounds[threadIdx.x];
    __syncthreads();
  }
  const int nvec = dim / kPerVec;
  const int n = *n_live_dev;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int W = (gridDim.x * blockDim.x) >> 5;
  KTimer* kt = g_kt ? g_kt + kTLoadRows : nullptr;
  kt_begin(kt);
  int b = blockIdx.x * kWarps + wib;
  // index chain of this warp's first batch
  int i = b * 32 + lane;
  bool ok = i < n;
  int loc = ok ? live[i] : 0;
  int id = ok ? src_nodes[loc] : 0;
  int fr = ok && feature_row_of ? feature_row_of[id] : -1;
  for (; b * 32 < n; b += W) {
    __syncwarp();
    bool remote = false;
    int own = -1;
    if (kShard) {
      const TIn* src = region + (long long)fr * dim;
      if (fr < 0) {
        int o = 0;
        while (o + 1 < sh.P && id >= s_bound[o + 1]) ++o;
        src = s_shard[o] + (long long)(id - s_bound[o]) * dim;
        remote = ok && o != sh.local;
        own = ok ? o : -1;
      }
      s_row[wib][lane] = src;
    } else {
      s_row[wib][lane] = fr >= 0 ? region + (long long)fr * dim : feats + (long long)id * dim;
    }
    s_loc[wib][lane] = loc;
    const unsigned valid = __ballot_sync(0xffffffffu, ok);
    const unsigned hits = __ballot_sync(0xffffffffu, ok && fr >= 0);
    const unsigned remotes = kShard ? __ballot_sync(0xffffffffu, remote) : 0u;
    __syncwarp();
    const int vtotal = __popc(valid) * nvec;  // valid rows are a prefix of the batch
    // next batch: the chain advances one dependent load per chunk
    i = (b + W) * 32 + lane;
    ok = i < n;
    int stage = 0;
    for (int c0 = 0; c0 < vtotal; c0 += 32 * kU) {
      uint4 val[kU];
      int dst[kU];
#pragma unroll
      for (int t = 0; t < kU; ++t) {
        const int k = c0 + t * 32 + lane;
        dst[t] = -1;
        if (k < vtotal) {
          const int r = k / nvec, v = k - r * nvec;
          val[t] = ldg_stream_u4(reinterpret_cast<const uint4*>(s_row[wib][r]) + v);
          dst[t] = s_loc[wib][r] * nvec + v;   // output vector index (in input vectors)
        }
      }
      if (stage == 0) loc = ok ? live[i] : 0;
      else if (stage == 1) id = ok ? src_nodes[loc] : 0;
      else if (stage == 2) fr = ok && feature_row_of ? feature_row_of[id] : -1;
      ++stage;
#pragma unroll
      for (int t = 0; t < kU; ++t) {
        if (dst[t] < 0) continue;
        if (sizeof(TIn) == 4) {
          reinterpret_cast<uint4*>(out)[dst[t]] = val[t];
        } else {
          const __half2* h = reinterpret_cast<const __half2*>(&val[t]);
          float2 a = __half22float2(h[0]), bb = __half22float2(h[1]);
          float2 c = __half22float2(h[2]), d = __half22float2(h[3]);
          reinterpret_cast<float4*>(out)[2 * (long long)dst[t]] = make_float4(a.x, a.y, bb.x, bb.y);
          reinterpret_cast<float4*>(out)[2 * (long long)dst[t] + 1] = make_float4(c.x, c.y, d.x, d.y);
        }
      }
    }
    if (stage <= 0) loc = ok ? live[i] : 0;
    if (stage <= 1) id = ok ? src_nodes[loc] : 0;
    if (stage <= 2) fr = ok && feature_row_of ? feature_row_of[id] : -1;
    if (lane == 0) {
      if (hits) atomicAdd(gctr + kGCtrFeatureHits, (unsigned long long)__popc(hits));
      if (valid & ~hits) atomicAdd(gctr + kGCtrFeatureMisses, (unsigned long long)__popc(valid & ~hits));
      if (remotes) atomicAdd(gctr + kGCtrRemoteRows, (unsigned long long)__popc(remotes));
    }
    if (kShard && sh.owner_rows) {   // per-owner transfer sizes (comms.py:326-337 requests_for_batch)
      for (int o = 0; o < sh.P; ++o) {
        const unsigned m = __ballot_sync(0xffffffffu, own == o);
        if (lane == 0 && m) atomicAdd(sh.owner_rows + o, (unsigned long long)__popc(m));
      }
    }
  }
  kt_end(kt);
}

// Layer-0 input by reference (K5 fused into K6): instead of copying every
// live source's feature row into an fp32 matrix, resolve its address once
// (region row, local table row, or owner shard row) into rowp[loc]; the
// layer-0 aggregation (k_aggregate<kSrc = 1 / 2>) reads the rows in place.
// Same I/O accounting as k_load_rows (feature hits / misses, remote and
// per-owner rows). One thread per live source.
template <bool kShard>
__global__ void k_resolve_rows(const int32_t* n_live_dev, const int32_t* __restrict__ live,
                               const int32_t* __restrict__ src_nodes, const int32_t* __restrict__ feature_row_of,
                               const char* __restrict__ region, const char* __restrict__ feats, long long row_bytes,
                               unsigned long long* __restrict__ rowp, unsigned long long* __restrict__ gctr,
                               Shards sh) {
  pdl_wait();
  const int n = *n_live_dev;
  const int lane = threadIdx.x & 31;
  for (int i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; i0 < n; i0 += gridDim.x * blockDim.x) {
    const int i = i0 + lane;
    const bool ok = i < n;
    int own = -1;
    bool remote = false, hit = false;
    if (ok) {
      const int loc = live[i];
      const int id = src_nodes[loc];
      const int fr = feature_row_of ? feature_row_of[id] : -1;
      const char* p;
      hit = fr >= 0;
      if (hit) {
        p = region + (long long)fr * row_bytes;
      } else if (kShard) {
        int o = 0;
        while (o + 1 < sh.P && id >= sh.bounds[o + 1]) ++o;
        p = static_cast<const char*>(sh.ptr[o]) + (long long)(id - sh.bounds[o]) * row_bytes;
        remote = o != sh.local;
        own = o;
      } else {
        p = feats + (long long)id * row_bytes;
      }
      rowp[loc] = reinterpret_cast<unsigned long long>(p);
    }
    const unsigned valid = __ballot_sync(0xffffffffu, ok);
    const unsigned hits = __ballot_sync(0xffffffffu, hit);
    const unsigned remotes = __ballot_sync(0xffffffffu, remote);
    if (lane == 0) {
      if (hits) atomicAdd(gctr + kGCtrFeatureHits, (unsigned long long)__popc(hits));
      if (valid & ~hits) atomicAdd(gctr + kGCtrFeatureMisses, (unsigned long long)__popc(valid & ~hits));
      if (remotes) atomicAdd(gctr + kGCtrRemoteRows, (unsigned long long)__popc(remotes));
    }
    if (kShard && sh.owner_rows) {
      for (int o = 0; o < sh.P; ++o) {
        const unsigned m = __ballot_sync(0xffffffffu, own == o);
        if (lane == 0 && m) atomicAdd(sh.owner_rows + o, (unsigned long long)__popc(m));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fp32 sources: the gather is a pure row copy, done by the TMA engine.
// Each warp streams groups of R rows (lane r < R owns row r of the group):
// cp.async.bulk global -> smem (one bulk copy per row, completion counted in
// bytes on the stage's mbarrier), then cp.async.bulk smem -> global into the
// row's frontier position. kS stages per warp keep kS-1 groups of loads in
// flight while earlier groups drain, without holding any row in registers.
constexpr int kBulkWarps = 2;
constexpr int kBulkStages = 4;
constexpr int kBulkSmem = 110 * 1024;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)));
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(su32(b)), "r"(parity)
                 : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// index chain (live -> node id -> region row) resolved for every live row at
// once, fully parallel and coalesced, so the copy kernel's issue loop has no
// dependent loads: src_ptr[i] = source row address; hit / miss counters
__global__ void __launch_bounds__(256) k_row_src(const int32_t* n_live_dev, const int32_t* __restrict__ live,
                                                 const int32_t* __restrict__ src_nodes,
                                                 const int32_t* __restrict__ feature_row_of,
                                                 const char* __restrict__ region, const char* __restrict__ feats,
                                                 int row_bytes, const char** __restrict__ src_ptr,
                                                 unsigned long long* __restrict__ gctr) {
  pdl_wait();
  const int n = *n_live_dev;
  unsigned long long* c = gctr;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i - (int)(threadIdx.x & 31) < n; i += gridDim.x * blockDim.x) {
    const bool valid = i < n;
    bool hit = false;
    if (valid) {
      const int id = src_nodes[live[i]];
      const int fr = feature_row_of ? feature_row_of[id] : -1;
      hit = fr >= 0;
      src_ptr[i] = hit ? region + (long long)fr * row_bytes : feats + (long long)id * row_bytes;
    }
    warp_count_add(c + kGCtrFeatureHits, hit);
    warp_count_add(c + kGCtrFeatureMisses, valid && !hit);
  }
}

__global__ void __launch_bounds__(kBulkWarps * 32) k_load_rows_bulk(
    const int32_t* n_live_dev, const int32_t* __restrict__ live, const char* const* __restrict__ src_ptr,
    int row_bytes, int rows_per_group, float* __restrict__ out) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = rows_per_group;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * kBulkStages;
  unsigned char* buf = smem + 128 + (size_t)warp * kBulkStages * R * row_bytes;
  if (lane == 0) {
    for (int s = 0; s < kBulkStages; ++s) bar_init(&bars[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  KTimer* kt = g_kt ? g_kt + kTLoadRows : nullptr;
  kt_begin(kt);
  const int n = *n_live_dev;
  const int ngroups = (n + R - 1) / R;
  const int W = gridDim.x * kBulkWarps;
  const int gw = blockIdx.x * kBulkWarps + warp;
  const int mine = gw < ngroups ? (ngroups - gw + W - 1) / W : 0;
  auto issue = [&](int it) {
    const int s = it % kBulkStages;
    const int i = (gw + it * W) * R + lane;
    const bool valid = lane < R && i < n;
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    if (lane == 0) bar_expect_tx(&bars[s], (uint32_t)__popc(vm) * (uint32_t)row_bytes);
    if (valid) bulk_load(buf + ((size_t)s * R + lane) * row_bytes, src_ptr[i], (uint32_t)row_bytes, &bars[s]);
  };
  for (int p = 0; p < kBulkStages - 1 && p < mine; ++p) issue(p);
  for (int it = 0; it < mine; ++it) {
    const int s = it % kBulkStages;
    bar_wait(&bars[s], (uint32_t)((it / kBulkStages) & 1));
    const int i = (gw + it * W) * R + lane;
    if (lane < R && i < n)
      bulk_store(reinterpret_cast<char*>(out) + (long long)live[i] * row_bytes, buf + ((size_t)s * R + lane) * row_bytes,
                 (uint32_t)row_bytes);
    const int nx = it + kBulkStages - 1;
    if (nx < mine) {
      bulk_wait_read1();  // the stage nx reuses was last stored from two groups ago
      issue(nx);
    }
  }
  bulk_wait_all();
  kt_end(kt);
}

// HG_GATHER=bulk selects the TMA copy path (given a workspace). Measured on
// C2 (400-byte rows): the bulk copies are TMA-issue bound (~67 us for 312K
// rows) and the index pre-pass adds ~16 us, so the register gather (~82 us)
// stays the default.
inline bool use_bulk_gather() {
  static const bool v = [] {
    const char* e = std::getenv("HG_GATHER");
    return e && std::strcmp(e, "bulk") == 0;
  }();
  return v;
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

long long hg_load_features_scratch_bytes(long long n_live_max) { return (n_live_max + 2) * 8 + 256; }

// dtype: 0 = fp32, 1 = fp16. dim * itemsize must be a multiple of 16 bytes.
// With a workspace (scratch, hg_load_features_scratch_bytes), fp32 rows are
// copied by the TMA engine (k_row_src + k_load_rows_bulk); otherwise, or for
// fp16 (converted on the fly), by the register gather k_load_rows.
int hg_load_features(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const int32_t* src_nodes,
                     const int32_t* feature_row_of, const void* region, const void* feats, int dim, int dtype,
                     float* h_out, long long* global_ctr, void* scratch, long long scratch_bytes,
                     cudaStream_t stream) {
  const char* W = "hg_load_features";
  const int isz = dtype == 1 ? 2 : 4;
  if ((dim * isz) % 16) return fail(W, kBadArg, "feature row bytes must be a multiple of 16");
  if ((reinterpret_cast<uintptr_t>(feats) | reinterpret_cast<uintptr_t>(h_out)) & 15)
    return fail(W, kBadArg, "feature / output pointers must be 16-byte aligned");
  if ((long long)dim * isz / 16 * 32 >= (1ll << 31)) return fail(W, kBadArg, "feature rows too wide");
  if (scratch && scratch_bytes < hg_load_features_scratch_bytes(n_live_max))
    return fail(W, kBadArg, "scratch too small");
  auto* g = reinterpret_cast<unsigned long long*>(global_ctr);
  if (dtype == 0 && scratch && use_bulk_gather()) {
    const int row_bytes = dim * 4;
    int R = (kBulkSmem - 128) / (kBulkWarps * kBulkStages * row_bytes);
    if (R > 32) R = 32;
    if (R >= 1) {
      const char** src_ptr = reinterpret_cast<const char**>((reinterpret_cast<uintptr_t>(scratch) + 15) & ~uintptr_t(15));
      k_row_src<<<grid_for(n_live_max, 256), 256, 0, stream>>>(n_live_dev, live, src_nodes, feature_row_of,
                                                               static_cast<const char*>(region),
                                                               static_cast<const char*>(feats), row_bytes, src_ptr, g);
      HG_LAUNCHED(W);
      const int sa = ensure_smem_attr((const void*)k_load_rows_bulk, kBulkSmem, W);
      if (sa) return sa;
      const long long groups = (n_live_max + R - 1) / R;
      long long blocks = (groups + kBulkWarps - 1) / kBulkWarps;
      if (blocks > 148 * 2) blocks = 148 * 2;
      if (blocks < 1) blocks = 1;
      const size_t smem = 128 + (size_t)kBulkWarps * kBulkStages * R * row_bytes;
      k_load_rows_bulk<<<(unsigned)blocks, kBulkWarps * 32, smem, stream>>>(n_live_dev, live, src_ptr, row_bytes, R,
                                                                              h_out);
      HG_LAUNCHED(W);
      return kOk;
    }
  }
  // persistent: one wave of 4 CTAs per SM (or fewer when the batch is small)
  const unsigned grid = grid_for((n_live_max + 31) / 32, kWarps, 148 * 4);
#define HG_LOAD(TT, U)                                                                                            \
  (void)hg::launch_pdl(k_load_rows<TT, U, false>, dim3(grid), dim3(kWarps * 32), 0, stream, n_live_dev, live,   \
                       src_nodes, feature_row_of, static_cast<const TT*>(region), static_cast<const TT*>(feats),  \
                       dim, h_out, g, Shards{nullptr, nullptr, 0, 0, nullptr})
  if (dtype == 1) HG_LOAD(__half, 6); else HG_LOAD(float, 8);
#undef HG_LOAD
  HG_LAUNCHED(W);
  return kOk;
}

// Sharded feature table: misses are read from shard o = owner(id) at
// shard_ptrs[o] + (id - bounds[o]) * dim (peer HBM over NVLink when the
// pointer is an IPC mapping of another GPU's shard). Region hits are local.
int hg_load_features_sharded(const int32_t* n_live_dev, long long n_live_max, const int32_t* live,
                             const int32_t* src_nodes, const int32_t* feature_row_of, const void* region,
                             const void* const* shard_ptrs, const long long* shard_bounds, int num_shards,
                             int local_shard, int dim, int dtype, float* h_out, long long* global_ctr,
                             long long* owner_rows, cudaStream_t stream) {
  const char* W = "hg_load_features_sharded";
  const int isz = dtype == 1 ? 2 : 4;
  if ((dim * isz) % 16) return fail(W, kBadArg, "feature row bytes must be a multiple of 16");
  if (num_shards < 1 || num_shards > kMaxShards) return fail(W, kBadArg, "num_shards must be in [1, 16]");
  if (!shard_ptrs || !shard_bounds) return fail(W, kBadArg, "shard tables must be given");
  if (reinterpret_cast<uintptr_t>(h_out) & 15) return fail(W, kBadArg, "output must be 16-byte aligned");
  auto* g = reinterpret_cast<unsigned long long*>(global_ctr);
  const unsigned grid = grid_for((n_live_max + 31) / 32, kWarps, 148 * 4);
  const Shards sh{shard_ptrs, shard_bounds, num_shards, local_shard,
                  reinterpret_cast<unsigned long long*>(owner_rows)};
  if (dtype == 1)
    { const cudaError_t _pe = hg::launch_pdl(k_load_rows<__half, 6, true>, dim3(grid), dim3(kWarps * 32), 0, stream, n_live_dev, live, src_nodes, feature_row_of,
                                                                  static_cast<const __half*>(region), nullptr, dim,
                                                                  h_out, g, sh); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  else
    { const cudaError_t _pe = hg::launch_pdl(k_load_rows<float, 8, true>, dim3(grid), dim3(kWarps * 32), 0, stream, n_live_dev, live, src_nodes, feature_row_of,
                                                                 static_cast<const float*>(region), nullptr, dim,
                                                                 h_out, g, sh); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

// K5 by reference: rowp[live[i]] = address of live source i's feature row
// (region / table / owner shard), with k_load_rows' accounting; the layer-0
// aggregation reads the rows in place (hg_aggregate_fwd_rows). shard_ptrs
// NULL = an unsharded table `feats`.
int hg_resolve_feature_rows(const int32_t* n_live_dev, long long n_live_max, const int32_t* live,
                            const int32_t* src_nodes, const int32_t* feature_row_of, const void* region,
                            const void* feats, const void* const* shard_ptrs, const long long* shard_bounds,
                            int num_shards, int local_shard, int dim, int dtype, unsigned long long* rowp,
                            long long* global_ctr, long long* owner_rows, cudaStream_t stream) {
  const char* W = "hg_resolve_feature_rows";
  const long long row_bytes = (long long)dim * (dtype == 1 ? 2 : 4);
  if (row_bytes % 16) return fail(W, kBadArg, "feature row bytes must be a multiple of 16");
  if (shard_ptrs && (num_shards < 1 || num_shards > kMaxShards)) return fail(W, kBadArg, "num_shards must be in [1, 16]");
  auto* g = reinterpret_cast<unsigned long long*>(global_ctr);
  const unsigned grid = grid_for(n_live_max, 256, 148 * 8);
  const Shards sh{shard_ptrs, shard_bounds, num_shards, local_shard, reinterpret_cast<unsigned long long*>(owner_rows)};
  cudaError_t pe;
  if (shard_ptrs)
    pe = hg::launch_pdl(k_resolve_rows<true>, dim3(grid), dim3(256), 0, stream, n_live_dev, live, src_nodes,
                        feature_row_of, static_cast<const char*>(region), nullptr, row_bytes, rowp, g, sh);
  else
    pe = hg::launch_pdl(k_resolve_rows<false>, dim3(grid), dim3(256), 0, stream, n_live_dev, live, src_nodes,
                        feature_row_of, static_cast<const char*>(region), static_cast<const char*>(feats), row_bytes,
                        rowp, g, sh);
  if (pe != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(pe));
  HG_LAUNCHED(W);
  return kOk;
}

// ---- shard memory + CUDA IPC (one-sided NVLink access to peer shards) ----
int hg_device_alloc(long long bytes, void** out) {
  if (!out || bytes < 1) return fail("hg_device_alloc", kBadArg, "bad arguments");
  cudaError_t e = cudaMalloc(out, (size_t)bytes);
  return e == cudaSuccess ? kOk : fail("hg_device_alloc", kCuda, cudaGetErrorString(e));
}

int hg_device_free(void* p) {
  cudaError_t e = cudaFree(p);
  return e == cudaSuccess ? kOk : fail("hg_device_free", kCuda, cudaGetErrorString(e));
}

long long hg_ipc_handle_bytes(void) { return (long long)sizeof(cudaIpcMemHandle_t); }

// handle_out: hg_ipc_handle_bytes() bytes; p must be the base of a cudaMalloc allocation
int hg_ipc_export(void* p, void* handle_out) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) return fail("hg_ipc_export", kCuda, cudaGetErrorString(e));
  std::memcpy(handle_out, &h, sizeof(h));
  return kOk;
}

int hg_ipc_open(const void* handle, void** out) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? kOk : fail("hg_ipc_open", kCuda, cudaGetErrorString(e));
}

int hg_ipc_close(void* p) {
  cudaError_t e = cudaIpcCloseMemHandle(p);
  return e == cudaSuccess ? kOk : fail("hg_ipc_close", kCuda, cudaGetErrorString(e));
}

}  // extern "C"
