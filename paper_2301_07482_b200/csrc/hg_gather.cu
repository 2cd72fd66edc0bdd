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
// A warp owns groups of kRows rows; consecutive lanes read consecutive 16 B of
// a row (coalesced 128-bit loads, no L1 allocation), and all loads of the group
// are issued before any store (memory-level parallelism per warp = kRows rows).
#include "hgb200.h"
#include <cuda_fp16.h>

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

constexpr int kRows = 8;        // rows a warp keeps in flight
constexpr int kMaxT = 4;        // 16-byte vectors per lane per row (rows <= 2 KB)

// One warp per group of kRows live rows. Lanes < kRows resolve the index chain
// (live -> node id -> region row) for the whole group at once, then every lane
// issues its 16-byte loads for all kRows rows before the first store, so each
// warp has up to kRows * kMaxT independent 128-bit loads in flight.
template <typename TIn, int kT>
__global__ void __launch_bounds__(256) k_load_rows(const int32_t* n_live_dev, const int32_t* __restrict__ live,
                                                   const int32_t* __restrict__ src_nodes,
                                                   const int32_t* __restrict__ feature_row_of,
                                                   const TIn* __restrict__ region, const TIn* __restrict__ feats,
                                                   int dim, float* __restrict__ out,
                                                   unsigned long long* __restrict__ gctr) {
  constexpr int kPerVec = 16 / sizeof(TIn);  // elements per 16-byte vector
  const int nvec = dim / kPerVec;
  const int n = *n_live_dev;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  KTimer* kt = g_kt ? g_kt + kTLoadRows : nullptr;
  kt_begin(kt);
  // index chain (live -> node id -> region row) of a group, resolved by lanes < kRows
  auto resolve = [&](int g, int& loc, const TIn*& row, bool& hit) {
    const int i = g * kRows + lane;
    loc = -1;
    row = nullptr;
    hit = false;
    if (lane < kRows && i < n) {
      loc = live[i];
      const int id = src_nodes[loc];
      const int fr = feature_row_of ? feature_row_of[id] : -1;
      hit = fr >= 0;
      row = hit ? region + (long long)fr * dim : feats + (long long)id * dim;
    }
  };
  int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int loc;
  const TIn* row;
  bool hit;
  resolve(g, loc, row, hit);
  // software pipeline: the next group's index chain is in flight while this
  // group's row loads complete
  for (; g * kRows < n; g += warps) {
    const unsigned hits = __ballot_sync(0xffffffffu, hit);
    const unsigned valid = __ballot_sync(0xffffffffu, loc >= 0);
    uint4 val[kRows][kT];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const TIn* p = reinterpret_cast<const TIn*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(row), r));
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int v = lane + 32 * t;
        if (((valid >> r) & 1u) && v < nvec) val[r][t] = ldg_stream_u4(reinterpret_cast<const uint4*>(p) + v);
      }
    }
    int cur_loc = loc;
    resolve(g + warps, loc, row, hit);
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int lr = __shfl_sync(0xffffffffu, cur_loc, r);
      if (!((valid >> r) & 1u)) continue;
      float* dst = out + (long long)lr * dim;
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int v = lane + 32 * t;
        if (v >= nvec) continue;
        if (sizeof(TIn) == 4) {
          reinterpret_cast<uint4*>(dst)[v] = val[r][t];
        } else {
          const __half2* h = reinterpret_cast<const __half2*>(&val[r][t]);
          float2 a = __half22float2(h[0]), b = __half22float2(h[1]);
          float2 c = __half22float2(h[2]), d = __half22float2(h[3]);
          reinterpret_cast<float4*>(dst)[2 * v] = make_float4(a.x, a.y, b.x, b.y);
          reinterpret_cast<float4*>(dst)[2 * v + 1] = make_float4(c.x, c.y, d.x, d.y);
        }
      }
    }
    if (lane == 0) {
      if (hits) atomicAdd(gctr + kGCtrFeatureHits, (unsigned long long)__popc(hits));
      if (valid & ~hits) atomicAdd(gctr + kGCtrFeatureMisses, (unsigned long long)__popc(valid & ~hits));
    }
  }
  kt_end(kt);
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

// dtype: 0 = fp32, 1 = fp16. dim * itemsize must be a multiple of 16 bytes.
int hg_load_features(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const int32_t* src_nodes,
                     const int32_t* feature_row_of, const void* region, const void* feats, int dim, int dtype,
                     float* h_out, long long* global_ctr, cudaStream_t stream) {
  const char* W = "hg_load_features";
  const int isz = dtype == 1 ? 2 : 4;
  if ((dim * isz) % 16) return fail(W, kBadArg, "feature row bytes must be a multiple of 16");
  if ((reinterpret_cast<uintptr_t>(feats) | reinterpret_cast<uintptr_t>(h_out)) & 15)
    return fail(W, kBadArg, "feature / output pointers must be 16-byte aligned");
  if (dim * isz > 16 * 32 * kMaxT) return fail(W, kBadArg, "feature rows above 2 KB are not supported");
  const unsigned grid = grid_for((n_live_max + kRows - 1) / kRows * 32, 256, 148 * 8);
  auto* g = reinterpret_cast<unsigned long long*>(global_ctr);
  const int T = (dim * isz / 16 + 31) / 32;
#define HG_LOAD(TT, KT)                                                                                     \
  k_load_rows<TT, KT><<<grid, 256, 0, stream>>>(n_live_dev, live, src_nodes, feature_row_of,               \
                                                static_cast<const TT*>(region), static_cast<const TT*>(feats), \
                                                dim, h_out, g)
  if (dtype == 1) {
    if (T == 1) HG_LOAD(__half, 1); else if (T == 2) HG_LOAD(__half, 2); else HG_LOAD(__half, 4);
  } else {
    if (T == 1) HG_LOAD(float, 1); else if (T == 2) HG_LOAD(float, 2); else HG_LOAD(float, 4);
  }
#undef HG_LOAD
  HG_LAUNCHED(W);
  return kOk;
}

}  // extern "C"
