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
// Work is flattened to (row, 16-byte vector) items so consecutive threads
// read consecutive 16 B of the same row (coalesced 128-bit loads, no L1
// allocation) and each thread keeps kUnroll independent loads in flight.
#include "hgb200.h"
#include <cuda_fp16.h>

#include "hg_common.cuh"
#include "hg_state.h"

namespace hg {
namespace {

constexpr int kUnroll = 4;

template <typename TIn>
__global__ void __launch_bounds__(256) k_load_rows(const int32_t* n_live_dev, const int32_t* __restrict__ live,
                                                   const int32_t* __restrict__ src_nodes,
                                                   const int32_t* __restrict__ feature_row_of,
                                                   const TIn* __restrict__ region, const TIn* __restrict__ feats,
                                                   int dim, float* __restrict__ out,
                                                   unsigned long long* __restrict__ gctr) {
  constexpr int kPerVec = 16 / sizeof(TIn);  // elements per 16-byte vector
  const int nvec = dim / kPerVec;
  const long long n_items = (long long)(*n_live_dev) * nvec;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x + threadIdx.x; base < n_items;
       base += stride * kUnroll) {
    uint4 val[kUnroll];
    float* dst[kUnroll];
    bool hit[kUnroll], first[kUnroll], ok[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const long long it = base + u * stride;
      ok[u] = it < n_items;
      first[u] = false;
      hit[u] = false;
      dst[u] = nullptr;
      if (ok[u]) {
        const int i = (int)(it / nvec);
        const int v = (int)(it - (long long)i * nvec);
        const int loc = live[i];
        const int id = src_nodes[loc];
        const int fr = feature_row_of ? feature_row_of[id] : -1;
        hit[u] = fr >= 0;
        first[u] = v == 0;
        const TIn* row = hit[u] ? region + (long long)fr * dim : feats + (long long)id * dim;
        val[u] = ldg_stream_u4(reinterpret_cast<const uint4*>(row) + v);
        dst[u] = out + (long long)loc * dim + (long long)v * kPerVec;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (!ok[u]) continue;
      if (sizeof(TIn) == 4) {
        *reinterpret_cast<uint4*>(dst[u]) = val[u];
      } else {
        const __half2* h = reinterpret_cast<const __half2*>(&val[u]);
        float2 a = __half22float2(h[0]), b = __half22float2(h[1]);
        float2 c = __half22float2(h[2]), d = __half22float2(h[3]);
        reinterpret_cast<float4*>(dst[u])[0] = make_float4(a.x, a.y, b.x, b.y);
        reinterpret_cast<float4*>(dst[u])[1] = make_float4(c.x, c.y, d.x, d.y);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      warp_count_add(gctr + kGCtrFeatureHits, ok[u] && first[u] && hit[u]);
      warp_count_add(gctr + kGCtrFeatureMisses, ok[u] && first[u] && !hit[u]);
    }
  }
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
  const long long items = n_live_max * (dim * isz / 16);
  const unsigned grid = grid_for((items + kUnroll - 1) / kUnroll, 256, 148 * 8);
  auto* g = reinterpret_cast<unsigned long long*>(global_ctr);
  if (dtype == 1)
    k_load_rows<__half><<<grid, 256, 0, stream>>>(n_live_dev, live, src_nodes, feature_row_of,
                                                  static_cast<const __half*>(region),
                                                  static_cast<const __half*>(feats), dim, h_out, g);
  else
    k_load_rows<float><<<grid, 256, 0, stream>>>(n_live_dev, live, src_nodes, feature_row_of,
                                                 static_cast<const float*>(region), static_cast<const float*>(feats),
                                                 dim, h_out, g);
  HG_LAUNCHED(W);
  return kOk;
}

}  // extern "C"
