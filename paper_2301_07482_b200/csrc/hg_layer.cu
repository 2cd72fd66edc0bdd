// K6/K8/K9 + loss + SGD: the block convolutions around the dense transform.
// Restates histgnn/nn.py (oracle: oracle/step.py):
//   _mean_matrix / _gcn_matrix + a @ h_in   nn.py:101-128,148-156  -> k_aggregate
//   h_full[rows] = z ; h_full[inj] = cached  nn.py:288-293          -> k_scatter_rows, k_inject
//   cross_entropy (fp64 log-sum-exp)         nn.py:326-343          -> k_ce_rows, k_ce_loss
//   dz = relu_mask * d_out                   nn.py:167              -> k_gather_dz (top layer); below it
//                                                                      written by the next layer's k_transpose_agg
//   d_in = A^T (dz W^T) (+ self)             nn.py:171,175-176      -> CSC build + k_transpose_agg
//   node_grad_norms (fp64)                   nn.py:346-349          -> fused in k_transpose_agg
//   sgd_step                                 nn.py:355-360          -> k_sgd
//
// Layout: the GEMM operand of block b is A[R x ldA] with ldA = K + 4:
//   SAGE: A = [h_self | mean_nbr | 1 | 0 0 0], K = 2 d_in
//   GCN : A = [A_hat h            | 1 | 0 0 0], K = d_in
// and the parameters P[(K+1) x d_out] = [W (W_self; W_neigh) ; bias], so
// z = A[:, :K+1] @ P carries the bias and dP = A[:, :K+1]^T dz carries db.
// Sparse accumulation mirrors scipy's CSR/CSC loops: per edge
// sum = sum + coef * x with separate fp32 roundings (no FMA contraction), in
// CSR order forward and ascending dst-row order backward; fixed-order warp
// trees for the fp64 norms, so every run is bit-identical.
#include "hgb200.h"
#include <cuda_fp16.h>

#include "hg_scan.cuh"
#include "hg_segsort.cuh"
#include "hg_state.h"
#include "hg_ts.cuh"

namespace hg {
namespace {

__device__ KTimer* g_kt = nullptr;
}  // namespace
int set_timers_layer(void* p) {
  cudaError_t e = cudaMemcpyToSymbol(g_kt, &p, sizeof(p));
  return e == cudaSuccess ? kOk : fail("set_timers_layer", kCuda, cudaGetErrorString(e));
}
namespace {

constexpr int kKindGCN = 0;
constexpr int kKindSAGE = 1;
constexpr int kMaxVecPerLane = 8;  // d_in <= 1024 floats (kT = float4 per lane, templated)
constexpr int kMaxRowFloats = 1056;
// resident CTAs forced for the d <= 256 (kT <= 2) aggregation kernels:
// latency-bound edge-row gathers, so occupancy is the lever (measured C2:
// k_aggregate 0.155 -> 0.125 ms/step at 6, k_transpose_agg 0.106 -> 0.089 at 8)
#ifndef HG_AGG_MINB
#define HG_AGG_MINB 6
#endif
// hidden-layer rows through rowp (cache-hit rows in place, kSrc 3)
#ifndef HG_AGG_MINB3
#define HG_AGG_MINB3 6
#endif
#ifndef HG_AGG_EB3
#define HG_AGG_EB3 4
#endif
#ifndef HG_AGG_PIPE3
#define HG_AGG_PIPE3 1
#endif
#ifndef HG_AGG_MINBH       // layer 0 over fp16 rows (papers100M shape)
#define HG_AGG_MINBH 8
#endif
// wide rows: kT 4 (d <= 512) / kT 8 (d <= 1024) resident CTAs; fp16 rows
// (MAG240M 768-d) fit 4 CTAs in 64 registers without spills
#ifndef HG_AGG_MINB4
#define HG_AGG_MINB4 4
#endif
#ifndef HG_AGG_MINB8
#define HG_AGG_MINB8 3
#endif
#ifndef HG_AGG_MINB8H
#define HG_AGG_MINB8H 4
#endif
#ifndef HG_TAGG_MINB
#define HG_TAGG_MINB 8
#endif
#ifndef HG_TAGG_EB
#define HG_TAGG_EB 2
#endif
#ifndef HG_AGG_PIPE
#define HG_AGG_PIPE 1
#endif
// matrix sources (layers >= 1): 8 edge rows in flight per warp at 4 CTAs / SM
// (measured C2: 63 -> 56 us / step); the layer-0 in-place variant keeps 4
// rows at 6 CTAs / SM (8 rows at 4 CTAs: 66 -> 89 us)
#ifndef HG_AGG_EB
#define HG_AGG_EB 4
#endif
#ifndef HG_AGG_EB0
#define HG_AGG_EB0 8
#endif
#ifndef HG_AGG_MINB0
#define HG_AGG_MINB0 4
#endif // k_gather_dz staging: d_out <= 1056

__device__ __forceinline__ float4 f4_fmadd_rn(float4 acc, float c, float4 x) {
  return make_float4(__fadd_rn(acc.x, __fmul_rn(c, x.x)), __fadd_rn(acc.y, __fmul_rn(c, x.y)),
                     __fadd_rn(acc.z, __fmul_rn(c, x.z)), __fadd_rn(acc.w, __fmul_rn(c, x.w)));
}

__device__ __forceinline__ float gcn_coef(int dd, int sd) {
  return (float)(1.0 / sqrt(((double)dd + 1.0) * ((double)sd + 1.0)));
}

// Source rows of the aggregation: kSrc 0 = rows of the fp32 matrix h_in
// (layers >= 1, or a gathered layer-0 input); kSrc 1 / 2 = layer-0 feature
// rows read in place through per-source addresses rowp[c] (fp32 / fp16
// tables, hg_resolve_feature_rows); kSrc 3 = a hidden layer's fp32 rows
// through rowp (layer output rows, cache-hit rows in place in the ring:
// hg_resolve_hit_rows): the fp32 copy of every live feature row
// and its re-read are gone (K5 fused into K6). fp16 -> fp32 is exact, so the
// sums are bit-identical to the gathered path.
template <int kSrc>
__device__ __forceinline__ const void* src_row(const float* __restrict__ h_in,
                                               const unsigned long long* __restrict__ rowp, int c, int d) {
  if (kSrc == 0) return h_in + (long long)c * d;
  return reinterpret_cast<const void*>(rowp[c]);
}
template <int kSrc>
__device__ __forceinline__ float4 row_vec(const void* base, int v) {
  if (kSrc != 2) return reinterpret_cast<const float4*>(base)[v];
  const uint2 u = reinterpret_cast<const uint2*>(base)[v];
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

// one warp per compute row; kT = float4 vectors per lane (d <= 128 kT); the
// [self | agg | 1 | pad] row is staged in dynamic shared memory (row_floats
// per warp) before it is emitted as TS core rows
// HG_ROW_W=0: the transposed SAGE aggregation recomputes 1/cnt per edge (A/B)
#ifndef HG_ROW_W
#define HG_ROW_W 1
#endif

template <int kKind, int kT, int kSrc>
__global__ void __launch_bounds__(256, kT <= 2 ? (kSrc == 2 ? HG_AGG_MINBH : kSrc == 3 ? HG_AGG_MINB3 : kSrc ? HG_AGG_MINB : HG_AGG_MINB0) : (kT <= 4 ? HG_AGG_MINB4 : (kSrc == 2 ? HG_AGG_MINB8H : HG_AGG_MINB8))) k_aggregate(const int32_t* R_dev, const int32_t* __restrict__ rows,
                                                   const int32_t* __restrict__ start, const int32_t* __restrict__ end,
                                                   const int32_t* __restrict__ col, const int32_t* __restrict__ dst_deg,
                                                   const int32_t* __restrict__ src_deg, const float* __restrict__ h_in,
                                                   const unsigned long long* __restrict__ rowp,
                                                   int d, uint8_t* __restrict__ A_ts, long long plane, int row_floats,
                                                   float* __restrict__ row_w) {
  pdl_wait();
  extern __shared__ __align__(16) float agg_smem[];
  const int R = *R_dev;
  const int lane = threadIdx.x & 31;
  const int nv = d >> 2;
  const int K = kKind == kKindSAGE ? 2 * d : d;
  const int nK = (K + 1 + 31) / 32;          // TS column chunks of [. | 1 | 0 pad]
  float* srow = agg_smem + (size_t)(threadIdx.x >> 5) * row_floats;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  KTimer* kt = g_kt ? g_kt + (kSrc == 1 || kSrc == 2 ? kTAggregateFeat : kTAggregate) : nullptr;
  kt_begin(kt);
  // software-pipelined over the warp's rows: the next row's id is fetched at
  // the start of a row and its extents after the edge loads, and a row's own
  // (self) feature row is loaded before its edges, so per row only the
  // col -> (rowp ->) neighbour-row chain is exposed (HG_AGG_PIPE=0: the
  // unpipelined loop, A/B)
  int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int r = 0, e0 = 0, e1 = 0;
  if (i < R) {
    r = rows[i];
    e0 = start[r];
    e1 = end[r];
  }
  // measured (C2): the pipelined loop helps the layer-0 rows-in-place variant
  // (one more dependent hop per edge) and costs the matrix variant ~20 %
  constexpr bool kPipe = HG_AGG_PIPE && kSrc >= 1 && (kSrc != 3 || HG_AGG_PIPE3);
  constexpr int kEB = kSrc == 3 ? HG_AGG_EB3 : kSrc ? HG_AGG_EB : HG_AGG_EB0;   // edges in flight per warp
  for (; i < R; i += warps) {
    const int i_next = i + warps;
    const int r_next = kPipe && i_next < R ? rows[i_next] : 0;
    const int cnt = e1 - e0;
    const void* hs = src_row<kSrc>(h_in, rowp, r, d);
    // wide rows (kT >= 4) park the self row in the warp's staging row right
    // away instead of holding kT float4 registers across the edge loop
    // (K<SAGE, 8, fp16> needed 154 registers = one CTA per SM)
    constexpr bool kSelfSmem = kT >= 4;
    float4 xs[kSelfSmem ? 1 : kT];
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int v = lane + 32 * t;
      const float4 x = v < nv ? row_vec<kSrc>(hs, v) : make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (kSelfSmem) {
        if (v < nv) stage_put4(srow, v, x);
      } else {
        xs[t] = x;
      }
    }
    float4 acc[kT];
#pragma unroll
    for (int t = 0; t < kT; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    float cs = 0.f;
    if (kKind == kKindSAGE) {
      cs = cnt > 0 ? (float)(1.0 / (double)cnt) : 0.f;
      if (row_w && lane == 0) row_w[i] = cs;   // the backward's per-row mean weight
    }
    const int dd = kKind == kKindGCN ? dst_deg[r] : 0;
    int e = e0;
    for (; e + kEB <= e1; e += kEB) {
      int c[kEB];
      float w[kEB];
      const void* bp[kEB];
#pragma unroll
      for (int q = 0; q < kEB; ++q) {
        c[q] = col[e + q];
        w[q] = kKind == kKindSAGE ? cs : gcn_coef(dd, src_deg[c[q]]);
      }
#pragma unroll
      for (int q = 0; q < kEB; ++q) bp[q] = src_row<kSrc>(h_in, rowp, c[q], d);
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int v = lane + 32 * t;
        if (v < nv) {
          float4 x[kEB];
#pragma unroll
          for (int q = 0; q < kEB; ++q) x[q] = row_vec<kSrc>(bp[q], v);
#pragma unroll
          for (int q = 0; q < kEB; ++q) acc[t] = f4_fmadd_rn(acc[t], w[q], x[q]);
        }
      }
    }
    for (; e < e1; ++e) {
      const int c0 = col[e];
      const float w0 = kKind == kKindSAGE ? cs : gcn_coef(dd, src_deg[c0]);
      const void* b0 = src_row<kSrc>(h_in, rowp, c0, d);
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int v = lane + 32 * t;
        if (v < nv) acc[t] = f4_fmadd_rn(acc[t], w0, row_vec<kSrc>(b0, v));
      }
    }
    const int r_cur = r;
    if (i_next < R) {
      r = kPipe ? r_next : rows[i_next];
      e0 = start[r];
      e1 = end[r];
    }
    // assemble [self | agg | 1 | 0...] (SAGE) or [agg | 1 | 0...] (GCN) in smem,
    // then emit it as bf16 hi/lo TS core-matrix rows (hg_ts.cuh)
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int v = lane + 32 * t;
      if (v < nv) {
        const float4 x_self = kSelfSmem ? stage_get4(srow, v) : xs[kSelfSmem ? 0 : t];
        if (kKind == kKindSAGE) {
          if (!kSelfSmem) stage_put4(srow, v, x_self);
          stage_put4(srow, (d >> 2) + v, acc[t]);
        } else {
          const float ws = gcn_coef(dd, src_deg[r_cur]);
          stage_put4(srow, v, f4_fmadd_rn(acc[t], ws, x_self));
        }
      }
    }
    for (int c = K + lane; c < nK * 32; c += 32) stage_put1(srow, c, c == K ? 1.f : 0.f);
    __syncwarp();
    for (int g = lane; g < nK * 4; g += 32) ts_store8_staged(A_ts, nK * 4, plane, i, g, srow);
    __syncwarp();
  }
  // zero the padding rows of the last 128-row tile (the weight-gradient GEMM
  // reduces over rows, so they must not hold garbage)
  const int R_pad = (R + kTsRows - 1) / kTsRows * kTsRows;
  const float zeros[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int i = R + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < R_pad; i += warps)
    for (int g = lane; g < nK * 4; g += 32) ts_store8(A_ts, nK * 4, plane, i, g, zeros);
  kt_end(kt);
}

__global__ void k_scatter_rows(const int32_t* R_dev, const int32_t* __restrict__ rows, const float* __restrict__ Z,
                               int dout, int relu, float* __restrict__ h_out) {
  pdl_wait();
  const long long n = (long long)(*R_dev) * dout;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / dout), j = (int)(t - (long long)i * dout);
    float z = Z[t];
    if (relu) z = z > 0.f ? z : 0.f;
    h_out[(long long)rows[i] * dout + j] = z;
  }
}

// rowp[r] = address of source row r of the next layer: its cache row when
// flagged (local table, or owner ring: owner << 26 | row), else h_out row r
__global__ void k_resolve_hits(const int32_t* n_dev, const uint8_t* __restrict__ flag,
                               const int32_t* __restrict__ hit_row, const float* __restrict__ table,
                               const float* const* __restrict__ tables, int dim, const float* __restrict__ h_out,
                               unsigned long long* __restrict__ rowp) {
  pdl_wait();
  const int n = *n_dev;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const float* p = h_out + (long long)r * dim;
    if (flag[r]) {
      const int h = hit_row[r];
      p = tables ? tables[(unsigned)h >> 26] + (long long)((unsigned)h & ((1u << 26) - 1)) * dim
                 : table + (long long)h * dim;
    }
    rowp[r] = reinterpret_cast<unsigned long long>(p);
  }
}

__global__ void k_inject(const int32_t* n_dev, const uint8_t* __restrict__ flag, const int32_t* __restrict__ hit_row,
                         const float* __restrict__ table, int dim, float* __restrict__ h_out) {
  pdl_wait();
  // a warp takes 4 rows: lanes < 4 read their flag / cache row, then lane
  // group q (8 lanes) copies row q if it is injected, 16-byte vectors, all
  // four rows in flight
  constexpr int kRows = 4, kGL = 32 / kRows;
  const int n = *n_dev;
  const int lane = threadIdx.x & 31;
  const int q = lane / kGL, gl = lane % kGL;
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const bool vec = (dim & 3) == 0;
  const int nv = dim >> 2;
  for (long long r0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRows; r0 < n;
       r0 += warps * kRows) {
    int hr = -1;
    if (lane < kRows && r0 + lane < n && flag[r0 + lane]) hr = hit_row[r0 + lane];
    const int h = __shfl_sync(0xffffffffu, hr, q);
    if (h < 0) continue;
    const float* src = table + (long long)h * dim;
    float* dst = h_out + (r0 + q) * dim;
    if (vec && nv <= 8 * kGL) {
      float4 x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = gl + kGL * u;
        if (v < nv) x[u] = reinterpret_cast<const float4*>(src)[v];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = gl + kGL * u;
        if (v < nv) reinterpret_cast<float4*>(dst)[v] = x[u];
      }
    } else if (vec) {
      for (int v = gl; v < nv; v += kGL) reinterpret_cast<float4*>(dst)[v] = reinterpret_cast<const float4*>(src)[v];
    } else {
      for (int v = gl; v < dim; v += kGL) dst[v] = src[v];
    }
  }
}

// one warp per seed row; fp64 throughout like the reference
__global__ void k_ce_rows(const float* __restrict__ logits, const int32_t* __restrict__ labels, int B, int C,
                          float* __restrict__ dlogits, double* __restrict__ row_logp) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < B; i += warps) {
    const float* z = logits + (long long)i * C;
    double m = -INFINITY;
    for (int j = lane; j < C; j += 32) m = fmax(m, (double)z[j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    double s = 0.0;
    for (int j = lane; j < C; j += 32) s += exp((double)z[j] - m);
    s = warp_sum_fixed(s);
    const double lse = log(s);
    const int y = labels[i];
    for (int j = lane; j < C; j += 32) {
      const double lp = ((double)z[j] - m) - lse;
      double g = exp(lp);
      if (j == y) {
        g -= 1.0;
        row_logp[i] = lp;
      }
      dlogits[(long long)i * C + j] = (float)(g / (double)B);
    }
  }
}

__global__ void __launch_bounds__(1024) k_ce_loss(const double* __restrict__ row_logp, int B, double* loss) {
  pdl_wait();
  __shared__ double part[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < B; i += blockDim.x) s += row_logp[i];
  s = warp_sum_fixed(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
    t = warp_sum_fixed(t);
    if (threadIdx.x == 0) *loss = -t / (double)B;
  }
}

// dz[i] = d_h[rows[i]] * (h_out[rows[i]] > 0), emitted as TS (hg_ts.cuh): one
// thread per (row, 8-column group) -- 8 gradients (and 8 outputs for the
// ReLU mask) loaded, split, stored; padding rows / columns zero. Rows whose
// width is not a multiple of 4 take the scalar loads.
__global__ void __launch_bounds__(256) k_gather_dz(const int32_t* R_dev, const int32_t* __restrict__ rows,
                                                   const float* __restrict__ d_h, const float* __restrict__ h_out,
                                                   int dout, int relu, uint8_t* __restrict__ dz_ts, long long plane) {
  pdl_wait();
  const int R = *R_dev;
  const int nG = (dout + 31) / 32 * 4;
  const long long total = (long long)((R + kTsRows - 1) / kTsRows * kTsRows) * nG;
  const bool vec = (dout & 3) == 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / nG), g = (int)(t - (long long)i * nG);
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int c0 = g * 8;
    if (i < R && c0 < dout) {
      const long long base = (long long)rows[i] * dout + c0;
      if (vec) {
        const float4 a = *reinterpret_cast<const float4*>(d_h + base);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        if (c0 + 8 <= dout) {
          const float4 b = *reinterpret_cast<const float4*>(d_h + base + 4);
          v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        }
        if (relu) {
          const float4 ha = *reinterpret_cast<const float4*>(h_out + base);
          const float hv[8] = {ha.x, ha.y, ha.z, ha.w, 0.f, 0.f, 0.f, 0.f};
          float hb[4] = {0.f, 0.f, 0.f, 0.f};
          if (c0 + 8 <= dout) {
            const float4 h2 = *reinterpret_cast<const float4*>(h_out + base + 4);
            hb[0] = h2.x; hb[1] = h2.y; hb[2] = h2.z; hb[3] = h2.w;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (!((q < 4 ? hv[q] : hb[q - 4]) > 0.f)) v[q] = 0.f;
        }
      } else {
        for (int q = 0; q < 8 && c0 + q < dout; ++q) {
          v[q] = d_h[base + q];
          if (relu && !(h_out[base + q] > 0.f)) v[q] = 0.f;
        }
      }
    }
    ts_store8(dz_ts, nG, plane, i, g, v);
  }
}

// GAT layer 0: the transform operand from feature rows read in place
// (hg_gather_rows_ts), one thread per (row, 8-column group): load 8 values
// (fp32 or fp16 -> fp32), split, store -- no staging, every row's groups in
// flight at once; padding rows / columns zero
template <int kSrc>
__global__ void __launch_bounds__(256) k_gather_ts_flat(const int32_t* R_dev, const int32_t* __restrict__ rows,
                                                        const unsigned long long* __restrict__ rowp, int d,
                                                        uint8_t* __restrict__ A_ts, long long plane) {
  pdl_wait();
  const int R = *R_dev;
  const int nK = (d + 31) / 32;
  const int nG = nK * 4;
  const long long total = (long long)((R + kTsRows - 1) / kTsRows * kTsRows) * nG;
  KTimer* kt = g_kt ? g_kt + kTLoadRows : nullptr;
  kt_begin(kt);
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / nG), g = (int)(t - (long long)i * nG);
    float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int c0 = g * 8;
    if (i < R && c0 < d) {
      const char* src = reinterpret_cast<const char*>(rowp[rows[i]]);
      if (kSrc == 2) {
        if (c0 + 8 <= d) {
          const uint4 u = *reinterpret_cast<const uint4*>(src + (size_t)c0 * 2);
          const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 f = __half22float2(h[q]);
            v[2 * q] = f.x;
            v[2 * q + 1] = f.y;
          }
        } else {
          const __half* h = reinterpret_cast<const __half*>(src);
          for (int q = 0; q < 8 && c0 + q < d; ++q) v[q] = __half2float(h[c0 + q]);
        }
      } else {
        const float* f = reinterpret_cast<const float*>(src);
        const float4 a = *reinterpret_cast<const float4*>(f + c0);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        if (c0 + 8 <= d) {
          const float4 b = *reinterpret_cast<const float4*>(f + c0 + 4);
          v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        }
      }
    }
    ts_store8(A_ts, nG, plane, i, g, v);
  }
  kt_end(kt);
}

// Transposed (CSC) view of the surviving edges of a pruned block, built
// without a library sort and sized by the surviving edges (not the block's
// upper bound): per-source counts (atomics), their exclusive scan (segment
// offsets), placement of each surviving edge's dst position at an atomic
// cursor, then every segment sorted ascending. The values of a segment are
// the compute positions pos_of[row], increasing with the dst row, so the
// sorted segment is the stable CSR-order transpose (ascending dst rows, the
// order the fixed-order accumulation of k_transpose_agg relies on).

__global__ void k_csc_count(const int32_t* n_dst_dev, const int32_t* __restrict__ blk_off,
                            const uint8_t* __restrict__ keep, const int32_t* __restrict__ col,
                            int32_t* __restrict__ cnt) {
  pdl_wait();
  const int n = *n_dst_dev;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (!keep[r]) continue;
    for (int e = blk_off[r]; e < blk_off[r + 1]; ++e) atomicAdd(&cnt[col[e]], 1);
  }
}

struct CscCount {
  const int32_t* cnt;
  __device__ int operator()(long long i) const { return cnt[i]; }
};
struct EmitCsc {
  int32_t* seg_lo;
  int32_t* seg_hi;
  int32_t* cursor;
  __device__ void operator()(long long i, int excl, int v) const {
    seg_lo[i] = excl;
    cursor[i] = excl;
    seg_hi[i] = excl + v;
  }
};
struct NoTotal {
  __device__ void operator()(int) const {}
};

__global__ void k_csc_place(const int32_t* n_dst_dev, const int32_t* __restrict__ blk_off,
                            const uint8_t* __restrict__ keep, const int32_t* __restrict__ pos_of,
                            const int32_t* __restrict__ col, int32_t* __restrict__ cursor,
                            unsigned* __restrict__ vals) {
  pdl_wait();
  const int n = *n_dst_dev;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    if (!keep[r]) continue;
    const unsigned p = (unsigned)pos_of[r];
    for (int e = blk_off[r]; e < blk_off[r + 1]; ++e) vals[atomicAdd(&cursor[col[e]], 1)] = p;
  }
}

// d_in rows for the live sources of block l + their fp64 norms (one warp per source)
// the previous layer's dz operand written by the transposed aggregation
// (ts null: d_in rows are written instead and k_gather_dz builds dz)
struct DzOut {
  uint8_t* ts;            // TS operand [R_pad x nK*32] (hg_ts.cuh)
  long long plane;
  int nK;
  const int32_t* pos;     // compute position of each source in the previous layer (-1: none)
  const float* h;         // the previous layer's output rows (ReLU mask)
  int relu;
  const int32_t* R_dev;   // the previous layer's compute-row count
};

template <int kKind, int kT>
__global__ void __launch_bounds__(256, kT <= 2 ? HG_TAGG_MINB : 1) k_transpose_agg(
    const int32_t* n_live_dev, const int32_t* __restrict__ live, const int32_t* __restrict__ seg_lo,
    const int32_t* __restrict__ seg_hi, const unsigned* __restrict__ srt_vals, const int32_t* __restrict__ rows,
    const int32_t* __restrict__ start, const int32_t* __restrict__ end, const int32_t* __restrict__ dst_deg,
    const int32_t* __restrict__ src_deg, const int32_t* n_dst_dev, const int32_t* __restrict__ pos_of,
    const float* __restrict__ SG, int ldSG, int d, float* __restrict__ d_in, double* __restrict__ norms,
    const uint8_t* __restrict__ need_row, const float* __restrict__ row_w, DzOut dzo) {
  pdl_wait();
  extern __shared__ __align__(16) float ta_smem[];
  const int n = *n_live_dev;
  const int n_dst = *n_dst_dev;
  const int lane = threadIdx.x & 31;
  const int nv = d >> 2;
  const int goff = kKind == kKindSAGE ? d : 0;  // neighbour half of [S | G]
  const int warps = (gridDim.x * blockDim.x) >> 5;
  constexpr int kTEB = HG_TAGG_EB;
  KTimer* kt = g_kt ? g_kt + kTTransposeAgg : nullptr;
  kt_begin(kt);
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int c = live[i];
    float4 acc[kT];
#pragma unroll
    for (int t = 0; t < kT; ++t) acc[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int p0 = seg_lo[c], p1 = seg_hi[c];
    const int sd = kKind == kKindGCN ? src_deg[c] : 0;
    int p = p0;
    if (kKind == kKindSAGE && HG_ROW_W && row_w) {
      // kTEB edges per batch: their positions, weights and gradient rows are
      // loaded before any is accumulated (same summation order as one by one)
      for (; p + kTEB <= p1; p += kTEB) {
        int pos[kTEB];
        float w[kTEB];
#pragma unroll
        for (int q = 0; q < kTEB; ++q) pos[q] = (int)srt_vals[p + q];
#pragma unroll
        for (int q = 0; q < kTEB; ++q) w[q] = row_w[pos[q]];
#pragma unroll
        for (int t = 0; t < kT; ++t) {
          const int v = lane + 32 * t;
          if (v < nv) {
            float4 x[kTEB];
#pragma unroll
            for (int q = 0; q < kTEB; ++q)
              x[q] = reinterpret_cast<const float4*>(SG + (long long)pos[q] * ldSG + goff)[v];
#pragma unroll
            for (int q = 0; q < kTEB; ++q) acc[t] = f4_fmadd_rn(acc[t], w[q], x[q]);
          }
        }
      }
    }
    for (; p < p1; ++p) {
      const int pos = (int)srt_vals[p];
      float w;
      if (kKind == kKindSAGE && HG_ROW_W && row_w) {
        w = row_w[pos];                       // 1 / cnt of the row, from the forward
      } else if (kKind == kKindSAGE) {
        const int r = rows[pos];
        const int cnt = end[r] - start[r];
        w = (float)(1.0 / (double)cnt);
      } else {
        w = gcn_coef(dst_deg[rows[pos]], sd);
      }
      const float4* g = reinterpret_cast<const float4*>(SG + (long long)pos * ldSG + goff);
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int v = lane + 32 * t;
        if (v < nv) acc[t] = f4_fmadd_rn(acc[t], w, g[v]);
      }
    }
    const int self = c < n_dst ? pos_of[c] : -1;
    if (self >= 0) {
      const float4* s = reinterpret_cast<const float4*>(SG + (long long)self * ldSG);
      const float ws = kKind == kKindSAGE ? 1.f : gcn_coef(dst_deg[c], sd);
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int v = lane + 32 * t;
        if (v < nv) {
          if (kKind == kKindSAGE) {
            const float4 x = s[v];
            acc[t] = make_float4(__fadd_rn(acc[t].x, x.x), __fadd_rn(acc[t].y, x.y), __fadd_rn(acc[t].z, x.z),
                                 __fadd_rn(acc[t].w, x.w));
          } else {
            acc[t] = f4_fmadd_rn(acc[t], ws, s[v]);
          }
        }
      }
    }
    double sq = 0.0;
    float4* out = reinterpret_cast<float4*>(d_in + (long long)c * d);
    // rows the next layer does not compute (cache-injected) need only their
    // norm (the admission key, cache.py:188-191), not the gradient row itself
    const bool write = !dzo.ts && (!need_row || need_row[c]);
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int v = lane + 32 * t;
      if (v < nv) {
        if (write) out[v] = acc[t];
        sq += (double)acc[t].x * acc[t].x + (double)acc[t].y * acc[t].y + (double)acc[t].z * acc[t].z +
              (double)acc[t].w * acc[t].w;
      }
    }
    if (dzo.ts) {
      // the previous layer's dz row (k_gather_dz fused): ReLU-masked by its
      // output, emitted as TS at its compute position
      const int pn = dzo.pos[c];
      if (pn >= 0) {
        float* srow = ta_smem + (threadIdx.x >> 5) * (dzo.nK * 32);
        const float4* hp = reinterpret_cast<const float4*>(dzo.h + (long long)c * d);
#pragma unroll
        for (int t = 0; t < kT; ++t) {
          const int v = lane + 32 * t;
          if (v < nv) {
            float4 g = acc[t];
            if (dzo.relu) {
              const float4 h = hp[v];
              g = make_float4(h.x > 0.f ? g.x : 0.f, h.y > 0.f ? g.y : 0.f, h.z > 0.f ? g.z : 0.f,
                              h.w > 0.f ? g.w : 0.f);
            }
            stage_put4(srow, v, g);
          }
        }
        for (int j = d + lane; j < dzo.nK * 32; j += 32) stage_put1(srow, j, 0.f);
        __syncwarp();
        for (int g = lane; g < dzo.nK * 4; g += 32) ts_store8_staged(dzo.ts, dzo.nK * 4, dzo.plane, pn, g, srow);
        __syncwarp();
      }
    }
    sq = warp_sum_fixed(sq);
    if (lane == 0) norms[i] = sqrt(sq);
  }
  if (dzo.ts) {
    // zero the padding rows of dz's last 128-row tile (the weight-gradient
    // GEMM reduces over rows)
    const int R = *dzo.R_dev;
    const int R_pad = (R + kTsRows - 1) / kTsRows * kTsRows;
    const float zeros[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = R + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); r < R_pad; r += warps)
      for (int g = lane; g < dzo.nK * 4; g += 32) ts_store8(dzo.ts, dzo.nK * 4, dzo.plane, r, g, zeros);
  }
  kt_end(kt);
}

__global__ void k_sgd(float* __restrict__ p, const float* __restrict__ g, long long n, float eta) {
  pdl_wait();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = __fsub_rn(p[i], __fmul_rn(eta, g[i]));
}

// row norms of arbitrary fp32 rows (API node_grad_norms)
__global__ void k_row_norms(const float* __restrict__ x, long long n, int d, double* __restrict__ out) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    double s = 0.0;
    for (int j = lane; j < d; j += 32) {
      const double v = x[i * d + j];
      s += v * v;
    }
    s = warp_sum_fixed(s);
    if (lane == 0) out[i] = sqrt(s);
  }
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

static int aggregate_launch(const char* W, int kind, int src, const int32_t* R_dev, long long R_max,
                            const int32_t* rows, const int32_t* start, const int32_t* end, const int32_t* col,
                            const int32_t* dst_deg, const int32_t* src_deg, const float* h_in,
                            const unsigned long long* rowp, int d, void* A_ts, float* row_w, cudaStream_t stream) {
  if (d % 4 || d > 32 * 4 * kMaxVecPerLane) return fail(W, kBadArg, "d must be a multiple of 4 and <= 1024");
  // grid covers the compute rows and the zero padding up to the next 128-row tile
  const long long rows_pad = (R_max + kTsRows - 1) / kTsRows * kTsRows;
  const unsigned grid = grid_for(rows_pad * 32, 256, 148 * 16);
  uint8_t* a = static_cast<uint8_t*>(A_ts);
  const int K1 = (kind == kKindSAGE ? 2 * d : d) + 1;
  const long long plane = ts_plane_bytes(R_max, K1);
  const int row_floats = (K1 + 31) / 32 * 32;
  const size_t smem = (size_t)8 * row_floats * 4;
  const int vpl = (d / 4 + 31) / 32;
  cudaError_t pe = cudaSuccess;
#define HG_AGG(KIND, T, S)                                                                                        \
  {                                                                                                              \
    if (smem > 48 * 1024) {                                                                                      \
      pe = cudaFuncSetAttribute(k_aggregate<KIND, T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      if (pe != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(pe));                                      \
    }                                                                                                            \
    pe = hg::launch_pdl(k_aggregate<KIND, T, S>, dim3(grid), dim3(256), smem, stream, R_dev, rows, start, end,    \
                        col, dst_deg, src_deg, h_in, rowp, d, a, plane, row_floats, row_w);                      \
  }
#define HG_AGG_T(KIND, S)                                                                                         \
  if (vpl <= 1) HG_AGG(KIND, 1, S) else if (vpl <= 2) HG_AGG(KIND, 2, S) else if (vpl <= 4) HG_AGG(KIND, 4, S)   \
  else HG_AGG(KIND, 8, S)
#define HG_AGG_S(KIND)                                                                                            \
  if (src == 0) { HG_AGG_T(KIND, 0) } else if (src == 1) { HG_AGG_T(KIND, 1) } else if (src == 2) {            \
    HG_AGG_T(KIND, 2) } else { HG_AGG_T(KIND, 3) }
  if (kind == kKindSAGE) {
    HG_AGG_S(kKindSAGE)
  } else {
    HG_AGG_S(kKindGCN)
  }
#undef HG_AGG_S
#undef HG_AGG_T
#undef HG_AGG
  if (pe != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(pe));
  HG_LAUNCHED(W);
  return kOk;
}

int hg_aggregate_fwd(int kind, const int32_t* R_dev, long long R_max, const int32_t* rows, const int32_t* start,
                     const int32_t* end, const int32_t* col, const int32_t* dst_deg, const int32_t* src_deg,
                     const float* h_in, int d, void* A_ts, float* row_w, cudaStream_t stream) {
  return aggregate_launch("hg_aggregate_fwd", kind, 0, R_dev, R_max, rows, start, end, col, dst_deg, src_deg, h_in,
                          nullptr, d, A_ts, row_w, stream);
}

// layer 0 over feature rows read in place (rowp from hg_resolve_feature_rows);
// dtype 0 = fp32 table, 1 = fp16; d = the table's (padded) row width
int hg_aggregate_fwd_rows(int kind, const int32_t* R_dev, long long R_max, const int32_t* rows, const int32_t* start,
                          const int32_t* end, const int32_t* col, const int32_t* dst_deg, const int32_t* src_deg,
                          const unsigned long long* rowp, int dtype, int d, void* A_ts, float* row_w,
                          cudaStream_t stream) {
  if (dtype == 1 && d % 8) return fail("hg_aggregate_fwd_rows", kBadArg, "fp16 rows need d % 8 == 0");
  if (dtype < 0 || dtype > 2) return fail("hg_aggregate_fwd_rows", kBadArg, "dtype must be 0, 1 or 2");
  return aggregate_launch("hg_aggregate_fwd_rows", kind, dtype == 1 ? 2 : dtype == 2 ? 3 : 1, R_dev, R_max, rows, start, end, col,
                          dst_deg, src_deg, nullptr, rowp, d, A_ts, row_w, stream);
}

int hg_scatter_rows(const int32_t* R_dev, long long R_max, const int32_t* rows, const float* Z, int dout, int relu,
                    float* h_out, cudaStream_t stream) {
  { const cudaError_t _pe = hg::launch_pdl(k_scatter_rows, dim3(grid_for(R_max * dout, 256)), dim3(256), 0, stream, R_dev, rows, Z, dout, relu, h_out); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_scatter_rows");
  return kOk;
}

int hg_resolve_hit_rows(const int32_t* n_dev, long long n_max, const uint8_t* flag, const int32_t* hit_row,
                        const float* table, const float* const* tables, int dim, const float* h_out,
                        unsigned long long* rowp, cudaStream_t stream) {
  const char* W = "hg_resolve_hit_rows";
  if (dim < 4 || (dim & 3)) return fail(W, kBadArg, "rows must be a multiple of 4 floats");
  if (!table && !tables) return fail(W, kBadArg, "no cache table");
  if (n_max <= 0) return kOk;
  { const cudaError_t _pe = hg::launch_pdl(k_resolve_hits, dim3(grid_for(n_max, 256)), dim3(256), 0, stream, n_dev,
                                           flag, hit_row, table, tables, dim, h_out, rowp);
    if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

int hg_inject_rows(const int32_t* n_dev, long long n_max, const uint8_t* flag, const int32_t* hit_row,
                   const float* table, int dim, float* h_out, cudaStream_t stream) {
  { const cudaError_t _pe = hg::launch_pdl(k_inject, dim3(grid_for(n_max * 8, 256, 148 * 16)), dim3(256), 0, stream, n_dev, flag, hit_row, table, dim, h_out); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_inject_rows");
  return kOk;
}

int hg_cross_entropy(const float* logits, const int32_t* labels, int B, int C, float* dlogits, double* row_logp,
                     double* loss, cudaStream_t stream) {
  if (B < 1 || C < 1) return fail("hg_cross_entropy", kBadArg, "empty logits");
  { const cudaError_t _pe = hg::launch_pdl(k_ce_rows, dim3(grid_for((long long)B * 32, 256, 148 * 16)), dim3(256), 0, stream, logits, labels, B, C, dlogits, row_logp); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_cross_entropy");
  { const cudaError_t _pe = hg::launch_pdl(k_ce_loss, dim3(1), dim3(1024), 0, stream, row_logp, B, loss); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_cross_entropy");
  return kOk;
}

int hg_gather_dz(const int32_t* R_dev, long long R_max, const int32_t* rows, const float* d_h, const float* h_out,
                 int dout, int relu, void* dz_ts, cudaStream_t stream) {
  if (dout > kMaxRowFloats) return fail("hg_gather_dz", kBadArg, "row too wide");
  const long long rows_pad = (R_max + kTsRows - 1) / kTsRows * kTsRows;
  { const cudaError_t _pe = hg::launch_pdl(k_gather_dz, dim3(grid_for(rows_pad * ((dout + 31) / 32 * 4), 256, 148 * 32)), dim3(256), 0,
      stream, R_dev, rows, d_h, h_out, dout, relu, static_cast<uint8_t*>(dz_ts), ts_plane_bytes(R_max, dout));
    if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_gather_dz");
  return kOk;
}

int hg_gather_rows_ts(const int32_t* n_dev, long long n_max, const int32_t* rows, const unsigned long long* rowp,
                      int dtype, int d, void* A_ts, cudaStream_t stream) {
  const char* W = "hg_gather_rows_ts";
  if (d > kMaxRowFloats || d % 4 || (dtype == 1 && d % 8)) return fail(W, kBadArg, "row width");
  const long long rows_pad = (n_max + kTsRows - 1) / kTsRows * kTsRows;
  const int nG = (d + 31) / 32 * 4;
  const unsigned fgrid = grid_for(rows_pad * nG, 256, 148 * 32);
  const cudaError_t pe =
      dtype == 1 ? hg::launch_pdl(k_gather_ts_flat<2>, dim3(fgrid), dim3(256), 0, stream, n_dev, rows, rowp, d,
                                  static_cast<uint8_t*>(A_ts), ts_plane_bytes(n_max, d))
                 : hg::launch_pdl(k_gather_ts_flat<1>, dim3(fgrid), dim3(256), 0, stream, n_dev, rows, rowp, d,
                                  static_cast<uint8_t*>(A_ts), ts_plane_bytes(n_max, d));
  if (pe != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(pe));
  HG_LAUNCHED(W);
  return kOk;
}

long long hg_csc_scratch_bytes(long long E_max, long long n_src_max) {
  // cursors + long-segment list + its count + scan partials + merge buffer
  return (n_src_max + 16) * 4 * 2 + 64 + (scan_tiles(n_src_max) + 1) * 4 + (E_max + 16) * 4 + 1024;
}

// Transposed (CSC) view of the surviving edges of a pruned block: for every
// source c, vals[seg_lo[c] .. seg_hi[c]) = the compute positions of the kept
// dst rows that sampled it, ascending (k_csc_count / scan / k_csc_place /
// k_csc_sort_small / k_csc_sort_big; no library sort, work sized by the
// surviving edges). keys_sorted is unused (kept for the ABI).
int hg_build_csc(const int32_t* n_dst_dev, const int32_t* blk_off, const uint8_t* keep, const int32_t* pos_of,
                 const int32_t* col, long long E_max, long long n_src_max, unsigned* keys_sorted,
                 unsigned* vals_sorted, int32_t* seg_lo, int32_t* seg_hi, void* scratch, long long scratch_bytes,
                 cudaStream_t stream) {
  const char* W = "hg_build_csc";
  (void)keys_sorted;
  if (scratch_bytes < hg_csc_scratch_bytes(E_max, n_src_max)) return fail(W, kBadArg, "scratch too small");
  if (n_src_max <= 0) return kOk;
  char* p = reinterpret_cast<char*>(scratch);
  int32_t* cursor = reinterpret_cast<int32_t*>(p);
  int32_t* big = cursor + (n_src_max + 16);
  int32_t* n_big = big + (n_src_max + 16);
  int* part = reinterpret_cast<int*>(reinterpret_cast<char*>(n_big) + 64);
  unsigned* tmp = reinterpret_cast<unsigned*>(part + scan_tiles(n_src_max) + 1);
  // counts accumulate in seg_hi (overwritten by the scan's emit)
  HG_CHECK_CUDA(W, cudaMemsetAsync(seg_hi, 0, (size_t)n_src_max * 4, stream));
  HG_CHECK_CUDA(W, cudaMemsetAsync(n_big, 0, 4, stream));
  const long long n_dst_max = n_src_max;   // dst rows are a prefix of the sources
  HG_CHECK_CUDA(W, hg::launch_pdl(k_csc_count, dim3(grid_for(n_dst_max, 256)), dim3(256), 0, stream, n_dst_dev,
                                  blk_off, keep, col, seg_hi));
  HG_LAUNCHED(W);
  const int sc = scan_launch<int>(W, CscCount{seg_hi}, ConstCount{n_src_max}, n_src_max, part,
                                  EmitCsc{seg_lo, seg_hi, cursor}, NoTotal{}, stream);
  if (sc) return sc;
  HG_CHECK_CUDA(W, hg::launch_pdl(k_csc_place, dim3(grid_for(n_dst_max, 256)), dim3(256), 0, stream, n_dst_dev,
                                  blk_off, keep, pos_of, col, cursor, vals_sorted));
  HG_LAUNCHED(W);
  return segsort_launch<int32_t>(W, n_src_max, seg_lo, seg_hi, vals_sorted, tmp, big, n_big, stream);
}

int hg_transpose_agg(int kind, const int32_t* n_live_dev, long long n_live_max, const int32_t* live,
                     const int32_t* seg_lo, const int32_t* seg_hi, const unsigned* vals_sorted, const int32_t* rows,
                     const int32_t* start, const int32_t* end, const int32_t* dst_deg, const int32_t* src_deg,
                     const int32_t* n_dst_dev, const int32_t* pos_of, const float* SG, int ldSG, int d,
                     float* d_in, double* norms, const uint8_t* need_row, const float* row_w,
                     void* dz_ts, const int32_t* R_prev_dev, long long R_prev_max, const int32_t* pos_prev,
                     const float* h_prev, int relu_prev, cudaStream_t stream) {
  const char* W = "hg_transpose_agg";
  if (d % 4 || d > 32 * 4 * kMaxVecPerLane) return fail(W, kBadArg, "d must be a multiple of 4 and <= 1024");
  if (dz_ts && (!R_prev_dev || !pos_prev || !h_prev)) return fail(W, kBadArg, "dz output needs R, pos and h");
  const unsigned grid = grid_for(n_live_max * 32, 256, 148 * 16);
  const int vpl = (d / 4 + 31) / 32;
  DzOut dzo{static_cast<uint8_t*>(dz_ts), dz_ts ? ts_plane_bytes(R_prev_max, d) : 0, (d + 31) / 32, pos_prev,
            h_prev, relu_prev, R_prev_dev};
  const size_t smem = dz_ts ? (size_t)8 * dzo.nK * 32 * 4 : 0;
  cudaError_t pe = cudaSuccess;
#define HG_TA(KIND, T)                                                                                            \
  {                                                                                                              \
    const int sa = ensure_smem_attr((const void*)k_transpose_agg<KIND, T>, (int)smem, W);                      \
    if (sa) return sa;                                                                                           \
    pe = hg::launch_pdl(k_transpose_agg<KIND, T>, dim3(grid), dim3(256), smem, stream, n_live_dev, live, seg_lo,  \
                        seg_hi, vals_sorted, rows, start, end, dst_deg, src_deg, n_dst_dev, pos_of, SG, ldSG, d,  \
                        d_in, norms, need_row, row_w, dzo);                                                      \
  }
#define HG_TA_T(KIND)                                                                                             \
  if (vpl <= 1) HG_TA(KIND, 1) else if (vpl <= 2) HG_TA(KIND, 2) else if (vpl <= 4) HG_TA(KIND, 4)              \
  else HG_TA(KIND, 8)
  if (kind == kKindSAGE) {
    HG_TA_T(kKindSAGE)
  } else {
    HG_TA_T(kKindGCN)
  }
#undef HG_TA_T
#undef HG_TA
  if (pe != cudaSuccess) return fail(W, kCuda, cudaGetErrorString(pe));
  HG_LAUNCHED(W);
  return kOk;
}

int hg_sgd(float* params, const float* grads, long long n, float eta, cudaStream_t stream) {
  { const cudaError_t _pe = hg::launch_pdl(k_sgd, dim3(grid_for(n, 256)), dim3(256), 0, stream, params, grads, n, eta); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_sgd");
  return kOk;
}

int hg_row_norms(const float* x, long long n, int d, double* out, cudaStream_t stream) {
  { const cudaError_t _pe = hg::launch_pdl(k_row_norms, dim3(grid_for(n * 32, 256, 148 * 16)), dim3(256), 0, stream, x, n, d, out); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_row_norms");
  return kOk;
}

}  // extern "C"
