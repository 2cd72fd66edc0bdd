// GAT block layer (BASELINE config 5). The reference has no
// GAT (histgnn/nn.py:28-30); the layer is defined by the CPU restatement in
// oracle/gat.py (dense + finite-difference pinned) and these kernels follow
// it step for step:
//   z = h_in[live] @ W                      tcgen05 GEMM (hg_ts_linear_fwd, rows = live)
//   el/er = per-head <z, a_src> / <z, a_dst> k_gat_scores (warp per live row)
//   softmax over surviving in-edges + self  k_gat_aggregate (warp per compute row,
//     + bias, ReLU, scatter to h_out[rows])   two passes: max, then exp-sum + weighted sum)
//   backward, per compute row i:            k_gat_bwd_dst: gz (ReLU-masked grad),
//                                             c_i = sum_j a_ij da_ij, der_i = sum_j ds_ij
//   backward, per live source j (CSC):      k_gat_bwd_src: dz_j = sum_i a_ij gz_i
//                                             + del_j a_src (+ der_j a_dst if j computes),
//                                             emitted as a TS operand for the dgrad / wgrad GEMMs
//   parameter vectors (a_src, a_dst, bias): per-CTA column partials accumulated by the two
//                                             backward kernels, k_gat_param_sum (fixed order)
//   d_in rows + fp64 node-gradient norms:   k_gat_scatter_norms
// No atomics on floats anywhere: every run is bit-identical.
#include "hgb200.h"

#include "hg_common.cuh"
#include "hg_ts.cuh"

// >= 4 resident CTAs for the attention kernels with rows <= 256 floats:
// their edge loops are latency-bound; measured C5 2.55e5 -> 3.04e5 seeds/s
// (backward 2.04 -> 1.42 ms/step) going from 1 (80 regs) to 4; 6 spills
#ifndef HG_GAT_MINB
#define HG_GAT_MINB 4
#endif
#ifndef HG_GAT_FWD_MINB
#define HG_GAT_FWD_MINB 6   // scores + aggregate: C5 3.24 -> 3.22 ms/step
#endif

namespace hg {
namespace {

constexpr int kMaxH = 8;
constexpr float kSlope = 0.2f;

__device__ __forceinline__ float leaky(float x) { return x > 0.f ? x : kSlope * x; }
__device__ __forceinline__ float leaky_d(float x) { return x > 0.f ? 1.f : kSlope; }

// per-head warp sums of per-lane partials (fixed shuffle tree)
template <int kH>
__device__ __forceinline__ void warp_sum_heads(float (&p)[kH]) {
#pragma unroll
  for (int h = 0; h < kH; ++h) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) p[h] += __shfl_xor_sync(0xffffffffu, p[h], o);
  }
}

// Column -> head map. kH > 0: compile-time (H == 1, or HF == 32 kT with kT a
// multiple of H, so lane column slot t always belongs to head t / (kT / kH));
// kH == 0: generic (runtime c / F, kMaxH select chain).
template <int kT, int kH>
struct Heads {
  static constexpr int N = kH > 0 ? kH : kMaxH;
  __device__ __forceinline__ static int of(int t, int c, int F) {
    if constexpr (kH == 1) return 0;
    else if constexpr (kH > 1) return t / (kT / kH);
    else return c / F;
  }
  __device__ __forceinline__ static void add(float (&p)[N], int t, int c, int F, float v) {
    if constexpr (kH > 0) {
      p[of(t, c, F)] += v;
    } else {
      const int h = c / F;
#pragma unroll
      for (int q = 0; q < kMaxH; ++q)
        if (q == h) p[q] += v;
    }
  }
  // lane q (< H) receives the value of head q
  __device__ __forceinline__ static float pick(const float (&p)[N], int lane) {
    float r = 0.f;
#pragma unroll
    for (int q = 0; q < N; ++q)
      if (lane == q) r = p[q];
    return r;
  }
  // warp sums of the per-lane head partials p, delivered to lane h (< H) for
  // head h. kH = 2^m: reduce-scatter (m halving exchanges, then 5 - m xor
  // steps on one value: kH - 1 + 5 - m shuffles) + one gather shuffle,
  // instead of kH full reductions; fixed order, so bit-reproducible.
  __device__ __forceinline__ static float sum_to_lanes(float (&p)[N], int lane) {
    if constexpr (kH == 2 || kH == 4 || kH == 8) {
      constexpr int m = kH == 2 ? 1 : (kH == 4 ? 2 : 3);
#pragma unroll
      for (int s = 0, half = kH / 2; s < m; ++s, half >>= 1) {
        const int o = 16 >> s;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
          const float send = up ? p[i] : p[i + half];
          const float keep = up ? p[i + half] : p[i];
          p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
#pragma unroll
      for (int o = 16 >> m; o > 0; o >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], o);
      return __shfl_sync(0xffffffffu, p[0], (lane & (kH - 1)) << (5 - m));
    } else {
      warp_sum_heads<N>(p);
      return pick(p, lane);
    }
  }
};

// el[j*H + h] = <z[j, hF:(h+1)F], a_src[hF:(h+1)F]>, er likewise with a_dst
template <int kT, int kH>
__global__ void __launch_bounds__(256, kT <= 8 ? HG_GAT_FWD_MINB : 1) k_gat_scores(const int32_t* n_dev, const int32_t* __restrict__ live,
                                                    const float* __restrict__ z, int HF, int H, int F,
                                                    const float* __restrict__ a_src, const float* __restrict__ a_dst,
                                                    float* __restrict__ el, float* __restrict__ er) {
  pdl_wait();
  using HM = Heads<kT, kH>;
  const int n = *n_dev;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
    const int j = live[i];
    float pl[HM::N], pr[HM::N];
#pragma unroll
    for (int h = 0; h < HM::N; ++h) pl[h] = pr[h] = 0.f;
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int c = lane + 32 * t;
      if (c < HF) {
        const float x = z[(long long)j * HF + c];
        HM::add(pl, t, c, F, x * a_src[c]);
        HM::add(pr, t, c, F, x * a_dst[c]);
      }
    }
    const float vl = HM::sum_to_lanes(pl, lane);
    const float vr = HM::sum_to_lanes(pr, lane);
    if (lane < H) {
      el[(long long)j * H + lane] = vl;
      er[(long long)j * H + lane] = vr;
    }
  }
}

// value of head h held by lane h of `v` (lanes < H hold one head each)
__device__ __forceinline__ float head_val(float v, int h) { return __shfl_sync(0xffffffffu, v, h); }

template <int kT, int kH>
__global__ void __launch_bounds__(256, kT <= 8 ? HG_GAT_FWD_MINB : 1) k_gat_aggregate(const int32_t* R_dev, const int32_t* __restrict__ rows,
                                                       const int32_t* __restrict__ start, const int32_t* __restrict__ end,
                                                       const int32_t* __restrict__ col, const float* __restrict__ z,
                                                       const float* __restrict__ el, const float* __restrict__ er,
                                                       int HF, int H, int F, const float* __restrict__ bias, int relu,
                                                       float* __restrict__ h_out, float* __restrict__ mx,
                                                       float* __restrict__ ssum) {
  pdl_wait();
  const int R = *R_dev;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += warps) {
    const int i = rows[r];
    const int e0 = start[i], e1 = end[i];
    const float eri = lane < H ? er[(long long)i * H + lane] : 0.f;
    // pass 1: per-head max of the attention logits (edges, then the self loop)
    float m = -INFINITY;
    for (int e = e0; e <= e1; ++e) {
      const int j = e < e1 ? col[e] : i;
      if (lane < H) m = fmaxf(m, leaky(el[(long long)j * H + lane] + eri));
    }
    // pass 2: exp-weights, their sum and the weighted sum of z rows
    float s = 0.f;
    float acc[kT];
#pragma unroll
    for (int t = 0; t < kT; ++t) acc[t] = 0.f;
    // software-pipelined: the next edge's source id is fetched while this
    // edge's z row is accumulated (same order)
    int j_n = e0 < e1 ? col[e0] : i;
    for (int e = e0; e <= e1; ++e) {
      const int j = j_n;
      if (e + 1 <= e1) j_n = e + 1 < e1 ? col[e + 1] : i;
      const float* zj = z + (long long)j * HF;
      float zv[kT];
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int c = lane + 32 * t;
        zv[t] = c < HF ? zj[c] : 0.f;
      }
      const float w = lane < H ? expf(leaky(el[(long long)j * H + lane] + eri) - m) : 0.f;
      s += w;
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int c = lane + 32 * t;
        const float wh = head_val(w, c < HF ? Heads<kT, kH>::of(t, c, F) : 0);
        if (c < HF) acc[t] = __fmaf_rn(wh, zv[t], acc[t]);
      }
    }
    float* out = h_out + (long long)i * HF;
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int c = lane + 32 * t;
      const float sh = head_val(s, c < HF ? Heads<kT, kH>::of(t, c, F) : 0);
      if (c < HF) {
        float v = acc[t] / sh + bias[c];
        if (relu) v = v > 0.f ? v : 0.f;
        out[c] = v;
      }
    }
    if (lane < H) {
      mx[(long long)r * H + lane] = m;
      ssum[(long long)r * H + lane] = s;
    }
  }
}

// Sum per-warp column partials v[kT] (lane owns columns lane + 32 t) over the
// 8 warps of the CTA in warp order and store them at out[c] (c < HF).
template <int kT>
__device__ __forceinline__ void block_colsum_store(float (&v)[kT], float (*red)[kT * 32], int HF, float* out) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < kT; ++t) red[wib][lane + 32 * t] = v[t];
  __syncthreads();
  for (int c = threadIdx.x; c < HF; c += blockDim.x) {
    float sacc = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) sacc += red[w][c];
    out[c] = sacc;
  }
  __syncthreads();
}

// backward, warp per compute row r (i = rows[r]):
//   gz = dL/dout masked by ReLU; c[r][h] = sum_j a_ij da_ij; der[r][h] = sum_j ds_ij
template <int kT, int kH>
__global__ void __launch_bounds__(256, kT <= 8 ? HG_GAT_MINB : 1) k_gat_bwd_dst(const int32_t* R_dev, const int32_t* __restrict__ rows,
                                                     const int32_t* __restrict__ start, const int32_t* __restrict__ end,
                                                     const int32_t* __restrict__ col, const float* __restrict__ z,
                                                     const float* __restrict__ el, const float* __restrict__ er,
                                                     const float* __restrict__ mx, const float* __restrict__ ssum,
                                                     const float* __restrict__ d_h, const float* __restrict__ h_out,
                                                     int relu, int HF, int H, int F, float* __restrict__ gz,
                                                     float* __restrict__ cc, float* __restrict__ der,
                                                     float* __restrict__ part) {
  pdl_wait();
  __shared__ float s_da[8][32][kMaxH], s_a[8][32][kMaxH], s_sl[8][32][kMaxH];
  __shared__ float s_red[8][kT * 32];
  const int R = *R_dev;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  // this warp's share of d bias = sum gz and d a_dst = sum der[h] z_i (rows in grid-stride order)
  float pb[kT], pd[kT];
#pragma unroll
  for (int t = 0; t < kT; ++t) pb[t] = pd[t] = 0.f;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += warps) {
    const int i = rows[r];
    float g[kT];
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int c = lane + 32 * t;
      g[t] = 0.f;
      if (c < HF) {
        const long long o = (long long)i * HF + c;
        g[t] = d_h[o];
        if (relu && !(h_out[o] > 0.f)) g[t] = 0.f;
        gz[(long long)r * HF + c] = g[t];
      }
    }
    const int e0 = start[i], e1 = end[i];
    const float eri = lane < H ? er[(long long)i * H + lane] : 0.f;
    const float mi = lane < H ? mx[(long long)r * H + lane] : 0.f;
    const float si = lane < H ? ssum[(long long)r * H + lane] : 1.f;
    float ci = 0.f, deri = 0.f;
    // rows of up to 32 edges (incl. the self loop; every sampled block, whose
    // degrees are bounded by the fanout) keep (da, a, slope) of each edge in
    // shared memory for the second pass instead of recomputing it
    const bool cached = e1 - e0 + 1 <= 32;
    for (int pass = 0; pass < 2; ++pass) {
      int j_n = e0 < e1 ? col[e0] : i;    // next edge's source, fetched one edge ahead
      for (int e = e0; e <= e1; ++e) {
        const int ei = e - e0;
        if (pass == 1 && cached) {
          if (lane < H) {
            const float da = s_da[wib][ei][lane], a = s_a[wib][ei][lane];
            deri += a * (da - ci) * s_sl[wib][ei][lane];
          }
          continue;
        }
        const int j = j_n;
        if (e + 1 <= e1) j_n = e + 1 < e1 ? col[e + 1] : i;
        const float* zj = z + (long long)j * HF;
        using HM = Heads<kT, kH>;
        float p[HM::N];
#pragma unroll
        for (int q = 0; q < HM::N; ++q) p[q] = 0.f;
#pragma unroll
        for (int t = 0; t < kT; ++t) {
          const int c = lane + 32 * t;
          if (c < HF) HM::add(p, t, c, F, g[t] * zj[c]);
        }
        const float da = HM::sum_to_lanes(p, lane);
        if (lane < H) {
          const float pre = el[(long long)j * H + lane] + eri;
          const float a = expf(leaky(pre) - mi) / si;
          if (pass == 0) {
            ci += a * da;
            if (cached) {
              s_da[wib][ei][lane] = da;
              s_a[wib][ei][lane] = a;
              s_sl[wib][ei][lane] = leaky_d(pre);
            }
          } else {
            deri += a * (da - ci) * leaky_d(pre);
          }
        }
      }
      __syncwarp();
    }
    if (lane < H) {
      cc[(long long)r * H + lane] = ci;
      der[(long long)r * H + lane] = deri;
    }
    const float* zi = z + (long long)i * HF;
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int c = lane + 32 * t;
      const float dh = head_val(deri, c < HF ? Heads<kT, kH>::of(t, c, F) : 0);
      if (c < HF) {
        pb[t] += g[t];
        pd[t] = __fmaf_rn(dh, zi[c], pd[t]);
      }
    }
  }
  float* pbk = part + (long long)blockIdx.x * 2 * HF;
  block_colsum_store<kT>(pb, s_red, HF, pbk);
  block_colsum_store<kT>(pd, s_red, HF, pbk + HF);
}

// backward, warp per live source j (CSC of the surviving edges; csc_pos[p]
// = compute position of the edge's dst row): dz_j and del_j. dz is emitted as
// TS row k (compact over the live list) for the dgrad / wgrad GEMMs.
template <int kT, int kH>
__global__ void __launch_bounds__(256, kT <= 8 ? HG_GAT_MINB : 1) k_gat_bwd_src(
    const int32_t* n_dev, const int32_t* __restrict__ live, const int32_t* __restrict__ seg_lo,
    const int32_t* __restrict__ seg_hi, const unsigned* __restrict__ csc_pos, const int32_t* __restrict__ rows,
    const int32_t* n_dst_dev, const int32_t* __restrict__ pos_of, const float* __restrict__ z,
    const float* __restrict__ el, const float* __restrict__ er, const float* __restrict__ mx,
    const float* __restrict__ ssum, const float* __restrict__ gz, const float* __restrict__ cc,
    const float* __restrict__ der, const float* __restrict__ a_src, const float* __restrict__ a_dst, int HF, int H,
    int F, uint8_t* __restrict__ dz_ts, long long plane, float* __restrict__ del, float* __restrict__ part) {
  pdl_wait();
  __shared__ __align__(16) float s_rows[8][kT * 32];
  __shared__ float s_red[8][kT * 32];
  float ps[kT];   // this warp's share of d a_src = sum del[h] z_j
#pragma unroll
  for (int t = 0; t < kT; ++t) ps[t] = 0.f;
  const int n = *n_dev;
  const int n_dst = *n_dst_dev;
  const int lane = threadIdx.x & 31;
  const int nK = (HF + 31) / 32;
  float* srow = s_rows[threadIdx.x >> 5];
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int k = w0; k < n; k += warps) {
    const int j = live[k];
    const float* zj = z + (long long)j * HF;
    float zr[kT], acc[kT];
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int c = lane + 32 * t;
      zr[t] = c < HF ? zj[c] : 0.f;
      acc[t] = 0.f;
    }
    const float elj = lane < H ? el[(long long)j * H + lane] : 0.f;
    float dl = 0.f;
    const int self = j < n_dst ? pos_of[j] : -1;
    const int p0 = seg_lo[j], p1 = seg_hi[j];
    // CSC edges (ascending dst row), then the self loop. Software-pipelined:
    // the next edge's position, dst row and per-head terms are fetched while
    // the current edge's gradient row is reduced (same summation order)
    const int p_end = self >= 0 ? p1 + 1 : p1;
    auto edge_pos = [&](int p) { return p < p1 ? (int)csc_pos[p] : self; };
    int pos_n = p0 < p_end ? edge_pos(p0) : 0;
    int i_n = p0 < p_end ? rows[pos_n] : 0;
    for (int p = p0; p < p_end; ++p) {
      const int pos = pos_n, i = i_n;
      float er_i = 0.f, mx_p = 0.f, ss_p = 1.f, cc_p = 0.f;
      if (lane < H) {
        er_i = er[(long long)i * H + lane];
        mx_p = mx[(long long)pos * H + lane];
        ss_p = ssum[(long long)pos * H + lane];
        cc_p = cc[(long long)pos * H + lane];
      }
      if (p + 1 < p_end) {
        pos_n = edge_pos(p + 1);
        i_n = rows[pos_n];
      }
      const float* gi = gz + (long long)pos * HF;
      using HM = Heads<kT, kH>;
      float gv[kT];
      float q8[HM::N];
#pragma unroll
      for (int q = 0; q < HM::N; ++q) q8[q] = 0.f;
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int c = lane + 32 * t;
        gv[t] = c < HF ? gi[c] : 0.f;
      }
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int c = lane + 32 * t;
        if (c < HF) HM::add(q8, t, c, F, gv[t] * zr[t]);
      }
      const float da = HM::sum_to_lanes(q8, lane);
      float a = 0.f;
      if (lane < H) {
        const float pre = elj + er_i;
        a = expf(leaky(pre) - mx_p) / ss_p;
        dl += a * (da - cc_p) * leaky_d(pre);
      }
#pragma unroll
      for (int t = 0; t < kT; ++t) {
        const int c = lane + 32 * t;
        const float ah = head_val(a, c < HF ? Heads<kT, kH>::of(t, c, F) : 0);
        if (c < HF) acc[t] = __fmaf_rn(ah, gv[t], acc[t]);
      }
    }
    const float dr = (self >= 0 && lane < H) ? der[(long long)self * H + lane] : 0.f;
#pragma unroll
    for (int t = 0; t < kT; ++t) {
      const int c = lane + 32 * t;
      const int h = c < HF ? Heads<kT, kH>::of(t, c, F) : 0;
      const float dlh = head_val(dl, h);
      const float drh = head_val(dr, h);
      float v = 0.f;
      if (c < HF) {
        v = __fmaf_rn(dlh, a_src[c], acc[t]);
        if (self >= 0) v = __fmaf_rn(drh, a_dst[c], v);
        ps[t] = __fmaf_rn(dlh, zr[t], ps[t]);
      }
      srow[c] = v;   // zero padding up to the 32-column chunk
    }
    if (lane < H) del[(long long)k * H + lane] = dl;
    __syncwarp();
    for (int g = lane; g < nK * 4; g += 32) ts_store8(dz_ts, nK * 4, plane, k, g, srow + g * 8);
    __syncwarp();
  }
  // zero the padding rows of the last 128-row tile (the weight-gradient GEMM reduces over rows)
  const int n_pad = (n + kTsRows - 1) / kTsRows * kTsRows;
  const float zeros[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int k = n + w0; k < n_pad; k += warps)
    for (int g = lane; g < nK * 4; g += 32) ts_store8(dz_ts, nK * 4, plane, k, g, zeros);
  block_colsum_store<kT>(ps, s_red, HF, part + (long long)blockIdx.x * HF);
}

constexpr int kGatMaxBlocks = 148 * 16;   // grid cap of the backward kernels (grid_for)

// d bias / d a_dst / d a_src: one warp per (vector, column) sums the
// per-CTA partials of the backward kernels in a fixed order (lane-strided
// runs, then a fixed shuffle tree), so every run gives the same bits.
__global__ void k_gat_param_sum(const float* __restrict__ part_dst, int nb_dst, const float* __restrict__ part_src,
                                int nb_src, int HF, float* __restrict__ d_att_src, float* __restrict__ d_att_dst,
                                float* __restrict__ d_bias) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < 3 * HF; w += warps) {
    const int q = w / HF, c = w - q * HF;
    float sacc = 0.f;
    if (q < 2) {
      for (int b = lane; b < nb_dst; b += 32) sacc += part_dst[(long long)b * 2 * HF + q * HF + c];
    } else {
      for (int b = lane; b < nb_src; b += 32) sacc += part_src[(long long)b * HF + c];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0) (q == 0 ? d_bias : (q == 1 ? d_att_dst : d_att_src))[c] = sacc;
  }
}

// d_in[live[k]] = SG[k]; norms[k] = ||SG[k]|| (fp64, fixed-order warp tree)
__global__ void k_gat_scatter_norms(const int32_t* n_dev, const int32_t* __restrict__ live,
                                    const float* __restrict__ SG, int d, float* __restrict__ d_in,
                                    double* __restrict__ norms) {
  pdl_wait();
  const int n = *n_dev;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n; k += warps) {
    const float* s = SG + (long long)k * d;
    float* o = d_in + (long long)live[k] * d;
    double sq = 0.0;
    for (int c = lane; c < d; c += 32) {
      const float v = s[c];
      o[c] = v;
      sq += (double)v * v;
    }
    sq = warp_sum_fixed(sq);
    if (lane == 0) norms[k] = sqrt(sq);
  }
}

inline int cols_per_lane(int HF) {
  const int t = (HF + 31) / 32;
  return t <= 1 ? 1 : t <= 2 ? 2 : t <= 4 ? 4 : t <= 8 ? 8 : t <= 16 ? 16 : -1;
}

}  // namespace
}  // namespace hg

using namespace hg;

// (kT, kH) dispatch: kH = H when the column -> head map is static (H == 1,
// or HF == 32 kT with kT % H == 0), else the generic kH = 0 variant
#define HG_GAT_T(T, KH, CALL)                            \
  switch (T) {                                          \
    case 1: { constexpr int kT = 1; constexpr int kH = (KH) <= 1 ? (KH) : 0; CALL; } break;   \
    case 2: { constexpr int kT = 2; constexpr int kH = (KH) <= 2 ? (KH) : 0; CALL; } break;   \
    case 4: { constexpr int kT = 4; constexpr int kH = (KH) <= 4 ? (KH) : 0; CALL; } break;   \
    case 8: { constexpr int kT = 8; constexpr int kH = (KH); CALL; } break;                    \
    default: { constexpr int kT = 16; constexpr int kH = (KH); CALL; } break;                 \
  }
#define HG_GAT_DISPATCH(HF_, H_, CALL)                                             \
  {                                                                                \
    const int T_ = cols_per_lane(HF_);                                             \
    const int kh_ = static_head_map(HF_, H_, T_);                                  \
    if (kh_ == 1) HG_GAT_T(T_, 1, CALL)                                            \
    else if (kh_ == 2) HG_GAT_T(T_, 2, CALL)                                       \
    else if (kh_ == 4) HG_GAT_T(T_, 4, CALL)                                       \
    else if (kh_ == 8) HG_GAT_T(T_, 8, CALL)                                       \
    else HG_GAT_T(T_, 0, CALL)                                                     \
  }

inline int static_head_map(int HF, int H, int T) {
  if (H == 1) return 1;
  if (HF == 32 * T && T % H == 0 && (H == 2 || H == 4 || H == 8)) return H;
  return 0;
}

static int gat_check(const char* W, int HF, int H) {
  if (H < 1 || H > kMaxH) return fail(W, kBadArg, "heads must be in [1, 8]");
  if (HF % H) return fail(W, kBadArg, "d_out must be a multiple of heads");
  if (cols_per_lane(HF) < 0) return fail(W, kBadArg, "d_out must be <= 512");
  return kOk;
}

extern "C" {

int hg_gat_scores(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const float* z, int HF, int H,
                  const float* att_src, const float* att_dst, float* el, float* er, cudaStream_t stream) {
  const char* W = "hg_gat_scores";
  if (int st = gat_check(W, HF, H)) return st;
  const unsigned grid = grid_for(n_live_max * 32, 256, 148 * 16);
  HG_GAT_DISPATCH(HF, H, ((void)hg::launch_pdl(k_gat_scores<kT, kH>, dim3(grid), dim3(256), 0, stream, n_live_dev, live, z, HF, H, HF / H,
                                                                                  att_src, att_dst, el, er)));
  HG_LAUNCHED(W);
  return kOk;
}

int hg_gat_aggregate(const int32_t* R_dev, long long R_max, const int32_t* rows, const int32_t* start,
                     const int32_t* end, const int32_t* col, const float* z, const float* el, const float* er, int HF,
                     int H, const float* bias, int relu, float* h_out, float* mx, float* ssum, cudaStream_t stream) {
  const char* W = "hg_gat_aggregate";
  if (int st = gat_check(W, HF, H)) return st;
  const unsigned grid = grid_for(R_max * 32, 256, 148 * 16);
  HG_GAT_DISPATCH(HF, H,
                  ((void)hg::launch_pdl(k_gat_aggregate<kT, kH>, dim3(grid), dim3(256), 0, stream, R_dev, rows, start, end, col, z, el, er, HF, H,
                                                                  HF / H, bias, relu, h_out, mx, ssum)));
  HG_LAUNCHED(W);
  return kOk;
}

int hg_gat_bwd_dst(const int32_t* R_dev, long long R_max, const int32_t* rows, const int32_t* start,
                   const int32_t* end, const int32_t* col, const float* z, const float* el, const float* er,
                   const float* mx, const float* ssum, const float* d_h, const float* h_out, int relu, int HF, int H,
                   float* gz, float* cc, float* der, float* part, cudaStream_t stream) {
  const char* W = "hg_gat_bwd_dst";
  if (int st = gat_check(W, HF, H)) return st;
  const unsigned grid = grid_for(R_max * 32, 256, 148 * 16);
  HG_GAT_DISPATCH(HF, H,
                  ((void)hg::launch_pdl(k_gat_bwd_dst<kT, kH>, dim3(grid), dim3(256), 0, stream, R_dev, rows, start, end, col, z, el, er, mx, ssum, d_h,
                                                                h_out, relu, HF, H, HF / H, gz, cc, der, part)));
  HG_LAUNCHED(W);
  return kOk;
}

int hg_gat_bwd_src(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const int32_t* seg_lo,
                   const int32_t* seg_hi, const unsigned* csc_pos, const int32_t* rows, const int32_t* n_dst_dev,
                   const int32_t* pos_of, const float* z, const float* el, const float* er, const float* mx,
                   const float* ssum, const float* gz, const float* cc, const float* der, const float* att_src,
                   const float* att_dst, int HF, int H, void* dz_ts, float* del, float* part, cudaStream_t stream) {
  const char* W = "hg_gat_bwd_src";
  if (int st = gat_check(W, HF, H)) return st;
  const long long rows_pad = (n_live_max + kTsRows - 1) / kTsRows * kTsRows;
  const unsigned grid = grid_for(rows_pad * 32, 256, 148 * 16);
  const long long plane = ts_plane_bytes(n_live_max, HF);
  HG_GAT_DISPATCH(HF, H,
                  ((void)hg::launch_pdl(k_gat_bwd_src<kT, kH>, dim3(grid), dim3(256), 0, stream, n_live_dev, live, seg_lo, seg_hi, csc_pos, rows,
                                                                n_dst_dev, pos_of, z, el, er, mx, ssum, gz, cc, der,
                                                                att_src, att_dst, HF, H, HF / H,
                                                                static_cast<uint8_t*>(dz_ts), plane, del, part)));
  HG_LAUNCHED(W);
  return kOk;
}

// partial buffers of the backward kernels: [kGatMaxBlocks][2][HF] (dst) then
// [kGatMaxBlocks][HF] (src)
long long hg_gat_param_scratch_bytes(int HF) { return (long long)kGatMaxBlocks * 3 * HF * 4; }

int hg_gat_param_grads(long long R_max, long long n_live_max, int HF, const float* part_dst, const float* part_src,
                       float* d_att_src, float* d_att_dst, float* d_bias, cudaStream_t stream) {
  const char* W = "hg_gat_param_grads";
  // the grids hg_gat_bwd_dst / hg_gat_bwd_src used (every CTA wrote its partial)
  const int nb_dst = (int)grid_for(R_max * 32, 256, 148 * 16);
  const long long rows_pad = (n_live_max + kTsRows - 1) / kTsRows * kTsRows;
  const int nb_src = (int)grid_for(rows_pad * 32, 256, 148 * 16);
  { const cudaError_t _pe = hg::launch_pdl(k_gat_param_sum, dim3(grid_for(3LL * HF * 32, 256)), dim3(256), 0, stream,
                                           part_dst, nb_dst, part_src, nb_src, HF, d_att_src, d_att_dst, d_bias);
    if (_pe != cudaSuccess) return hg::fail(W, hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

int hg_gat_scatter_norms(const int32_t* n_live_dev, long long n_live_max, const int32_t* live, const float* SG, int d,
                         float* d_in, double* norms, cudaStream_t stream) {
  { const cudaError_t _pe = hg::launch_pdl(k_gat_scatter_norms, dim3(grid_for(n_live_max * 32, 256, 148 * 16)), dim3(256), 0, stream, n_live_dev, live, SG, d, d_in,
                                                                                    norms); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_gat_scatter_norms");
  return kOk;
}

}  // extern "C"
