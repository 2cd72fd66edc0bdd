// K1 + K2: one layer of the layered fan-out sampler, bit-exact with
// histgnn/sampler.py:118-163 (see oracle/sampling.py for the restatement).
//
// Per layer (frontier F rows, device-side counts):
//   k_stamp     g2l[frontier[i]] = epoch<<32 | i ; src_out[i] = frontier[i]
//   scan        (deg, min(deg,fanout)) -> cand_off (PCG stream offsets), blk_off
//   k_plan      per row: the PCG64 state before its first draw, hub rows
//               (> kHuge candidates) cut into segments, a histogram of the
//               other rows by candidate count                 (fanout <= 32)
//   k_order     rows by descending candidate count
//   k_select_all  one persistent launch over a longest-first work list: hub
//               segments, one row per warp, short rows one per thread; one
//               53-bit key per candidate in-edge, the `fanout` smallest
//               (key, position) pairs recorded in key order
//   (fanout > 32: k_task_bounds + k_select_generic, repeated warp minima)
//   k_pick      picked edge -> global source id; non-frontier sources are
//               marked in a node bitmap
//   bitmap scan sorted-unique "new" nodes fall out of the bitmap in id order:
//               popcount scan -> src_out[F + rank], g2l[new] = epoch<<32 | F+rank,
//               the bitmap is cleared as it is consumed
//   k_relabel   col_local[e] = low32(g2l[src_flat[e]])
// No O(N) memset per call: g2l entries are epoch-stamped, the bitmap is
// self-clearing.
#include "hgb200.h"
#include <cstdlib>
#include <mutex>
#include "hg_pcg.cuh"

#ifndef HG_SEL_PREFIX
#define HG_SEL_PREFIX 1
#endif
#include "hg_scan.cuh"

namespace hg {

__device__ JumpTable g_jump;

namespace {

__device__ KTimer* g_kt = nullptr;
}  // namespace
int set_timers_sampler(void* p) {
  cudaError_t e = cudaMemcpyToSymbol(g_kt, &p, sizeof(p));
  return e == cudaSuccess ? kOk : fail("set_timers_sampler", kCuda, cudaGetErrorString(e));
}
namespace {

__device__ __forceinline__ bool kj_less(unsigned long long ak, unsigned aj, unsigned long long bk, unsigned bj) {
  return ak < bk || (ak == bk && aj < bj);
}

__device__ __forceinline__ void cmpx(unsigned long long& k, unsigned& j, int partner_mask, bool keep_min) {
  unsigned long long pk = __shfl_xor_sync(0xffffffffu, k, partner_mask);
  unsigned pj = __shfl_xor_sync(0xffffffffu, j, partner_mask);
  bool p_less = kj_less(pk, pj, k, j);
  bool s_less = kj_less(k, j, pk, pj);
  if (keep_min ? p_less : s_less) {
    k = pk;
    j = pj;
  }
}

// ascending bitonic sort of 32 (key, j) pairs held one per lane
__device__ __forceinline__ void bitonic_sort32(unsigned long long& k, unsigned& j) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      bool ascending = (lane & size) == 0 || size == 32;
      bool lower = (lane & stride) == 0;
      cmpx(k, j, stride, lower == ascending);
    }
  }
}

// ascending bitonic merge of a bitonic sequence of 32
__device__ __forceinline__ void bitonic_merge32(unsigned long long& k, unsigned& j) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) cmpx(k, j, stride, (lane & stride) == 0);
}

struct DegCount {
  const int64_t* g_start;
  const int64_t* g_end;
  const int32_t* frontier;
  int fanout;
  __device__ I64x2 operator()(long long i) const {
    int v = frontier[i];
    long long d = g_end[v] - g_start[v];
    return {d, d < fanout ? d : (long long)fanout};
  }
};

struct EmitDegCount {
  int64_t* cand_off;
  int32_t* blk_off;
  int32_t* blk_end;
  int32_t* dst_deg;
  int fanout;
  const int64_t* g_start;
  const int64_t* g_end;
  const int32_t* frontier;
  __device__ void operator()(long long i, I64x2 excl, I64x2 v) const {
    cand_off[i] = excl.a;
    blk_off[i] = (int32_t)excl.b;
    blk_end[i] = (int32_t)(excl.b + v.b);
    dst_deg[i] = (int32_t)v.b;
  }
};

struct TotalDegCount {
  const int32_t* F_dev;
  int64_t* cand_off;
  int32_t* blk_off;
  int32_t* counts_dev;
  __device__ void operator()(I64x2 t) const {
    int F = *F_dev;
    cand_off[F] = t.a;
    blk_off[F] = (int32_t)t.b;
    counts_dev[0] = (int32_t)t.b;  // E
  }
};

// device-resident sampler state (u64[6]): PCG64 state hi/lo, inc hi/lo,
// draws consumed so far in this batch, epoch of the g2l stamps
struct SampState {
  unsigned long long st_hi, st_lo, inc_hi, inc_lo;
  unsigned long long stream_pos;
  unsigned long long epoch;
};

__global__ void k_stamp(const int32_t* __restrict__ frontier, const int32_t* F_dev, const SampState* ss,
                        int64_t* __restrict__ g2l, int32_t* __restrict__ src_out) {
  pdl_wait();
  const int F = *F_dev;
  const unsigned epoch = (unsigned)ss->epoch;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < F; i += gridDim.x * blockDim.x) {
    int v = frontier[i];
    g2l[v] = (int64_t)(((unsigned long long)epoch << 32) | (unsigned)i);
    src_out[i] = v;
  }
}

constexpr int kSelThreads = 256;

// packed (key53 << 11 | j) compare-exchange: one 64-bit order == (key, j) order
__device__ __forceinline__ void cmpx64(unsigned long long& k, int partner_mask, bool keep_min) {
  const unsigned long long p = __shfl_xor_sync(0xffffffffu, k, partner_mask);
  if (keep_min ? (p < k) : (k < p)) k = p;
}
// ascending bitonic sort of every group of kSpan lanes (kSpan = 2..32),
// fully unrolled: the compare directions are compile-time lane-bit tests
template <int kSpan>
__device__ __forceinline__ void bitonic_sort_u64(unsigned long long& k) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= kSpan; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const bool ascending = size == kSpan || (lane & size) == 0;
      cmpx64(k, stride, ((lane & stride) == 0) == ascending);
    }
  }
}
// sorting network sized to a row of deg candidates (lanes >= deg hold ~0 and stay last)
__device__ __forceinline__ void sort_first_chunk(unsigned long long& k, long long deg) {
  if (deg > 16) bitonic_sort_u64<32>(k);
  else if (deg > 8) bitonic_sort_u64<16>(k);
  else if (deg > 4) bitonic_sort_u64<8>(k);
  else if (deg > 2) bitonic_sort_u64<4>(k);
  else bitonic_sort_u64<2>(k);
}

// ascending bitonic sort of every group of kSpan lanes of 32-bit values
template <int kSpan>
__device__ __forceinline__ void bitonic_sort_u32(unsigned& v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= kSpan; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const bool ascending = size == kSpan || (lane & size) == 0;
      const unsigned p = __shfl_xor_sync(0xffffffffu, v, stride);
      const bool keep_min = ((lane & stride) == 0) == ascending;
      if (keep_min ? (p < v) : (v < p)) v = p;
    }
  }
}

// The first chunk of a row (lane j holds key53 << 11 | j, lanes >= deg ~0),
// sorted ascending. Sorts 32-bit (top 27 key bits, lane) words -- half the
// shuffles and compares of the 64-bit network -- then fetches each rank's
// full key from its lane. Two valid keys sharing their top 27 bits (about
// 1 row in 10^5) make the order ambiguous: then the exact 64-bit network
// runs instead, so the result is always the (key53, j) order.
#if HG_SEL_PREFIX
__device__ __forceinline__ void sort_first_chunk_fast(unsigned long long& key, long long deg) {
  const int lane = threadIdx.x & 31;
  unsigned v = ((unsigned)(key >> 37) << 5) | (unsigned)lane;
  if (deg > 16) bitonic_sort_u32<32>(v);
  else if (deg > 8) bitonic_sort_u32<16>(v);
  else if (deg > 4) bitonic_sort_u32<8>(v);
  else if (deg > 2) bitonic_sort_u32<4>(v);
  else bitonic_sort_u32<2>(v);
  const unsigned prev = __shfl_up_sync(0xffffffffu, v, 1);
  const bool tie = lane > 0 && lane < deg && (prev >> 5) == (v >> 5);
  if (__any_sync(0xffffffffu, tie)) {
    sort_first_chunk(key, deg);
    return;
  }
  key = __shfl_sync(0xffffffffu, key, (int)(v & 31u));
}
#else
__device__ __forceinline__ void sort_first_chunk_fast(unsigned long long& key, long long deg) {
  sort_first_chunk(key, deg);
}
#endif

// jump with the per-batch constants C = inc * S precomputed (one 128-bit
// multiply-add per non-zero nibble of the offset)
struct JumpTableC {
  u128 A[16][16];
  u128 C[16][16];
};
__device__ __forceinline__ u128 pcg_jump_c(const JumpTableC& tab, u128 s, unsigned long long k) {
  int w = 0;
  while (k) {
    const unsigned d = (unsigned)(k & 15ull);
    if (d) s = fma128(tab.A[w][d], s, tab.C[w][d]);
    k >>= 4;
    ++w;
  }
  return s;
}

// k_pick resolves each pick (global edge index, split into the low
// (src_flat) and high (col_local) 32-bit words) to its column -- a random read
// of the full graph's col -- and marks non-frontier sources, with full
// memory-level parallelism, off the selection's per-row critical path.
__device__ __forceinline__ void put_pick(int32_t* src_flat, int32_t* col_local, int e, long long pos) {
  src_flat[e] = (int32_t)(unsigned)(pos & 0xffffffffll);
  col_local[e] = (int32_t)(unsigned)((unsigned long long)pos >> 32);
}

__global__ void k_pick(const int32_t* __restrict__ g_col, const int32_t* counts_dev, const SampState* ss,
                       const int64_t* __restrict__ g2l, uint32_t* __restrict__ bitmap, int32_t* __restrict__ src_flat,
                       const int32_t* __restrict__ col_local) {
  pdl_wait();
  const int E = counts_dev[0];
  const unsigned epoch = (unsigned)ss->epoch;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const long long pos = (long long)(((unsigned long long)(unsigned)col_local[e] << 32) | (unsigned)src_flat[e]);
    const int u = g_col[pos];
    src_flat[e] = u;
    if ((unsigned)(g2l[u] >> 32) != epoch) atomicOr(&bitmap[u >> 5], 1u << (u & 31));
  }
}

// ------------------------------------------------------------------------
// Selection, fanout <= 32: one persistent launch over a work list.
//
// k_plan (thread per row): the PCG64 state just before the row's first draw
// (jump from the batch state, so no selector ever jumps far), hub rows
// (> kHuge candidates) split into segments of kSegC candidates, and a
// histogram of the other rows by candidate count. k_order lists those rows
// by descending count. k_select_all's warps then pull work items from one
// atomic counter, longest first:
//   hub segments   exact top-fanout of kSegC candidates (packed key53 << 11 |
//                  j); the warp finishing a row's last segment merges them
//   warp rows      rows of > lane_max candidates: lane = candidate, 32 keys
//                  per chunk, the first chunk sorted by a bitonic network, later
//                  ones inserted by ballot rank against the fanout-th key
//   lane groups    32 rows of <= lane_max candidates (fanout <= 16), one per
//                  THREAD: the row's keys drawn one after the other and the
//                  top-fanout kept sorted in registers by an unrolled
//                  compare-select network. The ordering groups rows of equal
//                  count, so the 32 loops of a warp have the same length.
// Every path keeps the (key53, j) order of the reference's argsort.
// ------------------------------------------------------------------------
// rows of more than kHuge candidates are split into segments of kSegC: a
// warp's item is then at most ~kHuge candidates long, which bounds the
// latency tail of the small layers (1024 seeds: a few long rows per layer)
#ifndef HG_SEL_HUGE
#define HG_SEL_HUGE 1024
#endif
#ifndef HG_SEL_SEG
#define HG_SEL_SEG 512
#endif
constexpr long long kHuge = HG_SEL_HUGE;
constexpr int kSegC = HG_SEL_SEG;
static_assert(kSegC <= 2048 && kSegC >= 32 && kHuge >= kSegC, "segments are packed with 11-bit positions");
constexpr int kMaxSegs = 1 << 16;     // per layer; hubs beyond are warp rows
constexpr int kBins = 320;            // candidate counts 0..255 exact, then 64 wide, last bin open
constexpr int kLaneCap = 255;         // lane_max <= kLaneCap

__device__ __forceinline__ int deg_bin(long long d) {
  if (d < 256) return (int)d;
  const long long b = 256 + ((d - 256) >> 6);
  return b > kBins - 1 ? kBins - 1 : (int)b;
}

struct Plan {
  int* ctr;            // [0] hub rows [1] segments claimed [2] item counter [3] items [4] warp rows [5] lane rows [6] segments
  int* hist;           // [kBins] rows per bin
  int* cursor;         // [kBins]
  int32_t* order;      // [F_max] non-hub rows, descending candidate count
  u128* row_state;     // [F_max] PCG64 state before the row's first draw
  int32_t* hub_row;    // [F_max]
  int32_t* hub_base;   // [F_max] first segment of the hub
  int* hub_done;       // [F_max] segments finished
  int32_t* seg_hub;    // [kMaxSegs] hub of the segment (-1: unused)
  unsigned long long* seg_key;  // [kMaxSegs * 32] key53 of the segment's picks
  int32_t* seg_j;      // [kMaxSegs * 32] row-global candidate position
  uint8_t* flag;       // [F_max] 1 = hub row
};

__global__ void __launch_bounds__(256) k_plan(const int32_t* F_dev, const int64_t* __restrict__ cand_off,
                                              const SampState* ss, Plan P) {
  pdl_wait();
  __shared__ int lh[kBins];
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) lh[b] = 0;
  __syncthreads();
  const int F = *F_dev;
  const u128 s0{ss->st_hi, ss->st_lo}, inc{ss->inc_hi, ss->inc_lo};
  const unsigned long long base0 = ss->stream_pos;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F; j += gridDim.x * blockDim.x) {
    const long long a = cand_off[j], d = cand_off[j + 1] - a;
    const u128 st = pcg_jump(g_jump, s0, inc, base0 + (unsigned long long)a);
    P.row_state[j] = st;
    uint8_t hub = 0;
    if (d > kHuge) {
      const int nseg = (int)((d + kSegC - 1) / kSegC);
      const int base = atomicAdd(&P.ctr[1], nseg);
      if (base + nseg <= kMaxSegs) {
        hub = 1;
        const int i = atomicAdd(&P.ctr[0], 1);
        P.hub_row[i] = j;
        P.hub_base[i] = base;
        P.hub_done[i] = 0;
        for (int q = 0; q < nseg; ++q) P.seg_hub[base + q] = i;
      } else {
        for (int q = base; q < kMaxSegs && q < base + nseg; ++q) P.seg_hub[q] = -1;
      }
    }
    P.flag[j] = hub;
    if (!hub && d >= 1) atomicAdd(&lh[deg_bin(d)], 1);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x)
    if (lh[b]) atomicAdd(&P.hist[b], lh[b]);
}

// non-hub rows -> P.order by descending bin (block scan of the histogram,
// per-CTA ranks by shared-memory atomics, one cursor reservation per CTA and
// bin); block 0 publishes the work-list sizes
__global__ void __launch_bounds__(kBins) k_order(const int32_t* F_dev, const int64_t* __restrict__ cand_off,
                                                 int lane_max, Plan P) {
  pdl_wait();
  __shared__ int off[kBins], cnt[kBins], res[kBins], wsum[kBins / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int bin = kBins - 1 - t;            // descending
  const int h = P.hist[bin];
  int x = h;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  int pre = 0;
  for (int q = 0; q < w; ++q) pre += wsum[q];
  off[bin] = pre + x - h;
  __syncthreads();
  if (blockIdx.x == 0 && t == 0) {
    int total = 0;
    for (int q = 0; q < kBins / 32; ++q) total += wsum[q];
    const int n_warp = lane_max > 0 ? off[lane_max] : total;   // bins above lane_max come first
    const int n_lane = total - n_warp;
    const int nseg = P.ctr[1] < kMaxSegs ? P.ctr[1] : kMaxSegs;
    P.ctr[4] = n_warp;
    P.ctr[5] = n_lane;
    P.ctr[6] = nseg;
    P.ctr[3] = nseg + n_warp + (n_lane + 31) / 32;
  }
  const int F = *F_dev;
  for (int base = blockIdx.x * kBins; base < F; base += gridDim.x * kBins) {
    cnt[t] = 0;
    __syncthreads();
    const int j = base + t;
    int b = -1, r = 0;
    if (j < F && !P.flag[j]) {
      const long long d = cand_off[j + 1] - cand_off[j];
      if (d >= 1) {
        b = deg_bin(d);
        r = atomicAdd(&cnt[b], 1);
      }
    }
    __syncthreads();
    if (cnt[t]) res[t] = atomicAdd(&P.cursor[t], cnt[t]);
    __syncthreads();
    if (b >= 0) P.order[off[b] + res[b] + r] = j;
    __syncthreads();
  }
}

// sorted insertion of key into b[0..kF) (ascending), no data-dependent
// indexing, so the list stays in registers
template <int kF>
__device__ __forceinline__ void lane_insert(unsigned long long (&b)[kF], unsigned long long key) {
  bool c[kF];
#pragma unroll
  for (int i = 0; i < kF; ++i) c[i] = key < b[i];
#pragma unroll
  for (int i = kF - 1; i > 0; --i) b[i] = c[i - 1] ? b[i - 1] : (c[i] ? key : b[i]);
  b[0] = c[0] ? key : b[0];
}

// top-fanout of `len` (<= 2048) consecutive candidates starting at lane state
// s (lane l at candidate l): packed (key53 << 11 | j) words, ascending, one
// per lane (lanes >= min(len, fanout) hold larger keys or ~0)
__device__ __forceinline__ unsigned long long warp_topk_packed(u128 s, long long len, int fanout, u128 a32, u128 c32) {
  const int lane = threadIdx.x & 31;
  unsigned long long best = ~0ull;
  for (long long c = 0; c < len; c += 32) {
    const long long jj = c + lane;
    unsigned long long key = jj < len ? ((pcg_key53(s) << 11) | (unsigned long long)jj) : ~0ull;
    if (c + 32 < len) s = fma128(a32, s, c32);
    if (c == 0) {
      sort_first_chunk_fast(key, len);
      best = key;
      continue;
    }
    // later chunks: insert only the candidates that beat the current
    // fanout-th key, one at a time (rank by ballot, shift by shfl_up)
    unsigned long long thr = __shfl_sync(0xffffffffu, best, fanout - 1);
    unsigned m = __ballot_sync(0xffffffffu, key < thr);
    while (m) {
      const int l = __ffs(m) - 1;
      const unsigned long long cand = __shfl_sync(0xffffffffu, key, l);
      const int pos = __popc(__ballot_sync(0xffffffffu, best < cand));
      const unsigned long long up = __shfl_up_sync(0xffffffffu, best, 1);
      if (lane == pos) best = cand;
      else if (lane > pos) best = up;
      thr = __shfl_sync(0xffffffffu, best, fanout - 1);
      m &= ~(1u << l);
      m &= __ballot_sync(0xffffffffu, key < thr);
    }
  }
  return best;
}

template <int kF>
__global__ void __launch_bounds__(kSelThreads, 4) k_select_all(
    const int64_t* __restrict__ g_start, const int32_t* __restrict__ frontier, int fanout, const SampState* ss,
    const int64_t* __restrict__ cand_off, const int32_t* __restrict__ blk_off, int32_t* __restrict__ src_flat,
    int32_t* __restrict__ col_local, Plan P) {
  pdl_wait();
  __shared__ u128 dA[33], dC[33];          // jump by d = 0..32 steps
  const u128 inc{ss->inc_hi, ss->inc_lo};
  if (threadIdx.x <= 32) {
    const int d = threadIdx.x, l = d & 15, h = d >> 4;
    u128 a = g_jump.A[0][l], c = mul128(inc, g_jump.S[0][l]);
    if (h) {
      const u128 ah = g_jump.A[1][h];
      c = fma128(ah, c, mul128(inc, g_jump.S[1][h]));
      a = mul128(ah, a);
    }
    dA[d] = a;
    dC[d] = c;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int n_items = P.ctr[3], nseg = P.ctr[6], n_warp = P.ctr[4], n_lane = P.ctr[5];
  const u128 a32 = dA[32], c32 = dC[32], a1 = dA[lane + 1], c1 = dC[lane + 1];
  const u128 mult{kMultHi, kMultLo};
  KTimer* kt = g_kt ? g_kt + kTSelect : nullptr;
  kt_begin(kt);
  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(&P.ctr[2], 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    if (item < nseg) {
      // ---- hub segment
      const int i = P.seg_hub[item];
      if (i < 0) continue;
      const int row = P.hub_row[i];
      const long long a = cand_off[row], deg = cand_off[row + 1] - a;
      const int sidx = item - P.hub_base[i];
      const long long j0 = (long long)sidx * kSegC;
      const long long len = deg - j0 < kSegC ? deg - j0 : kSegC;
      // the segment's start state: a short jump from the row's
      const u128 sst = pcg_jump(g_jump, P.row_state[row], inc, (unsigned long long)j0);
      const unsigned long long best = warp_topk_packed(fma128(a1, sst, c1), len, fanout, a32, c32);
      const int cnt = (int)(len < fanout ? len : fanout);
      P.seg_key[(long long)item * 32 + lane] = lane < cnt ? (best >> 11) : ~0ull;
      P.seg_j[(long long)item * 32 + lane] = lane < cnt ? (int32_t)(j0 + (long long)(best & 2047ull)) : 0x7fffffff;
      __syncwarp();
      const int nsr = (int)((deg + kSegC - 1) / kSegC);
      int last = 0;
      if (lane == 0) {
        __threadfence();
        last = atomicAdd(&P.hub_done[i], 1) == nsr - 1;
      }
      if (!__shfl_sync(0xffffffffu, last, 0)) continue;
      __threadfence();
      // the row's last segment: merge the segments' sorted picks
      const int sb = P.hub_base[i];
      unsigned long long bk = ~0ull;
      unsigned bj = ~0u;
      for (int g = sb; g < sb + nsr; ++g) {
        unsigned long long key = __ldcg(&P.seg_key[(long long)g * 32 + lane]);
        unsigned j = (unsigned)__ldcg(&P.seg_j[(long long)g * 32 + lane]);
        if (lane >= fanout) {
          key = ~0ull;
          j = ~0u;
        }
        const unsigned long long k0 = __shfl_sync(0xffffffffu, key, 0);
        const unsigned j0s = __shfl_sync(0xffffffffu, j, 0);
        const unsigned long long tk = __shfl_sync(0xffffffffu, bk, fanout - 1);
        const unsigned tj = __shfl_sync(0xffffffffu, bj, fanout - 1);
        if (!kj_less(k0, j0s, tk, tj)) continue;        // nothing of it enters the top-fanout
        const unsigned long long rk = __shfl_sync(0xffffffffu, key, 31 - lane);
        const unsigned rj = __shfl_sync(0xffffffffu, j, 31 - lane);
        if (kj_less(rk, rj, bk, bj)) {
          bk = rk;
          bj = rj;
        }
        bitonic_merge32(bk, bj);
      }
      if (lane < fanout) put_pick(src_flat, col_local, blk_off[row] + lane, g_start[frontier[row]] + (long long)bj);
    } else if (item < nseg + n_warp) {
      // ---- one row per warp
      const int j = P.order[item - nseg];
      const long long a = cand_off[j], deg = cand_off[j + 1] - a;
      const long long lo = g_start[frontier[j]];
      const int out0 = blk_off[j];
      const int count = (int)(deg < fanout ? deg : fanout);
      u128 s = fma128(a1, P.row_state[j], c1);
      if (deg <= 2048) {
        const unsigned long long best = warp_topk_packed(s, deg, fanout, a32, c32);
        if (lane < count) put_pick(src_flat, col_local, out0 + lane, lo + (long long)(best & 2047ull));
      } else {
        // (key53, j) pairs: rows too long for the 11-bit packing
        unsigned long long bk = ~0ull;
        unsigned bj = ~0u;
        for (long long c = 0; c < deg; c += 32) {
          const long long jj = c + lane;
          const bool valid = jj < deg;
          unsigned long long key = valid ? pcg_key53(s) : ~0ull;
          unsigned jv = valid ? (unsigned)jj : ~0u;
          if (c + 32 < deg) s = fma128(a32, s, c32);
          const unsigned long long tk = __shfl_sync(0xffffffffu, bk, fanout - 1);
          const unsigned tj = __shfl_sync(0xffffffffu, bj, fanout - 1);
          if (!__ballot_sync(0xffffffffu, valid && kj_less(key, jv, tk, tj))) continue;
          bitonic_sort32(key, jv);
          const unsigned long long rk = __shfl_sync(0xffffffffu, key, 31 - lane);
          const unsigned rj = __shfl_sync(0xffffffffu, jv, 31 - lane);
          if (kj_less(rk, rj, bk, bj)) {
            bk = rk;
            bj = rj;
          }
          bitonic_merge32(bk, bj);
        }
        if (lane < count) put_pick(src_flat, col_local, out0 + lane, lo + bj);
      }
    } else if (kF > 0) {
      // ---- one row per thread
      const int idx = n_warp + (item - nseg - n_warp) * 32 + lane;
      if (idx >= n_warp + n_lane) continue;
      const int j = P.order[idx];
      const long long a = cand_off[j];
      const int deg = (int)(cand_off[j + 1] - a);
      const long long lo = g_start[frontier[j]];
      const int out0 = blk_off[j];
      constexpr int kK = kF > 0 ? kF : 1;
      unsigned long long b[kK];
#pragma unroll
      for (int q = 0; q < kK; ++q) b[q] = ~0ull;
      u128 s = fma128(mult, P.row_state[j], inc);   // one step: draw 0
      for (int c = 0; c < deg; ++c) {
        const unsigned long long key = (pcg_key53(s) << 11) | (unsigned long long)c;
        s = fma128(mult, s, inc);
        if (key < b[kK - 1]) lane_insert<kK>(b, key);
      }
      const int count = deg < fanout ? deg : fanout;
#pragma unroll
      for (int q = 0; q < kK; ++q)
        if (q < count) put_pick(src_flat, col_local, out0 + q, lo + (long long)(b[q] & 2047ull));
    }
  }
  kt_end(kt);
}

// ------------------------------------------------------------------------
// fanout > 32: warp tasks of contiguous rows (balanced by candidates: task
// t starts at the first row whose stream offset is >= t*C) and repeated
// warp-min selection, O(count * deg / 32) per row.
constexpr int kMaxTasks = 1 << 18;

__global__ void k_task_bounds(const int32_t* F_dev, const int64_t* __restrict__ cand_off, int32_t* __restrict__ task_row,
                              long long* __restrict__ meta) {
  pdl_wait();
  const int F = *F_dev;
  const long long total = cand_off[F];
  long long C = (total + 148 * 32 - 1) / (148 * 32);       // aim for >= 32 tasks per SM
  C = C < 64 ? 64 : (C > 512 ? 512 : C);
  const long long cmin = (total + kMaxTasks - 1) / kMaxTasks;
  if (C < cmin) C = cmin;
  const long long T = (total + C - 1) / C;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    meta[0] = T;
    meta[1] = C;
    task_row[0] = 0;
    task_row[T] = F;
  }
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < F; j += gridDim.x * blockDim.x) {
    const long long a = cand_off[j], b = cand_off[j + 1];
    for (long long t = a / C + 1; t * C <= b && t < T; ++t) task_row[t] = j + 1;
  }
}

__global__ void __launch_bounds__(kSelThreads, 4) k_select_generic(
    const int64_t* __restrict__ g_start, const int64_t* __restrict__ g_end,
    const int32_t* __restrict__ frontier, int fanout, const SampState* ss,
    const int64_t* __restrict__ cand_off, const int32_t* __restrict__ blk_off, int32_t* __restrict__ src_flat,
    int32_t* __restrict__ col_local, const int32_t* __restrict__ task_row, const long long* __restrict__ task_meta) {
  pdl_wait();
  __shared__ JumpTableC tab;
  const u128 s0{ss->st_hi, ss->st_lo}, inc{ss->inc_hi, ss->inc_lo};
  for (int t = threadIdx.x; t < 256; t += blockDim.x) {
    (&tab.A[0][0])[t] = (&g_jump.A[0][0])[t];
    (&tab.C[0][0])[t] = mul128(inc, (&g_jump.S[0][0])[t]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const unsigned long long base0 = ss->stream_pos;
  const u128 a32 = tab.A[1][2];            // MULT^32 and its increment term
  const u128 c32 = tab.C[1][2];
  KTimer* kt = g_kt ? g_kt + kTSelect : nullptr;
  kt_begin(kt);
  const long long ntask = task_meta[0];
  for (long long task = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; task < ntask; task += warps) {
    for (int r = task_row[task]; r < task_row[task + 1]; ++r) {
      const int v = frontier[r];
      const long long lo = g_start[v], deg = g_end[v] - lo;
      if (deg == 0) continue;
      const int out0 = blk_off[r];
      const int count = (int)(deg < fanout ? deg : fanout);
      // lane state: stream index k0 + lane needs k0 + lane + 1 steps
      const u128 first = pcg_jump_c(tab, s0, base0 + (unsigned long long)cand_off[r] + (unsigned long long)lane + 1ull);
      unsigned long long pk = 0;
      unsigned pj = 0;
      bool have_prev = false;
      for (int q = 0; q < count; ++q) {
        unsigned long long bk = ~0ull;
        unsigned bj = ~0u;
        u128 s = first;
        for (long long c = 0; c < deg; c += 32) {
          const long long jj = c + lane;
          if (jj < deg) {
            const unsigned long long key = pcg_key53(s);
            const unsigned j = (unsigned)jj;
            const bool after = !have_prev || kj_less(pk, pj, key, j);
            if (after && kj_less(key, j, bk, bj)) {
              bk = key;
              bj = j;
            }
          }
          if (c + 32 < deg) s = fma128(a32, s, c32);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
          const unsigned oj = __shfl_xor_sync(0xffffffffu, bj, o);
          if (kj_less(ok, oj, bk, bj)) {
            bk = ok;
            bj = oj;
          }
        }
        pk = bk;
        pj = bj;
        have_prev = true;
        if (lane == 0) put_pick(src_flat, col_local, out0 + q, lo + pj);
      }
    }
  }
  kt_end(kt);
}

struct PopWord {
  const uint32_t* bitmap;
  __device__ int operator()(long long i) const { return __popc(bitmap[i]); }
};

struct EmitNew {
  uint32_t* bitmap;
  const int32_t* F_dev;
  const SampState* ss;
  int64_t* g2l;
  int32_t* src_out;
  __device__ void operator()(long long w, int excl, int v) const {
    if (!v) return;
    uint32_t bits = bitmap[w];
    const int pos0 = *F_dev + excl;
    const unsigned epoch = (unsigned)ss->epoch;
    int r = 0;
    while (bits) {
      int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int id = (int)(w * 32 + b);
      const int pos = pos0 + r++;
      src_out[pos] = id;
      g2l[id] = (int64_t)(((unsigned long long)epoch << 32) | (unsigned)pos);
    }
    bitmap[w] = 0u;
  }
};

struct TotalNew {
  const int32_t* F_dev;
  int32_t* counts_dev;
  SampState* ss;
  const int64_t* cand_off;
  __device__ void operator()(int t) const {
    const int F = *F_dev;
    counts_dev[1] = F + t;  // n_src of this block = next frontier size
    ss->stream_pos += (unsigned long long)cand_off[F];
  }
};

__global__ void k_relabel(const int32_t* __restrict__ src_flat, const int32_t* counts_dev,
                          const int64_t* __restrict__ g2l, int32_t* __restrict__ col_local, SampState* ss) {
  pdl_wait();
  const int E = counts_dev[0];
  // every reader of this layer's epoch has finished (stream order): advance it
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long e = ss->epoch + 1;
    ss->epoch = (e >= 0xFFFFFFFEull) ? 1ull : e;   // never the 0xFFFFFFFF fill of g2l
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x)
    col_local[e] = (int32_t)(g2l[src_flat[e]] & 0xffffffffll);
}

}  // namespace

int ensure_jump_table() {
  // once per device (the __constant__ table is per-device module state);
  // a mutex-guarded device mask keeps concurrent callers thread-safe
  static std::mutex mu;
  static unsigned long long done_mask = 0;
  int dev = 0;
  HG_CHECK_CUDA("jump_table", cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (done_mask >> (dev & 63) & 1ull) return kOk;
  JumpTable* h = new JumpTable;
  const unsigned __int128 mult = ((unsigned __int128)kMultHi << 64) | kMultLo;
  unsigned __int128 base = mult;  // MULT^(16^w)
  unsigned __int128 base_s = 1;   // S for m = 16^w
  for (int w = 0; w < 16; ++w) {
    unsigned __int128 a = 1, s = 0;  // map for m = d*16^w, accumulated
    for (int d = 0; d < 16; ++d) {
      h->A[w][d] = {(unsigned long long)(a >> 64), (unsigned long long)a};
      h->S[w][d] = {(unsigned long long)(s >> 64), (unsigned long long)s};
      // compose one more base step: x -> base*x + base_s  (after current map)
      s = base * s + base_s;
      a = base * a;
    }
    // next window base: apply base 16 times
    unsigned __int128 na = 1, ns = 0;
    for (int d = 0; d < 16; ++d) {
      ns = base * ns + base_s;
      na = base * na;
    }
    base = na;
    base_s = ns;
  }
  cudaError_t e = cudaMemcpyToSymbol(g_jump, h, sizeof(JumpTable));
  delete h;
  if (e != cudaSuccess) return fail("jump_table", kCuda, cudaGetErrorString(e));
  done_mask |= 1ull << (dev & 63);
  return kOk;
}

}  // namespace hg

using namespace hg;

static long long a16(long long x) { return (x + 15) & ~15ll; }
static long long plan_scratch_bytes(long long F_max) {
  const long long F = F_max + 16;
  return a16((16 + 2 * kBins) * 4) + a16(F * 4) + a16(F * 16) + 3 * a16(F * 4) + a16((long long)kMaxSegs * 4) +
         a16((long long)kMaxSegs * 32 * 8) + a16((long long)kMaxSegs * 32 * 4) +
         a16(F) + 64;
}

static Plan carve_plan(char* p, long long F_max) {
  const long long F = F_max + 16;
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  Plan P;
  auto take = [&](long long bytes) {
    char* q = p;
    p += a16(bytes);
    return q;
  };
  P.ctr = reinterpret_cast<int*>(take((16 + 2 * kBins) * 4));   // ctr, hist, cursor: one memset
  P.hist = P.ctr + 16;
  P.cursor = P.hist + kBins;
  P.order = reinterpret_cast<int32_t*>(take(F * 4));
  P.row_state = reinterpret_cast<u128*>(take(F * 16));
  P.hub_row = reinterpret_cast<int32_t*>(take(F * 4));
  P.hub_base = reinterpret_cast<int32_t*>(take(F * 4));
  P.hub_done = reinterpret_cast<int*>(take(F * 4));
  P.seg_hub = reinterpret_cast<int32_t*>(take((long long)kMaxSegs * 4));
  P.seg_key = reinterpret_cast<unsigned long long*>(take((long long)kMaxSegs * 32 * 8));
  P.seg_j = reinterpret_cast<int32_t*>(take((long long)kMaxSegs * 32 * 4));
  P.flag = reinterpret_cast<uint8_t*>(take(F));
  return P;
}

// HG_SEL_LANE_MAX: longest row (candidates) selected one row per thread
// (fanout <= 16); 0 = one row per warp throughout (A/B)
static int lane_max_env() {
  static const int v = [] {
    const char* e = std::getenv("HG_SEL_LANE_MAX");
    const int x = e ? std::atoi(e) : 64;
    return x < 0 ? 0 : (x > kLaneCap ? kLaneCap : x);
  }();
  return v;
}

extern "C" {

long long hg_sample_layer_scratch_bytes(long long F_max, long long num_nodes) {
  long long words = (num_nodes + 31) / 32;
  return (scan_tiles(F_max) + 1) * (long long)sizeof(I64x2) + (scan_tiles(words, 1) + 1) * 4 + 256 +
         (long long)(kMaxTasks + 2) * 4 + 64 + plan_scratch_bytes(F_max);
}

int hg_sample_layer(const int64_t* g_start, const int64_t* g_end, const int32_t* g_col, long long num_nodes,
                    const int32_t* frontier, const int32_t* F_dev, long long F_max, int fanout,
                    unsigned long long* state_dev, int64_t* g2l,
                    uint32_t* bitmap, int64_t* cand_off, int32_t* blk_off, int32_t* blk_end, int32_t* dst_deg, int32_t* src_flat,
                    int32_t* col_local, int32_t* src_out, int32_t* counts_dev, void* scratch,
                    long long scratch_bytes, cudaStream_t stream) {
  const char* W = "hg_sample_layer";
  if (fanout < 1 || F_max < 1 || num_nodes < 1) return fail(W, kBadArg, "fanout, F_max and num_nodes must be >= 1");
  if (scratch_bytes < hg_sample_layer_scratch_bytes(F_max, num_nodes)) return fail(W, kBadArg, "scratch too small");
  int st = ensure_jump_table();
  if (st) return st;
  const long long words = (num_nodes + 31) / 32;
  I64x2* part_dc = reinterpret_cast<I64x2*>(scratch);
  int* part_w = reinterpret_cast<int*>(reinterpret_cast<char*>(scratch) + (scan_tiles(F_max) + 1) * sizeof(I64x2));
  long long* task_meta = reinterpret_cast<long long*>(part_w + scan_tiles(words, 1) + 2);
  task_meta = reinterpret_cast<long long*>((reinterpret_cast<uintptr_t>(task_meta) + 15) & ~uintptr_t(15));
  int32_t* task_row = reinterpret_cast<int32_t*>(task_meta + 2);
  Plan P = carve_plan(reinterpret_cast<char*>(task_row + kMaxTasks + 2), F_max);

  SampState* ss = reinterpret_cast<SampState*>(state_dev);
  { const cudaError_t _pe = hg::launch_pdl(k_stamp, dim3(grid_for(F_max, 256)), dim3(256), 0, stream, frontier, F_dev, ss, g2l, src_out); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  DegCount f{g_start, g_end, frontier, fanout};
  st = scan_launch<I64x2>(W, f, DevCount{F_dev}, F_max, part_dc,
                          EmitDegCount{cand_off, blk_off, blk_end, dst_deg, fanout, g_start, g_end, frontier},
                          TotalDegCount{F_dev, cand_off, blk_off, counts_dev}, stream);
  if (st) return st;
  cudaError_t e;
  if (fanout <= 32) {
    const int lane_max = fanout <= 16 ? lane_max_env() : 0;
    HG_CHECK_CUDA(W, cudaMemsetAsync(P.ctr, 0, (16 + 2 * kBins) * 4, stream));
    e = hg::launch_pdl(k_plan, dim3(grid_for(F_max, 256)), dim3(256), 0, stream, F_dev, (const int64_t*)cand_off,
                       (const SampState*)ss, P);
    if (e != cudaSuccess) return fail("launch", kCuda, cudaGetErrorString(e));
    HG_LAUNCHED(W);
    e = hg::launch_pdl(k_order, dim3(grid_for(F_max, kBins, 148u * 4u)), dim3(kBins), 0, stream, F_dev,
                       (const int64_t*)cand_off, lane_max, P);
    if (e != cudaSuccess) return fail("launch", kCuda, cudaGetErrorString(e));
    HG_LAUNCHED(W);
    // persistent: 3 CTAs (24 warps) per SM pulling work items -- the
    // selection's CTAs hold their slots until the queue drains, and the
    // forward runs beside them (C2: 444 CTAs 1.533 / 1.540e6 seeds/s vs
    // 592: 1.521e6, 296: 1.531e6, 148: 1.458e6); HG_SEL_BLOCKS overrides
    // (C3, 111M nodes: 2 CTAs per SM measured better -- 1.324-1.326e6 vs
    // 1.299-1.307e6 seeds/s -- the selection's random candidate reads over
    // a multi-GB graph contend less with the training kernels; C2 keeps 3:
    // 1.609-1.612e6 vs 1.586e6 with 2)
    static const long long sel_env = [] {
      const char* v = std::getenv("HG_SEL_BLOCKS");
      const long long x = v ? std::atoll(v) : 0;
      return x < 1 ? 0ll : x;
    }();
    const long long sel_cap = sel_env ? sel_env : (num_nodes >= (32ll << 20) ? 148 * 2 : 148 * 3);
    const int fk = lane_max == 0 ? 0 : fanout <= 2 ? 2 : fanout <= 4 ? 4 : fanout <= 5 ? 5 : fanout <= 6 ? 6
                 : fanout <= 8 ? 8 : fanout <= 10 ? 10 : fanout <= 12 ? 12 : fanout <= 15 ? 15 : 16;
#define HG_SEL_CASE(K)                                                                                          \
  case K:                                                                                                       \
    e = hg::launch_pdl(k_select_all<K>, dim3((unsigned)sel_cap), dim3(kSelThreads), 0, stream, g_start, frontier, \
                       fanout, (const SampState*)ss, (const int64_t*)cand_off, (const int32_t*)blk_off, src_flat, \
                       col_local, P);                                                                           \
    break;
    switch (fk) {
      HG_SEL_CASE(0) HG_SEL_CASE(2) HG_SEL_CASE(4) HG_SEL_CASE(5) HG_SEL_CASE(6) HG_SEL_CASE(8) HG_SEL_CASE(10)
      HG_SEL_CASE(12) HG_SEL_CASE(15) HG_SEL_CASE(16)
    }
#undef HG_SEL_CASE
    if (e != cudaSuccess) return fail("launch", kCuda, cudaGetErrorString(e));
    HG_LAUNCHED(W);
  } else {
    e = hg::launch_pdl(k_task_bounds, dim3(grid_for(F_max, 256)), dim3(256), 0, stream, F_dev,
                       (const int64_t*)cand_off, task_row, task_meta);
    if (e != cudaSuccess) return fail("launch", kCuda, cudaGetErrorString(e));
    HG_LAUNCHED(W);
    e = hg::launch_pdl(k_select_generic, dim3(148 * 4), dim3(kSelThreads), 0, stream, g_start, g_end, frontier,
                       fanout, (const SampState*)ss, (const int64_t*)cand_off, (const int32_t*)blk_off, src_flat,
                       col_local, (const int32_t*)task_row, (const long long*)task_meta);
    if (e != cudaSuccess) return fail("launch", kCuda, cudaGetErrorString(e));
    HG_LAUNCHED(W);
  }
  { const cudaError_t _pe = hg::launch_pdl(k_pick, dim3(grid_for(F_max * (long long)fanout, 256)), dim3(256), 0, stream, g_col, counts_dev, ss, g2l, bitmap, src_flat,
                                                                       col_local); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  // one bitmap word per thread: a dense word emits up to 32 ids serially,
  // so short threads and many CTAs (words / 256) keep the emission parallel
  st = scan_launch<int, 1>(W, PopWord{bitmap}, ConstCount{words}, words, part_w,
                        EmitNew{bitmap, F_dev, ss, g2l, src_out},
                        TotalNew{F_dev, counts_dev, ss, cand_off}, stream);
  if (st) return st;
  { const cudaError_t _pe = hg::launch_pdl(k_relabel, dim3(grid_for(F_max * (long long)fanout, 256)), dim3(256), 0, stream, src_flat, counts_dev, g2l, col_local, ss); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  return kOk;
}

}  // extern "C"
