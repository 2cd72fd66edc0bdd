// K1 + K2: one layer of the layered fan-out sampler, bit-exact with
// histgnn/sampler.py:118-163 (see oracle/sampling.py for the restatement).
//
// Per layer (frontier F rows, device-side counts):
//   k_stamp     g2l[frontier[i]] = epoch<<32 | i ; src_out[i] = frontier[i]
//   scan        (deg, min(deg,fanout)) -> cand_off (PCG stream offsets), blk_off
//   k_task_bounds  split the layer's stream into warp tasks of ~C draws
//               (contiguous rows, balanced by candidates)
//   k_select    one warp per task: jump the PCG64 stream to the task's first
//               candidate (later rows: one multiply-add), draw one 53-bit key
//               per candidate in-edge, keep the `fanout` smallest (key,
//               position) pairs (warp bitonic network + ballot insertion) and
//               record the picked edge indices in key order
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
#ifndef HG_SEL_PAIRS
#define HG_SEL_PAIRS 1
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

struct KeyJ {
  unsigned long long k;
  unsigned j;
};

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

// Two short rows in one warp pass (lanes 0-15 row q, 16-31 row q+1; each
// row's lanes j < deg valid): every kSpan group sorted ascending by (key53, j),
// via the 32-bit prefix words with the same exact fallback on prefix ties.
__device__ __forceinline__ void sort_pair_fast(unsigned long long& key, long long span, long long dh) {
  const int lane = threadIdx.x & 31;
  unsigned v = ((unsigned)(key >> 37) << 5) | (unsigned)lane;
  if (span > 8) bitonic_sort_u32<16>(v);
  else if (span > 4) bitonic_sort_u32<8>(v);
  else if (span > 2) bitonic_sort_u32<4>(v);
  else bitonic_sort_u32<2>(v);
  const unsigned prev = __shfl_up_sync(0xffffffffu, v, 1);
  const int jl = lane & 15;
  const bool tie = jl > 0 && jl < dh && (prev >> 5) == (v >> 5);
  if (__any_sync(0xffffffffu, tie)) {
    if (span > 8) bitonic_sort_u64<16>(key);
    else if (span > 4) bitonic_sort_u64<8>(key);
    else if (span > 2) bitonic_sort_u64<4>(key);
    else bitonic_sort_u64<2>(key);
    return;
  }
  key = __shfl_sync(0xffffffffu, key, (int)(v & 31u));
}

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

// Warp tasks of k_select: contiguous frontier rows grouped by where their
// candidate stretch STARTS in the layer's PCG64 stream (tasks of C draws), so
// tasks are balanced by candidates, not rows (low ids = hubs cluster in the
// sorted-unique frontier). task_row[t] = first row whose stream offset is
// >= t*C (a lower bound on cand_off), task_row[T] = F; meta = {T, C}.
constexpr int kMaxTasks = 1 << 18;

// Hub rows (more than kHuge candidates, fanout <= 32) are split into
// segments of kSegC candidates, one warp each (k_select_huge: exact top-fanout
// of the segment by (key53, j)), then merged per row (k_merge_huge). The
// top-fanout of a row is contained in the union of its segments' top-fanout,
// so the result is exact; without the split one warp walks a 56K-candidate
// hub alone (papers100M shape) and sets the layer's duration.
constexpr long long kHuge = 4096;
constexpr int kSegC = 2048;
constexpr int kMaxSegs = 1 << 16;     // per layer; hubs beyond stay on the warp path
struct HugeState {
  int* ctr;             // [0] accepted hub rows, [1] segments claimed
  int32_t* rows;        // [F_max] accepted hub rows
  int32_t* base;        // [F_max] first segment of each accepted hub
  uint8_t* flag;        // [F_max] 1 = row handled by the hub path
  int32_t* seg_row;     // [kMaxSegs] row of each segment (-1 unused)
  int32_t* seg_s;       // [kMaxSegs] segment index within its row
  unsigned long long* seg_key;   // [kMaxSegs * 32] key53 of the segment's picks
  int32_t* seg_j;       // [kMaxSegs * 32] row-global candidate position
};

__global__ void k_task_bounds(const int32_t* F_dev, const int64_t* __restrict__ cand_off, int32_t* __restrict__ task_row,
                              long long* __restrict__ meta, int fanout, HugeState hs) {
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
    uint8_t huge = 0;
    if (fanout <= 32 && b - a > kHuge) {
      const int nseg = (int)((b - a + kSegC - 1) / kSegC);
      const int base = atomicAdd(&hs.ctr[1], nseg);
      if (base + nseg <= kMaxSegs) {
        huge = 1;
        const int i = atomicAdd(&hs.ctr[0], 1);
        hs.rows[i] = j;
        hs.base[i] = base;
        for (int q = 0; q < nseg; ++q) {
          hs.seg_row[base + q] = j;
          hs.seg_s[base + q] = q;
        }
      } else {
        for (int q = base; q < kMaxSegs && q < base + nseg; ++q) hs.seg_row[q] = -1;
      }
    }
    hs.flag[j] = huge;
  }
}


// One warp per task of kRowsPerTask consecutive frontier rows. Consecutive
// rows draw consecutive stretches of the PCG64 stream, so only a task's first
// row jumps from the batch state (O(log offset) table steps); each later row
// advances the lane states by the 1..32 draws left over from the previous row
// with a single precomputed multiply-add (tables D[d] = jump by d).
// k_select records each pick as its global edge index, split into the low
// (src_flat) and high (col_local) 32-bit words; k_pick resolves the column
// (a random read of the full graph's col) and marks non-frontier sources with
// full memory-level parallelism, off k_select's per-row critical path.
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

template <bool kSmallFanout>
__global__ void __launch_bounds__(kSelThreads, 4) k_select(
    const int64_t* __restrict__ g_start, const int64_t* __restrict__ g_end,
    const int32_t* __restrict__ frontier, const int32_t* F_dev, int fanout, const SampState* ss,
    const int64_t* __restrict__ cand_off, const int32_t* __restrict__ blk_off, int32_t* __restrict__ src_flat,
    int32_t* __restrict__ col_local, const int32_t* __restrict__ task_row, const long long* __restrict__ task_meta,
    const uint8_t* __restrict__ huge_flag) {
  pdl_wait();
  __shared__ JumpTableC tab;
  __shared__ u128 dA[33], dC[33];
  const u128 s0{ss->st_hi, ss->st_lo}, inc{ss->inc_hi, ss->inc_lo};
  for (int t = threadIdx.x; t < 256; t += blockDim.x) {
    (&tab.A[0][0])[t] = (&g_jump.A[0][0])[t];
    (&tab.C[0][0])[t] = mul128(inc, (&g_jump.S[0][0])[t]);
  }
  __syncthreads();
  if (threadIdx.x <= 32) {
    // jump by d = 16*h + l: low nibble first, then the high one
    const int d = threadIdx.x, l = d & 15, h = d >> 4;
    u128 a = tab.A[0][l], c = tab.C[0][l];
    if (h) {
      c = fma128(tab.A[1][h], c, tab.C[1][h]);
      a = mul128(tab.A[1][h], a);
    }
    dA[d] = a;
    dC[d] = c;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const unsigned long long base0 = ss->stream_pos;
  KTimer* kt = g_kt ? g_kt + kTSelect : nullptr;
  kt_begin(kt);
  const u128 a32 = tab.A[1][2];            // MULT^32 and its increment term
  const u128 c32 = tab.C[1][2];
  const long long ntask = task_meta[0];
  for (long long task = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; task < ntask; task += warps) {
    const int r_begin = task_row[task], r_end = task_row[task + 1];
    bool have = false;                     // cur = lane state at stream index cur_pos + lane
    u128 cur{0, 0};
    unsigned long long cur_pos = 0;
    for (int r0 = r_begin; r0 < r_end; r0 += 32) {
      const int nr = r_end - r0 < 32 ? r_end - r0 : 32;
      // the rows' metadata, fetched by lanes < nr at once
      long long lo_l = 0, deg_l = 0, off_l = 0;
      int out_l = 0;
      if (lane < nr) {
        const int v = frontier[r0 + lane];
        lo_l = g_start[v];
        deg_l = g_end[v] - lo_l;
        off_l = cand_off[r0 + lane];
        out_l = blk_off[r0 + lane];
        if (huge_flag && huge_flag[r0 + lane]) deg_l = 0;   // selected by k_select_huge / k_merge_huge
      }
      for (int q = 0; q < nr; ++q) {
        const long long lo = __shfl_sync(0xffffffffu, lo_l, q);
        const long long deg = __shfl_sync(0xffffffffu, deg_l, q);
        const int out0 = __shfl_sync(0xffffffffu, out_l, q);
        const int count = (int)(deg < fanout ? deg : fanout);
        if (deg == 0) continue;
        const unsigned long long k0 = base0 + (unsigned long long)__shfl_sync(0xffffffffu, off_l, q);
        // lane state: output index k0+lane needs k0+lane+1 steps
        u128 first;
        if (!have) {
          first = pcg_jump_c(tab, s0, k0 + (unsigned long long)lane + 1ull);
        } else {
          const unsigned long long delta = k0 - cur_pos;
          first = delta <= 32ull ? fma128(dA[delta], cur, dC[delta]) : pcg_jump_c(tab, cur, delta);
        }
        have = false;
#if HG_SEL_PAIRS
        // two short consecutive rows share one pass: their candidates are
        // consecutive in the stream, so row q+1's lanes take the states of
        // lanes deg .. deg+15 of this jump (the layouts of C3-like graphs,
        // m = 7, are dominated by rows of <= 16 candidates)
        if (kSmallFanout && deg <= 16 && q + 1 < nr) {
          const long long deg2 = __shfl_sync(0xffffffffu, deg_l, q + 1);
          if (deg2 >= 1 && deg2 <= 16) {
            const long long lo2 = __shfl_sync(0xffffffffu, lo_l, q + 1);
            const int out2 = __shfl_sync(0xffffffffu, out_l, q + 1);
            const int count2 = (int)(deg2 < fanout ? deg2 : fanout);
            const int srcl = lane < 16 ? lane : (int)deg + lane - 16;
            u128 st;
            st.hi = __shfl_sync(0xffffffffu, first.hi, srcl);
            st.lo = __shfl_sync(0xffffffffu, first.lo, srcl);
            const int jl = lane & 15;
            const long long dh = lane < 16 ? deg : deg2;
            unsigned long long key = jl < dh ? ((pcg_key53(st) << 11) | (unsigned long long)jl) : ~0ull;
            sort_pair_fast(key, deg > deg2 ? deg : deg2, dh);
            const int ch = lane < 16 ? count : count2;
            if (jl < ch)
              put_pick(src_flat, col_local, (lane < 16 ? out0 : out2) + jl, (lane < 16 ? lo : lo2) + (long long)(key & 2047ull));
            cur = first;
            cur_pos = k0;
            have = true;
            ++q;     // row q+1 done
            continue;
          }
        }
#endif
        if (kSmallFanout && deg <= 2048) {
          // fast path: (key53, j) packed into one u64, j < 2^11
          unsigned long long best = ~0ull;
          u128 s = first;
          for (long long c = 0; c < deg; c += 32) {
            const long long jj = c + lane;
            const bool valid = jj < deg;
            unsigned long long key = valid ? ((pcg_key53(s) << 11) | (unsigned long long)jj) : ~0ull;
            if (c + 32 < deg) s = fma128(a32, s, c32);
            if (c == 0) {
              sort_first_chunk_fast(key, deg);
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
          cur = s;
          cur_pos = k0 + 32ull * (unsigned long long)((deg - 1) / 32);
          have = true;
          if (lane < count) put_pick(src_flat, col_local, out0 + lane, lo + (long long)(best & 2047ull));
        } else if (kSmallFanout) {
          unsigned long long bk = ~0ull;
          unsigned bj = ~0u;
          u128 s = first;
          for (long long c = 0; c < deg; c += 32) {
            const long long jj = c + lane;
            const bool valid = jj < deg;
            unsigned long long key = valid ? pcg_key53(s) : ~0ull;
            unsigned j = valid ? (unsigned)jj : ~0u;
            if (c + 32 < deg) s = fma128(a32, s, c32);
            const unsigned long long tk = __shfl_sync(0xffffffffu, bk, fanout - 1);
            const unsigned tj = __shfl_sync(0xffffffffu, bj, fanout - 1);
            if (!__ballot_sync(0xffffffffu, valid && kj_less(key, j, tk, tj))) continue;
            bitonic_sort32(key, j);
            unsigned long long rk = __shfl_sync(0xffffffffu, key, 31 - lane);
            unsigned rj = __shfl_sync(0xffffffffu, j, 31 - lane);
            if (kj_less(rk, rj, bk, bj)) {
              bk = rk;
              bj = rj;
            }
            bitonic_merge32(bk, bj);
          }
          if (lane < count) put_pick(src_flat, col_local, out0 + lane, lo + bj);
        } else {
          // generic fanout: repeated warp-min selection (O(count * deg / 32))
          unsigned long long pk = 0;
          unsigned pj = 0;
          bool have_prev = false;
          for (int r = 0; r < count; ++r) {
            unsigned long long bk = ~0ull;
            unsigned bj = ~0u;
            u128 s = first;
            for (long long c = 0; c < deg; c += 32) {
              const long long jj = c + lane;
              if (jj < deg) {
                unsigned long long key = pcg_key53(s);
                unsigned j = (unsigned)jj;
                bool after = !have_prev || kj_less(pk, pj, key, j);
                if (after && kj_less(key, j, bk, bj)) {
                  bk = key;
                  bj = j;
                }
              }
              if (c + 32 < deg) s = fma128(a32, s, c32);
            }
    #pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
              unsigned oj = __shfl_xor_sync(0xffffffffu, bj, o);
              if (kj_less(ok, oj, bk, bj)) {
                bk = ok;
                bj = oj;
              }
            }
            pk = bk;
            pj = bj;
            have_prev = true;
            if (lane == 0) put_pick(src_flat, col_local, out0 + r, lo + pj);
          }
        }
      }
    }
  }
  kt_end(kt);
}

// one warp per hub segment: exact top-fanout (packed key53 << 11 | j_local)
// of kSegC consecutive candidates, written as (key53, row-global j)
__global__ void __launch_bounds__(kSelThreads, 4) k_select_huge(
    const int64_t* __restrict__ g_start, const int64_t* __restrict__ g_end, const int32_t* __restrict__ frontier,
    int fanout, const SampState* ss, const int64_t* __restrict__ cand_off, HugeState hs) {
  pdl_wait();
  __shared__ JumpTableC tab;
  const u128 s0{ss->st_hi, ss->st_lo}, inc{ss->inc_hi, ss->inc_lo};
  for (int t = threadIdx.x; t < 256; t += blockDim.x) {
    (&tab.A[0][0])[t] = (&g_jump.A[0][0])[t];
    (&tab.C[0][0])[t] = mul128(inc, (&g_jump.S[0][0])[t]);
  }
  __syncthreads();
  const int nseg = min(hs.ctr[1], kMaxSegs);
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const u128 a32 = tab.A[1][2];
  const u128 c32 = tab.C[1][2];
  for (int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < nseg; g += warps) {
    const int row = hs.seg_row[g];
    if (row < 0) continue;
    const int sidx = hs.seg_s[g];
    const int v = frontier[row];
    const long long deg = g_end[v] - g_start[v];
    const long long j0 = (long long)sidx * kSegC;
    const long long len = deg - j0 < kSegC ? deg - j0 : kSegC;
    const unsigned long long k0 = ss->stream_pos + (unsigned long long)cand_off[row] + (unsigned long long)j0;
    u128 s = pcg_jump_c(tab, s0, k0 + (unsigned long long)lane + 1ull);
    unsigned long long best = ~0ull;
    for (long long c = 0; c < len; c += 32) {
      const long long jj = c + lane;
      const bool valid = jj < len;
      unsigned long long key = valid ? ((pcg_key53(s) << 11) | (unsigned long long)jj) : ~0ull;
      if (c + 32 < len) s = fma128(a32, s, c32);
      if (c == 0) {
        sort_first_chunk_fast(key, len);
        best = key;
        continue;
      }
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
    const int cnt = (int)(len < fanout ? len : fanout);
    hs.seg_key[(long long)g * 32 + lane] = lane < cnt ? (best >> 11) : ~0ull;
    hs.seg_j[(long long)g * 32 + lane] = lane < cnt ? (int32_t)(j0 + (long long)(best & 2047ull)) : 0x7fffffff;
  }
}

// one warp per accepted hub row: top-fanout by (key53, j) over its segments'
// picks, emitted in key order like every other row
__global__ void __launch_bounds__(256) k_merge_huge(const int64_t* __restrict__ g_start,
                                                    const int32_t* __restrict__ frontier, int fanout,
                                                    const int64_t* __restrict__ cand_off,
                                                    const int32_t* __restrict__ blk_off, int32_t* __restrict__ src_flat,
                                                    int32_t* __restrict__ col_local, HugeState hs) {
  pdl_wait();
  const int nh = hs.ctr[0];
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nh; i += warps) {
    const int row = hs.rows[i];
    const int base = hs.base[i];
    const long long deg = cand_off[row + 1] - cand_off[row];
    const int nseg = (int)((deg + kSegC - 1) / kSegC);
    unsigned long long bk = ~0ull;
    unsigned bj = ~0u;
    for (int g = base; g < base + nseg; ++g) {
      unsigned long long key = hs.seg_key[(long long)g * 32 + lane];
      unsigned j = (unsigned)hs.seg_j[(long long)g * 32 + lane];
      if (lane >= fanout) {
        key = ~0ull;
        j = ~0u;
      }
      // a segment's picks are sorted: skip it when its best does not beat
      // the current fanout-th pick (nothing of it can enter the top-fanout)
      const unsigned long long k0 = __shfl_sync(0xffffffffu, key, 0);
      const unsigned j0 = __shfl_sync(0xffffffffu, j, 0);
      const unsigned long long tk = __shfl_sync(0xffffffffu, bk, fanout - 1);
      const unsigned tj = __shfl_sync(0xffffffffu, bj, fanout - 1);
      if (!kj_less(k0, j0, tk, tj)) continue;
      // (already ascending across lanes: k_select_huge stores its sorted picks)
      unsigned long long rk = __shfl_sync(0xffffffffu, key, 31 - lane);
      unsigned rj = __shfl_sync(0xffffffffu, j, 31 - lane);
      if (kj_less(rk, rj, bk, bj)) {
        bk = rk;
        bj = rj;
      }
      bitonic_merge32(bk, bj);
    }
    if (lane < fanout) put_pick(src_flat, col_local, blk_off[row] + lane, g_start[frontier[row]] + (long long)bj);
  }
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

static long long huge_scratch_bytes(long long F_max) {
  return 64 + (F_max + 16) * 9 + (long long)kMaxSegs * (4 + 4 + 32 * 8 + 32 * 4) + 256;
}

extern "C" {

long long hg_sample_layer_scratch_bytes(long long F_max, long long num_nodes) {
  long long words = (num_nodes + 31) / 32;
  return (scan_tiles(F_max) + 1) * (long long)sizeof(I64x2) + (scan_tiles(words, 1) + 1) * 4 + 256 +
         (long long)(kMaxTasks + 2) * 4 + 64 + huge_scratch_bytes(F_max);
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
  // hub-row state after the task table (16-byte aligned pieces)
  char* hp = reinterpret_cast<char*>(task_row + kMaxTasks + 2);
  hp = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(hp) + 15) & ~uintptr_t(15));
  HugeState hs;
  hs.ctr = reinterpret_cast<int*>(hp);
  hs.seg_key = reinterpret_cast<unsigned long long*>(hp + 64);
  hs.seg_j = reinterpret_cast<int32_t*>(hs.seg_key + (long long)kMaxSegs * 32);
  hs.seg_row = hs.seg_j + (long long)kMaxSegs * 32;
  hs.seg_s = hs.seg_row + kMaxSegs;
  hs.rows = hs.seg_s + kMaxSegs;
  hs.base = hs.rows + (F_max + 16);
  hs.flag = reinterpret_cast<uint8_t*>(hs.base + (F_max + 16));

  SampState* ss = reinterpret_cast<SampState*>(state_dev);
  { const cudaError_t _pe = hg::launch_pdl(k_stamp, dim3(grid_for(F_max, 256)), dim3(256), 0, stream, frontier, F_dev, ss, g2l, src_out); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  DegCount f{g_start, g_end, frontier, fanout};
  st = scan_launch<I64x2>(W, f, DevCount{F_dev}, F_max, part_dc,
                          EmitDegCount{cand_off, blk_off, blk_end, dst_deg, fanout, g_start, g_end, frontier},
                          TotalDegCount{F_dev, cand_off, blk_off, counts_dev}, stream);
  if (st) return st;
  HG_CHECK_CUDA(W, cudaMemsetAsync(hs.ctr, 0, 8, stream));
  { const cudaError_t _pe = hg::launch_pdl(k_task_bounds, dim3(grid_for(F_max, 256)), dim3(256), 0, stream, F_dev, cand_off, task_row, task_meta, fanout, hs); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED(W);
  // persistent warps over the tasks; HG_SEL_BLOCKS caps the grid (leaves SMs
  // to the training stream that runs concurrently with the pipelined sampler)
  // 4 CTAs (32 warps) per SM: the selection is latency-bound per row, so
  // more rows in flight help (C2: k_select 81 -> 59 ms / 200 steps; C3
  // step 1.29 -> 1.23 ms); 6/SM gains little more (profiles/r01/notes)
  static const long long sel_cap = [] {
    const char* e = std::getenv("HG_SEL_BLOCKS");
    const long long v = e ? std::atoll(e) : 148 * 4;
    return v < 1 ? 148ll * 4 : v;
  }();
  const unsigned sel_grid = (unsigned)sel_cap;
  if (fanout <= 32) {
    { const cudaError_t _pe = hg::launch_pdl(k_select<true>, dim3(sel_grid), dim3(kSelThreads), 0, stream, g_start, g_end, frontier, F_dev, fanout, ss, cand_off,
                                                          blk_off, src_flat, col_local, task_row, task_meta, hs.flag); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
    HG_LAUNCHED(W);
    { const cudaError_t _pe = hg::launch_pdl(k_select_huge, dim3(148 * 4), dim3(kSelThreads), 0, stream, g_start, g_end, frontier, fanout, ss, cand_off, hs); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
    HG_LAUNCHED(W);
    { const cudaError_t _pe = hg::launch_pdl(k_merge_huge, dim3(148), dim3(256), 0, stream, g_start, frontier, fanout, cand_off, blk_off, src_flat, col_local, hs); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
    HG_LAUNCHED(W);
  } else {
    { const cudaError_t _pe = hg::launch_pdl(k_select<false>, dim3(sel_grid), dim3(kSelThreads), 0, stream, g_start, g_end, frontier, F_dev, fanout, ss, cand_off,
                                                           blk_off, src_flat, col_local, task_row, task_meta, nullptr); if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
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
