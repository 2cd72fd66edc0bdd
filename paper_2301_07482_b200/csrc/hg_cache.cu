// K10: historical-cache admission / eviction / ring scatter-update for one
// layer, bit-exact with histgnn/cache.py:131-204 (oracle: oracle/histcache.py).
//
//   U1  keys (norm fp64 bits, node id) for the live nodes; a device bucket
//       sort ranks them "norm ascending, ties by id" (cache.py:191); ids are
//       unique, so the order is total and independent of the algorithm
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
#include <cub/device/device_radix_sort.cuh>   // setup only: the feature-region degree sort
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

// ---------------------------------------------------------------------------
// Bucket sort of the (norm bits, id) keys. fp64 norms are >= 0, so their bit
// patterns order like the values. The occupied bit range [lo, hi] is cut into
// kNB buckets by (bits - lo) >> shift (monotone; equal norms share a bucket).
// Keys are distinct (ids are), so the result is the unique sorted order.
//   k_norm_keys   keys + the min / max norm bits (block-reduced)
//   k_bs_count    bucket of every key and its arrival rank in the bucket
//   k_bs_offsets  one CTA per super-bucket of 256: in-super offsets, the
//                 super total; the last CTA to finish scans the super totals
//                 (offset of bucket b = loc[b] + spre[b / 256])
//   k_bs_place    keys to their bucket slots (offset + arrival rank)
//   k_bs_rank     one thread per key of a bucket of <= kShortMax keys: its
//                 final position = bucket offset + the number of the bucket's
//                 keys below it (exact because keys are distinct); then one
//                 CTA per longer bucket: bitonic sort in shared memory up to
//                 kBucketCap keys, chunk sorts + merge passes above
// The writers of the sorted positions also apply U2 (admission / gradient
// eviction flags) when an Admit is given, so no separate pass reads the
// sorted keys back. 64K buckets: the C2 layer-1 norms (~130K over 2.4
// decades) leave buckets of median 2 / 99th percentile ~65 keys
// (tools/norm_dist.py); at 16K buckets 77 % of them sat in buckets of > 32.
#ifndef HG_CACHE_NB
#define HG_CACHE_NB 65536
#endif
constexpr int kNB = HG_CACHE_NB;
constexpr int kSuperB = 256;                 // buckets per super-bucket
constexpr int kNSuper = kNB / kSuperB;
static_assert((kNB & (kNB - 1)) == 0 && kNSuper >= 1 && kNSuper <= kSuperB,
              "bucket count: a power of two, at most 256 super-buckets");
constexpr int kBucketCap = 2048;
constexpr int kShortMax = 128;

struct BucketState {            // device scratch
  unsigned long long lo, hi;    // min / max norm bits over the n live keys
  int n_long;                   // buckets above kShortMax
  int ticket;                   // k_bs_offsets CTAs done
  int pad[2];
};

struct Admit {                  // U2 applied by the sort's writers (ctr null: off)
  const int32_t* live;
  const uint8_t* computed;
  int32_t* row_of;
  int32_t* row_owner;
  uint8_t* wflag;
  uint8_t* retained;
  long long* ctr;
};

// sorted position j holds key id (input index i): admission (j < k), write /
// retained flags, gradient eviction of a cached loser; returns evicted
__device__ __forceinline__ bool admit_pos(const Admit& A, long long k, int j, unsigned id, int i) {
  const bool admitted = j < k;
  const bool computed = A.computed[A.live[i]] != 0;
  bool evicted = false;
  if (!admitted) {
    const int r = A.row_of[id];
    if (r >= 0) {
      A.row_owner[r] = -1;
      A.row_of[id] = -1;
      evicted = true;
    }
  }
  A.wflag[j] = admitted && computed;
  A.retained[j] = admitted && !computed;
  return evicted;
}
// every thread of the CTA: add the evictions counted by its threads
__device__ __forceinline__ void admit_flush(const Admit& A, int evicted) {
  if (!A.ctr) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) evicted += __shfl_xor_sync(0xffffffffu, evicted, o);
  if ((threadIdx.x & 31) == 0 && evicted) {
    unsigned long long* c = reinterpret_cast<unsigned long long*>(A.ctr);
    atomicAdd(c + kCtrGradientEvictions, (unsigned long long)evicted);
    atomicAdd(c + kCtrValid, (unsigned long long)(-(long long)evicted));
  }
}

__device__ __forceinline__ int bucket_of(unsigned long long bits, unsigned long long lo, int shift) {
  const unsigned long long b = (bits - lo) >> shift;
  return b < (unsigned long long)kNB ? (int)b : kNB - 1;
}
__device__ __forceinline__ int bucket_shift(unsigned long long lo, unsigned long long hi) {
  const unsigned long long r = hi - lo;
  const int bits = r ? 64 - __clzll((long long)r) : 0;
  constexpr int kLog = __builtin_ctz(kNB);
  return bits > kLog ? bits - kLog : 0;
}
__device__ __forceinline__ bool key_less(unsigned long long an, unsigned ai, unsigned long long bn, unsigned bi) {
  return an < bn || (an == bn && ai < bi);
}
__device__ __forceinline__ int bucket_off(const int* loc, const int* spre, int b) {
  return loc[b] + spre[b / kSuperB];
}

__global__ void k_bs_count(const int32_t* n_dev, const NormKey* __restrict__ keys, const BucketState* st,
                           int* __restrict__ count, int* __restrict__ arrival) {
  pdl_wait();
  const int n = *n_dev;
  const unsigned long long lo = st->lo;
  const int shift = bucket_shift(lo, st->hi);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    arrival[i] = atomicAdd(&count[bucket_of(keys[i].norm, lo, shift)], 1);
}

// exclusive block scan of one int per thread (blockDim.x <= 1024)
__device__ __forceinline__ int block_excl_scan(int x, int* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int xs = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, xs, d);
    if (lane >= d) xs += t;
  }
  if (lane == 31) wsum[w] = xs;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    const int t = lane < nw ? wsum[lane] : 0;
    int ts = t;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, ts, d);
      if (lane >= d) ts += u;
    }
    if (lane < nw) wsum[lane] = ts - t;
  }
  __syncthreads();
  const int r = wsum[w] + xs - x;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kSuperB) k_bs_offsets(const int* __restrict__ count, int* __restrict__ loc,
                                                        int* __restrict__ stot, int* __restrict__ spre,
                                                        int* __restrict__ longl, BucketState* st) {
  pdl_wait();
  __shared__ int wsum[32];
  __shared__ int last;
  const int s = blockIdx.x, t = threadIdx.x;
  const int b = s * kSuperB + t;
  const int c = count[b];
  const int e = block_excl_scan(c, wsum);
  loc[b] = e;
  if (c > kShortMax) longl[atomicAdd(&st->n_long, 1)] = b;
  if (t == kSuperB - 1) {
    stot[s] = e + c;
    __threadfence();
    last = atomicAdd(&st->ticket, 1) == kNSuper - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int v = t < kNSuper ? __ldcg(&stot[t]) : 0;
  const int pe = block_excl_scan(v, wsum);
  if (t < kNSuper) spre[t] = pe;
}

__global__ void k_bs_place(const int32_t* n_dev, const NormKey* __restrict__ keys, const BucketState* st,
                           const int* __restrict__ loc, const int* __restrict__ spre, const int* __restrict__ arrival,
                           NormKey* __restrict__ tkeys, int32_t* __restrict__ tvals) {
  pdl_wait();
  const int n = *n_dev;
  const unsigned long long lo = st->lo;
  const int shift = bucket_shift(lo, st->hi);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const NormKey k = keys[i];
    const int pos = bucket_off(loc, spre, bucket_of(k.norm, lo, shift)) + arrival[i];
    tkeys[pos] = k;
    tvals[pos] = i;
  }
}

// in-smem bitonic sort of m (power of 2) (norm, id, val) items
__device__ __forceinline__ void smem_bitonic(unsigned long long* sn, unsigned* si, int* sv, int m) {
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (m >> 1); t += blockDim.x) {
        const int a = 2 * t - (t & (stride - 1));
        const int b = a + stride;
        const bool up = (a & size) == 0;
        if (key_less(sn[b], si[b], sn[a], si[a]) == up) {
          const unsigned long long tn = sn[a];
          const unsigned ti = si[a];
          const int tv = sv[a];
          sn[a] = sn[b]; si[a] = si[b]; sv[a] = sv[b];
          sn[b] = tn; si[b] = ti; sv[b] = tv;
        }
      }
      __syncthreads();
    }
  }
}

// merge path: number of items taken from A among the first d of merge(A, B)
__device__ __forceinline__ int merge_split(const NormKey* A, int na, const NormKey* B, int nb, int d) {
  int lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    // take A[mid] before B[d-1-mid] ?
    if (key_less(A[mid].norm, A[mid].id, B[d - 1 - mid].norm, B[d - 1 - mid].id)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// one CTA per listed bucket of > kShortMax keys: up to kBucketCap keys one
// shared-memory bitonic sort; above, sorted chunks of kBucketCap and
// bottom-up merge passes ping-ponging between tkeys/tvals and k2/v2
__device__ __forceinline__ void sort_long_buckets(const int* __restrict__ count, const int* __restrict__ loc,
                                                  const int* __restrict__ spre, const int* __restrict__ longl,
                                                  const BucketState* st, NormKey* __restrict__ tkeys,
                                                  int32_t* __restrict__ tvals, NormKey* __restrict__ k2,
                                                  int32_t* __restrict__ v2, NormKey* __restrict__ okeys,
                                                  int32_t* __restrict__ ovals, const Admit& A, long long k,
                                                  int& evicted) {
  __shared__ unsigned long long sn[kBucketCap];
  __shared__ unsigned si[kBucketCap];
  __shared__ int sv[kBucketCap];
  const int nlong = st->n_long;
  for (int q = blockIdx.x; q < nlong; q += gridDim.x) {
    const int b = longl[q];
    const int o = bucket_off(loc, spre, b), cnt = count[b];
    // 1. sorted chunks of up to kBucketCap (one chunk: straight to the output)
    const bool one = cnt <= kBucketCap;
    for (int c0 = 0; c0 < cnt; c0 += kBucketCap) {
      const int len = cnt - c0 < kBucketCap ? cnt - c0 : kBucketCap;
      int m = 2;
      while (m < len) m <<= 1;
      for (int t = threadIdx.x; t < m; t += blockDim.x) {
        if (t < len) {
          sn[t] = tkeys[o + c0 + t].norm;
          si[t] = tkeys[o + c0 + t].id;
          sv[t] = tvals[o + c0 + t];
        } else {
          sn[t] = ~0ull;
          si[t] = ~0u;
          sv[t] = -1;
        }
      }
      __syncthreads();
      smem_bitonic(sn, si, sv, m);
      for (int t = threadIdx.x; t < len; t += blockDim.x) {
        if (one) {
          okeys[o + t] = NormKey{sn[t], si[t]};
          ovals[o + t] = sv[t];
          if (A.ctr) evicted += admit_pos(A, k, o + t, si[t], sv[t]);
        } else {
          tkeys[o + c0 + t] = NormKey{sn[t], si[t]};
          tvals[o + c0 + t] = sv[t];
        }
      }
      __syncthreads();
    }
    if (one) continue;
    // 2. merge passes: runs of width w -> 2w
    NormKey* sk = tkeys + o;
    int32_t* svv = tvals + o;
    NormKey* dk = k2 + o;
    int32_t* dvv = v2 + o;
    for (int w = kBucketCap; w < cnt; w <<= 1) {
      for (int p0 = 0; p0 < cnt; p0 += 2 * w) {
        const int na = cnt - p0 < w ? cnt - p0 : w;
        const int nb = cnt - p0 - na < w ? (cnt - p0 - na > 0 ? cnt - p0 - na : 0) : w;
        const NormKey* Aa = sk + p0;
        const NormKey* B = Aa + na;
        const int tot = na + nb;
        const int per = (tot + blockDim.x - 1) / blockDim.x;
        const int d0 = threadIdx.x * per < tot ? threadIdx.x * per : tot;
        const int d1 = d0 + per < tot ? d0 + per : tot;
        int ia = merge_split(Aa, na, B, nb, d0), ib = d0 - ia;
        for (int d = d0; d < d1; ++d) {
          const bool takeA = ib >= nb || (ia < na && key_less(Aa[ia].norm, Aa[ia].id, B[ib].norm, B[ib].id));
          if (takeA) {
            dk[p0 + d] = Aa[ia];
            dvv[p0 + d] = svv[p0 + ia];
            ++ia;
          } else {
            dk[p0 + d] = B[ib];
            dvv[p0 + d] = svv[p0 + na + ib];
            ++ib;
          }
        }
      }
      __syncthreads();
      NormKey* tk = sk; sk = dk; dk = tk;
      int32_t* tv = svv; svv = dvv; dvv = tv;
    }
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
      const NormKey x = sk[t];
      okeys[o + t] = x;
      ovals[o + t] = svv[t];
      if (A.ctr) evicted += admit_pos(A, k, o + t, x.id, svv[t]);
    }
    __syncthreads();
  }
}

// one thread per key of a short bucket (<= kShortMax keys): its position is
// the bucket offset + the number of the bucket's keys below it; then the
// CTAs take the listed longer buckets one each (sort_long_buckets)
__global__ void __launch_bounds__(256) k_bs_rank(const int32_t* n_dev, const BucketState* st,
                                                 const int* __restrict__ count, const int* __restrict__ loc,
                                                 const int* __restrict__ spre, const int* __restrict__ longl,
                                                 NormKey* __restrict__ tkeys, int32_t* __restrict__ tvals,
                                                 NormKey* __restrict__ k2, int32_t* __restrict__ v2,
                                                 NormKey* __restrict__ okeys, int32_t* __restrict__ ovals, Admit A) {
  pdl_wait();
  const int n = *n_dev;
  const unsigned long long lo = st->lo;
  const int shift = bucket_shift(lo, st->hi);
  const long long k = A.ctr ? A.ctr[kCtrK] : 0;
  int evicted = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const NormKey key = tkeys[p];
    const int b = bucket_of(key.norm, lo, shift);
    const int c = count[b];
    if (c > kShortMax) continue;
    const int o = bucket_off(loc, spre, b);
    int r = 0;
#pragma unroll 4
    for (int q = 0; q < c; ++q) {
      const NormKey x = tkeys[o + q];
      r += key_less(x.norm, x.id, key.norm, key.id);
    }
    const int j = o + r;
    const int i = tvals[p];
    okeys[j] = key;
    ovals[j] = i;
    if (A.ctr) evicted += admit_pos(A, k, j, key.id, i);
  }
  sort_long_buckets(count, loc, spre, longl, st, tkeys, tvals, k2, v2, okeys, ovals, A, k, evicted);
  admit_flush(A, evicted);
}

// keys for i < n (the tail up to n_max gets sentinels that sort last) and the
// min / max norm bits over the n keys (one atomic pair per CTA)
__global__ void __launch_bounds__(256) k_norm_keys(const int32_t* n_dev, int n_max, double p_grad,
                                                   const int32_t* __restrict__ live,
                                                   const int32_t* __restrict__ src_nodes,
                                                   const double* __restrict__ norms, NormKey* __restrict__ keys,
                                                   int32_t* __restrict__ vals, long long* k_out, BucketState* st) {
  pdl_wait();
  __shared__ unsigned long long smn[8], smx[8];
  const int n = *n_dev;
  if (blockIdx.x == 0 && threadIdx.x == 0) *k_out = (long long)floor(p_grad * (double)n);  // cache.py:190
  unsigned long long mn = ~0ull, mx = 0ull;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_max; i += gridDim.x * blockDim.x) {
    if (i < n) {
      const unsigned long long v = (unsigned long long)__double_as_longlong(norms[i]);
      keys[i] = NormKey{v, (unsigned)src_nodes[live[i]]};
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    } else {
      keys[i] = NormKey{~0ull, ~0u};
    }
    vals[i] = i;
  }
  if (!st) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o), c = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = c > mx ? c : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = smn[w] < mn ? smn[w] : mn;
      mx = smx[w] > mx ? smx[w] : mx;
    }
    if (mn != ~0ull) {
      atomicMin(&st->lo, mn);
      atomicMax(&st->hi, mx);
    }
  }
}

// sharded cache (hg_shard_cache.cu): the batch-wide admission rank as
// per-position actions for the owners, in admit-rank order; no cache state
// is touched here. act 0 = not admitted (owner evicts it if held),
// 1 = admitted & computed (ring write), 2 = admitted & injected (retained).
// The rows to be written are staged at req_emb[j] (this rank's IPC-mapped
// request area: the owners read them from there, never from the tape). One
// warp per 32 positions: lane-parallel actions, then the warp copies the
// write rows with 16-byte vectors.
__global__ void k_request(const int32_t* n_dev, const NormKey* __restrict__ skeys, const int32_t* __restrict__ svals,
                          const int32_t* __restrict__ live, const uint8_t* __restrict__ computed_flag,
                          const float* __restrict__ emb, int row_words, int32_t* __restrict__ req_id,
                          uint8_t* __restrict__ req_act, int32_t* __restrict__ req_src, float* __restrict__ req_emb,
                          long long* hdr) {
  pdl_wait();
  const int n = *n_dev;
  const long long k = hdr[1];
  if (blockIdx.x == 0 && threadIdx.x == 0) hdr[0] = n;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int nv = row_words >> 2;
  for (int j0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; j0 < n; j0 += warps * 32) {
    const int j = j0 + lane;
    int loc = 0, act = 0;
    if (j < n) {
      loc = live[svals[j]];
      act = j >= k ? 0 : (computed_flag[loc] ? 1 : 2);
      req_id[j] = (int32_t)skeys[j].id;
      req_src[j] = loc;
      req_act[j] = (uint8_t)act;
    }
    unsigned m = __ballot_sync(0xffffffffu, act == 1);
    while (m) {
      const int q = __ffs(m) - 1;
      m &= m - 1;
      const int ql = __shfl_sync(0xffffffffu, loc, q);
      const uint4* s = reinterpret_cast<const uint4*>(emb + (long long)ql * row_words);
      uint4* d = reinterpret_cast<uint4*>(req_emb + (long long)(j0 + q) * row_words);
      for (int x = lane; x < nv; x += 32) d[x] = s[x];
    }
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

// a warp takes kWSlots consecutive write slots: lanes < kWSlots resolve their
// slot's node, source row and ring row (and set the ownership maps), then the
// warp copies the rows at once, lane group q (32 / kWSlots lanes) on row q
// with 16-byte vectors (all of a warp's rows in flight; many warps per SM)
constexpr int kWSlots = 4;
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
  const bool vec = (H & 3) == 0;
  const int nv = H >> 2;
  constexpr int kGL = 32 / kWSlots;   // lanes per row
  const int q = lane / kGL, gl = lane % kGL;
  for (long long g = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kWSlots; g < neff;
       g += warps * kWSlots) {
    long long srow = -1, drow = 0;
    if (lane < kWSlots && g + lane < neff) {
      const long long w = g + lane;
      const int j = wlist[w0 + w];
      const int id = (int)skeys[j].id;
      const int row = wrap_all ? (int)w : (int)((header + w) % cap);
      srow = live[svals[j]];
      drow = row;
      row_owner[row] = id;
      row_of[id] = row;
      admit_iter[id] = it;
    }
    const long long sr = __shfl_sync(0xffffffffu, srow, q);
    const long long dr = __shfl_sync(0xffffffffu, drow, q);
    if (sr < 0) continue;
    const float* src = emb + sr * H;
    float* dst = table + dr * H;
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
      for (int v = gl; v < H; v += kGL) dst[v] = src[v];
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

__global__ void k_sweep(long long* ctr, long long limit) {
  pdl_wait();
  const long long wa = ctr[kCtrWindowAdmissions], wf = ctr[kCtrWindowForced];
  long long cap = ctr[kCtrCapacity];
  if (wa != 0 && (double)wf > 0.01 * (double)wa && cap < limit) cap = cap * 2 < limit ? cap * 2 : limit;
  ctr[kCtrCapacity] = cap;
  ctr[kCtrWindowAdmissions] = 0;
  ctr[kCtrWindowForced] = 0;
  ctr[kCtrHeader] = 0;
}

}  // namespace
}  // namespace hg

using namespace hg;

extern "C" {

static long long bucket_tail_bytes(long long nn) {
  // k2 (16 B), v2, arrival (4 B each), state, count, loc, stot, spre, long list
  return nn * 24 + 64 + 4LL * (3 * kNB + 2 * kNSuper) + 64;
}

long long hg_cache_update_scratch_bytes(long long n_max) {
  const long long n = n_max + 16;
  // keys_in, keys_out (16 B), vals_in, vals_out, wlist (4 B), wflag, retained (1 B), scan partials,
  // bucket-sort tail
  return n * 16 * 2 + n * 4 * 3 + n * 2 + (scan_tiles(n_max) + 1) * 4 + 2048 + bucket_tail_bytes(n);
}

}  // extern "C"

namespace hg {
namespace {
struct RankBufs {
  NormKey *keys_in, *keys_out;
  int32_t *vals_in, *vals_out, *wlist;
  uint8_t *wflag, *retained;
  int* part;
  void* tmp;
  size_t tmp_bytes;
};

RankBufs carve(void* scratch, long long scratch_bytes, long long n_max) {
  RankBufs b;
  const long long nn = n_max + 16;
  char* p = reinterpret_cast<char*>(scratch);
  b.keys_in = reinterpret_cast<NormKey*>(p);
  b.keys_out = b.keys_in + nn;
  b.vals_in = reinterpret_cast<int32_t*>(b.keys_out + nn);
  b.vals_out = b.vals_in + nn;
  b.wlist = b.vals_out + nn;
  b.wflag = reinterpret_cast<uint8_t*>(b.wlist + nn);
  b.retained = b.wflag + nn;
  b.part = reinterpret_cast<int*>(b.retained + nn + 16 - ((uintptr_t)(b.retained + nn) & 15));
  b.tmp = b.part + scan_tiles(n_max) + 4;
  b.tmp_bytes = (size_t)(scratch_bytes - ((char*)b.tmp - p));
  return b;
}

// U1 (+ U2 when A.ctr is set): (norm bits, id) keys of the n live nodes
// sorted into keys_out / vals_out by the bucket sort; *k_out = floor(p_grad * n)
int bucket_rank(const char* W, const int32_t* n_dev, int n_max, double p_grad, const int32_t* live,
                const int32_t* src_nodes, const double* norms, long long* k_out, const RankBufs& rb, const Admit& A,
                cudaStream_t stream) {
  const long long nn = n_max + 16;
  const size_t need = (size_t)bucket_tail_bytes(nn);
  const uintptr_t end = reinterpret_cast<uintptr_t>(rb.tmp) + rb.tmp_bytes;
  char* bp = reinterpret_cast<char*>((end - need - 16) & ~uintptr_t(15));   // 16-byte aligned tail region
  NormKey* k2 = reinterpret_cast<NormKey*>(bp);
  int32_t* v2 = reinterpret_cast<int32_t*>(k2 + nn);
  int* arrival = v2 + nn;
  BucketState* bst = reinterpret_cast<BucketState*>((reinterpret_cast<uintptr_t>(arrival + nn) + 15) & ~uintptr_t(15));
  int* count = reinterpret_cast<int*>(bst + 1);
  int* loc = count + kNB;
  int* stot = loc + kNB;
  int* spre = stot + kNSuper;
  int* longl = spre + kNSuper;
  HG_CHECK_CUDA(W, cudaMemsetAsync(&bst->lo, 0xFF, 8, stream));
  // hi, n_long, ticket, pad, count: one zero fill
  HG_CHECK_CUDA(W, cudaMemsetAsync(&bst->hi, 0x00, 24 + 4 * (size_t)kNB, stream));
  const unsigned g = grid_for(n_max, 256, 148 * 4);
#define HG_L(K, G, B, ...)                                                                   \
  {                                                                                          \
    const cudaError_t _pe = hg::launch_pdl(K, dim3(G), dim3(B), 0, stream, __VA_ARGS__);     \
    if (_pe != cudaSuccess) return hg::fail(W, hg::kCuda, cudaGetErrorString(_pe));          \
    HG_LAUNCHED(W);                                                                          \
  }
  // keys -> k2 / v2; bucketed -> keys_in / vals_in; sorted -> keys_out / vals_out
  HG_L(k_norm_keys, grid_for(n_max, 256), 256, n_dev, n_max, p_grad, live, src_nodes, norms, k2, v2, k_out, bst);
  HG_L(k_bs_count, g, 256, n_dev, (const NormKey*)k2, (const BucketState*)bst, count, arrival);
  HG_L(k_bs_offsets, kNSuper, kSuperB, (const int*)count, loc, stot, spre, longl, bst);
  HG_L(k_bs_place, g, 256, n_dev, (const NormKey*)k2, (const BucketState*)bst, (const int*)loc, (const int*)spre,
       (const int*)arrival, rb.keys_in, rb.vals_in);
  HG_L(k_bs_rank, g, 256, n_dev, (const BucketState*)bst, (const int*)count, (const int*)loc, (const int*)spre,
       (const int*)longl, rb.keys_in, rb.vals_in, k2, v2, rb.keys_out, rb.vals_out, A);
#undef HG_L
  return kOk;
}
}  // namespace
}  // namespace hg

extern "C" {

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
  const RankBufs rb = carve(scratch, scratch_bytes, n_max);
  const Admit A{live, computed_flag, row_of, row_owner, rb.wflag, rb.retained, layer_ctr};
  const int s = bucket_rank(W, n_dev, n_max, p_grad, live, src_nodes, norms, layer_ctr + kCtrK, rb, A, stream);
  if (s) return s;
  return scan_launch<int>(W, FlagU8{rb.wflag}, DevCount{n_dev}, n_max, rb.part, EmitCompact{rb.wlist},
                          StoreNWrite{layer_ctr}, stream);
}

// Sharded cache, rank side (hg_shard_cache.cu): the same admission rank,
// published as (req_id, req_act, req_src, req_emb rows of the writes) in
// rank order with the header [0] n, [1] k (hdr[2] = it, hdr[3] = expiries:
// set by the reset / lookup side); the owners apply it. Scratch:
// hg_cache_update_scratch_bytes.
int hg_cache_request(const int32_t* n_dev, int n_max, double p_grad, const int32_t* live, const int32_t* src_nodes,
                     const double* norms, const uint8_t* computed_flag, const float* emb, int row_words,
                     int32_t* req_id, uint8_t* req_act, int32_t* req_src, float* req_emb, long long* req_hdr,
                     void* scratch, long long scratch_bytes, cudaStream_t stream) {
  const char* W = "hg_cache_request";
  if (scratch_bytes < hg_cache_update_scratch_bytes(n_max)) return fail(W, kBadArg, "scratch too small");
  if (row_words < 4 || (row_words & 3)) return fail(W, kBadArg, "rows must be a multiple of 4 words");
  if (n_max <= 0) return kOk;
  const RankBufs rb = carve(scratch, scratch_bytes, n_max);
  const int s = bucket_rank(W, n_dev, n_max, p_grad, live, src_nodes, norms, req_hdr + 1, rb, Admit{}, stream);
  if (s) return s;
  HG_CHECK_CUDA(W, hg::launch_pdl(k_request, dim3(grid_for((long long)n_max * 32, 256, 148 * 16)), dim3(256), 0,
                                  stream, n_dev, (const NormKey*)rb.keys_out, (const int32_t*)rb.vals_out, live,
                                  computed_flag, emb, row_words, req_id, req_act, req_src, req_emb, req_hdr));
  HG_LAUNCHED(W);
  return kOk;
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
  { const cudaError_t _pe = hg::launch_pdl(k_write_rows, dim3(grid_for((long long)n_max * 8, 256, 148 * 16)), dim3(256), 0, stream, 
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

// cache.py:206-211 (_LayerCache.sweep) on the device: grow when the window's
// forced overwrites exceed 1% of its admissions (doubling, up to `limit`
// rows, which the caller guarantees are allocated), reset the window
// counters and the ring header. The comparison is the reference's
// `forced > 0.01 * admissions` in float64 (exact for counts < 2^53).
int hg_cache_sweep(long long* layer_ctr, long long limit, cudaStream_t stream) {
  if (limit < 1) return fail("hg_cache_sweep", kBadArg, "limit must be >= 1");
  { const cudaError_t _pe = hg::launch_pdl(k_sweep, dim3(1), dim3(1), 0, stream, layer_ctr, limit);
    if (_pe != cudaSuccess) return hg::fail("launch", hg::kCuda, cudaGetErrorString(_pe)); }
  HG_LAUNCHED("hg_cache_sweep");
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
