// Device-count-aware exclusive scan / stream compaction (reduce-then-scan).
//
// The element count lives in device memory (`n_dev`), the host only supplies an
// upper bound that sizes the grid, so scans chain after kernels whose output
// size is not yet known on the host. Three launches (the second folded into
// the third for scans of <= kSelfPrefixTiles tiles):
//   1. per-tile reduction of f(i) into partials[tile]
//   2. single-CTA exclusive scan of the partials (sequential carry over chunks)
//   3. per-tile block scan; emit(i, exclusive_prefix, f(i)) for every i < n and
//      total(sum) once.
// Integer-only use (offsets, compaction) -> associativity is exact.
#pragma once

#include "hg_common.cuh"

namespace hg {

struct I64x2 {
  long long a, b;
  __host__ __device__ I64x2 operator+(const I64x2& o) const { return {a + o.a, b + o.b}; }
  __host__ __device__ I64x2 operator-(const I64x2& o) const { return {a - o.a, b - o.b}; }
};

template <typename T>
__host__ __device__ inline T zero_of() { return T(0); }
template <>
__host__ __device__ inline I64x2 zero_of<I64x2>() { return {0, 0}; }

template <typename T>
__device__ __forceinline__ T shfl_up(T v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
template <>
__device__ __forceinline__ I64x2 shfl_up<I64x2>(I64x2 v, int d) {
  return {__shfl_up_sync(0xffffffffu, v.a, d), __shfl_up_sync(0xffffffffu, v.b, d)};
}
template <typename T>
__device__ __forceinline__ T shfl_idx(T v, int l) { return __shfl_sync(0xffffffffu, v, l); }
template <>
__device__ __forceinline__ I64x2 shfl_idx<I64x2>(I64x2 v, int l) {
  return {__shfl_sync(0xffffffffu, v.a, l), __shfl_sync(0xffffffffu, v.b, l)};
}

// element-count sources: produced on device, or a host constant
struct DevCount {
  const int32_t* p;
  __device__ long long get() const { return *p; }
};
struct ConstCount {
  long long n;
  __device__ long long get() const { return n; }
};

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// inclusive scan across the CTA of one value per thread; returns exclusive prefix,
// *block_total receives the CTA total.
template <typename T>
__device__ __forceinline__ T block_exclusive(T v, T* block_total) {
  __shared__ T warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T t = shfl_up(inc, d);
    if (lane >= d) inc = inc + t;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T w = lane < kScanThreads / 32 ? warp_tot[lane] : zero_of<T>();
    T wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T t = shfl_up(wi, d);
      if (lane >= d) wi = wi + t;
    }
    if (lane < kScanThreads / 32) warp_tot[lane] = wi;  // inclusive over warps
  }
  __syncthreads();
  T warp_prefix = wid ? warp_tot[wid - 1] : zero_of<T>();
  *block_total = warp_tot[kScanThreads / 32 - 1];
  __syncthreads();
  return warp_prefix + inc - v;
}

template <typename T, typename F, typename NC, int kItems = kScanItems>
__global__ void __launch_bounds__(kScanThreads) k_tile_reduce(F f, NC nc, T* partials) {
  pdl_wait();
  const long long n = nc.get();
  const long long base = (long long)blockIdx.x * (kScanThreads * kItems);
  T acc = zero_of<T>();
  if (base < n) {
    for (int k = 0; k < kItems; ++k) {
      long long i = base + (long long)k * kScanThreads + threadIdx.x;
      if (i < n) acc = acc + f(i);
    }
  }
  T tot;
  block_exclusive(acc, &tot);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

template <typename T>
__global__ void __launch_bounds__(1024) k_scan_partials(T* partials, int tiles) {
  __shared__ T wt[32];
  __shared__ T carry_s;
  pdl_wait();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = zero_of<T>();
  __syncthreads();
  for (int c0 = 0; c0 < tiles; c0 += 1024) {
    int i = c0 + threadIdx.x;
    T v = i < tiles ? partials[i] : zero_of<T>();
    T inc = v;
    for (int d = 1; d < 32; d <<= 1) {
      T t = shfl_up(inc, d);
      if (lane >= d) inc = inc + t;
    }
    if (lane == 31) wt[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      T w = wt[lane], wi = w;
      for (int d = 1; d < 32; d <<= 1) {
        T t = shfl_up(wi, d);
        if (lane >= d) wi = wi + t;
      }
      wt[lane] = wi;
    }
    __syncthreads();
    T carry = carry_s;
    T excl = carry + (wid ? wt[wid - 1] : zero_of<T>()) + inc - v;
    if (i < tiles) partials[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + wt[31];
    __syncthreads();
  }
}

// kSelfPrefix: `partials` holds the raw tile totals of k_tile_reduce and each
// CTA sums the ones before it itself (short scans: no single-CTA
// k_scan_partials launch between the two passes)
template <typename T, typename F, typename NC, typename Emit, typename Total, int kItems = kScanItems,
          bool kSelfPrefix = false>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(F f, NC nc, const T* partials, Emit emit,
                                                            Total total) {
  pdl_wait();
  const long long n = nc.get();
  const long long base = (long long)blockIdx.x * (kScanThreads * kItems);
  if (n == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) total(zero_of<T>());
    return;
  }
  if (base >= n) return;
  // each thread owns kItems consecutive items
  const long long tb = base + (long long)threadIdx.x * kItems;
  T v[kItems];
  T sum = zero_of<T>();
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    long long i = tb + k;
    v[k] = i < n ? f(i) : zero_of<T>();
    sum = sum + v[k];
  }
  T tot;
  T prefix;
  if constexpr (kSelfPrefix) {
    T acc = zero_of<T>();
    for (int t = threadIdx.x; t < (int)blockIdx.x; t += kScanThreads) acc = acc + partials[t];
    block_exclusive(acc, &prefix);
  } else {
    prefix = partials[blockIdx.x];
  }
  T run = prefix + block_exclusive(sum, &tot);
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    long long i = tb + k;
    if (i < n) {
      emit(i, run, v[k]);
      if (i == n - 1) total(run + v[k]);
    }
    run = run + v[k];
  }
}

// scans of at most this many tiles run in two launches (k_tile_scan sums the
// tile totals before its own tile); longer ones keep the single-CTA pass
#ifndef HG_SCAN_SELF_PREFIX_TILES
#define HG_SCAN_SELF_PREFIX_TILES 1024
#endif
constexpr long long kSelfPrefixTiles = HG_SCAN_SELF_PREFIX_TILES;

// Launch the three-kernel scan (two kernels up to kSelfPrefixTiles tiles). partials must hold >= scan_tiles(n_max) T
// (tiles of kScanThreads x kItems items; kItems < kScanItems for items whose
// emit is heavy, e.g. the sampler's bitmap words: more, shorter threads).
inline long long scan_tiles(long long n_max, int items = kScanItems) {
  return (n_max + (long long)kScanThreads * items - 1) / ((long long)kScanThreads * items);
}

template <typename T, int kItems = kScanItems, typename F, typename NC, typename Emit, typename Total>
int scan_launch(const char* where, F f, NC nc, long long n_max, T* partials, Emit emit, Total total,
                cudaStream_t s) {
  long long tiles = scan_tiles(n_max, kItems);
  if (tiles < 1) tiles = 1;
  HG_CHECK_CUDA(where, launch_pdl(k_tile_reduce<T, F, NC, kItems>, dim3((unsigned)tiles), dim3(kScanThreads), 0, s,
                                   f, nc, partials));
  HG_LAUNCHED(where);
  if (tiles <= kSelfPrefixTiles) {
    HG_CHECK_CUDA(where, launch_pdl(k_tile_scan<T, F, NC, Emit, Total, kItems, true>, dim3((unsigned)tiles),
                                     dim3(kScanThreads), 0, s, f, nc, (const T*)partials, emit, total));
    HG_LAUNCHED(where);
    return kOk;
  }
  HG_CHECK_CUDA(where, launch_pdl(k_scan_partials<T>, dim3(1), dim3(1024), 0, s, partials, (int)tiles));
  HG_LAUNCHED(where);
  HG_CHECK_CUDA(where, launch_pdl(k_tile_scan<T, F, NC, Emit, Total, kItems>, dim3((unsigned)tiles),
                                   dim3(kScanThreads), 0, s, f, nc, (const T*)partials, emit, total));
  HG_LAUNCHED(where);
  return kOk;
}

// ---- common functors ----

struct FlagU8 {
  const uint8_t* flags;
  __device__ int operator()(long long i) const { return flags[i] ? 1 : 0; }
};

// out_idx[rank] = i for every set flag; *count = number of set flags
struct EmitCompact {
  int32_t* out_idx;
  __device__ void operator()(long long i, int excl, int v) const {
    if (v) out_idx[excl] = (int32_t)i;
  }
};
struct StoreTotalI32 {
  int32_t* dst;
  __device__ void operator()(int t) const { *dst = t; }
};

}  // namespace hg
