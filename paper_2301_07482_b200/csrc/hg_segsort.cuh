// Segmented sort of 32-bit values (ascending) inside given segments
// [lo[c], hi[c]): used where a counting placement by atomics has to be made
// deterministic (the per-step CSC of a pruned block, the startup CSR2 build).
// Segments of <= kSegSmall values are insertion-sorted in registers by one
// thread each; longer ones are listed and sorted by one CTA each (chunks of
// kSegChunk in shared memory, then merge-path passes through `tmp`, which
// must cover the same index range as `vals`). Values are compared as
// unsigned, so the order is unique whatever the placement order was.
#pragma once

#include "hg_common.cuh"

namespace hg {
namespace {

constexpr int kSegSmall = 16;
constexpr int kSegChunk = 4096;

template <typename O>
__global__ void k_seg_sort_small(long long n_seg, const O* __restrict__ seg_lo, const O* __restrict__ seg_hi,
                                 unsigned* __restrict__ vals, int32_t* __restrict__ big, int32_t* n_big) {
  pdl_wait();
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n_seg; c += (long long)gridDim.x * blockDim.x) {
    const long long lo = seg_lo[c], len = (long long)seg_hi[c] - lo;
    if (len < 2) continue;
    if (len > kSegSmall) {
      big[atomicAdd(n_big, 1)] = (int32_t)c;
      continue;
    }
    unsigned v[kSegSmall];
#pragma unroll
    for (int k = 0; k < kSegSmall; ++k) v[k] = k < len ? vals[lo + k] : 0xffffffffu;
#pragma unroll
    for (int k = 1; k < kSegSmall; ++k) {
#pragma unroll
      for (int q = k; q > 0; --q) {
        const unsigned a = v[q - 1], b = v[q];
        v[q - 1] = a < b ? a : b;
        v[q] = a < b ? b : a;
      }
    }
#pragma unroll
    for (int k = 0; k < kSegSmall; ++k)
      if (k < len) vals[lo + k] = v[k];
  }
}

__device__ __forceinline__ void smem_bitonic_u32(unsigned* sv, int m) {
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (m >> 1); t += blockDim.x) {
        const int a = 2 * t - (t & (stride - 1));
        const int b = a + stride;
        const bool up = (a & size) == 0;
        if ((sv[b] < sv[a]) == up) {
          const unsigned x = sv[a];
          sv[a] = sv[b];
          sv[b] = x;
        }
      }
      __syncthreads();
    }
  }
}

template <typename O>
__global__ void __launch_bounds__(512) k_seg_sort_big(const int32_t* __restrict__ big, const int32_t* n_big,
                                                      const O* __restrict__ seg_lo, const O* __restrict__ seg_hi,
                                                      unsigned* __restrict__ vals, unsigned* __restrict__ tmp) {
  pdl_wait();
  __shared__ unsigned sv[kSegChunk];
  const int nb = *n_big;
  for (int q = blockIdx.x; q < nb; q += gridDim.x) {
    const int c = big[q];
    const long long lo = seg_lo[c], len = (long long)seg_hi[c] - lo;
    for (long long c0 = 0; c0 < len; c0 += kSegChunk) {
      const int n = (int)(len - c0 < kSegChunk ? len - c0 : kSegChunk);
      int m = 32;
      while (m < n) m <<= 1;
      for (int t = threadIdx.x; t < m; t += blockDim.x) sv[t] = t < n ? vals[lo + c0 + t] : 0xffffffffu;
      __syncthreads();
      smem_bitonic_u32(sv, m);
      for (int t = threadIdx.x; t < n; t += blockDim.x) vals[lo + c0 + t] = sv[t];
      __syncthreads();
    }
    unsigned* src = vals + lo;
    unsigned* dst = tmp + lo;
    bool in_tmp = false;
    for (long long w = kSegChunk; w < len; w <<= 1) {
      for (long long p0 = 0; p0 < len; p0 += 2 * w) {
        const long long na = len - p0 < w ? len - p0 : w;
        const long long rest = len - p0 - na;
        const long long nb2 = rest < w ? (rest > 0 ? rest : 0) : w;
        const unsigned* A = src + p0;
        const unsigned* B = A + na;
        const long long tot = na + nb2;
        const long long per = (tot + blockDim.x - 1) / blockDim.x;
        const long long d0 = threadIdx.x * per < tot ? threadIdx.x * per : tot;
        const long long d1 = d0 + per < tot ? d0 + per : tot;
        long long l2 = d0 > nb2 ? d0 - nb2 : 0, h2 = d0 < na ? d0 : na;
        while (l2 < h2) {      // merge path: items of A among the first d0
          const long long mid = (l2 + h2) >> 1;
          if (A[mid] <= B[d0 - 1 - mid]) l2 = mid + 1;
          else h2 = mid;
        }
        long long ia = l2, ib = d0 - l2;
        for (long long d = d0; d < d1; ++d) dst[p0 + d] = (ib >= nb2 || (ia < na && A[ia] <= B[ib])) ? A[ia++] : B[ib++];
      }
      __syncthreads();
      unsigned* t2 = src;
      src = dst;
      dst = t2;
      in_tmp = !in_tmp;
    }
    if (in_tmp)
      for (long long t = threadIdx.x; t < len; t += blockDim.x) vals[lo + t] = tmp[lo + t];
    __syncthreads();
  }
}

// n_big must be zero on entry (the caller's memset, on the same stream)
template <typename O>
int segsort_launch(const char* W, long long n_seg, const O* seg_lo, const O* seg_hi, unsigned* vals, unsigned* tmp,
                   int32_t* big, int32_t* n_big, cudaStream_t stream) {
  HG_CHECK_CUDA(W, hg::launch_pdl(k_seg_sort_small<O>, dim3(grid_for(n_seg, 256)), dim3(256), 0, stream, n_seg,
                                  seg_lo, seg_hi, vals, big, n_big));
  HG_LAUNCHED(W);
  HG_CHECK_CUDA(W, hg::launch_pdl(k_seg_sort_big<O>, dim3(148), dim3(512), 0, stream, (const int32_t*)big,
                                  (const int32_t*)n_big, seg_lo, seg_hi, vals, tmp));
  HG_LAUNCHED(W);
  return kOk;
}

}  // namespace
}  // namespace hg
