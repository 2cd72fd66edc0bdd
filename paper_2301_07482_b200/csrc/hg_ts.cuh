// "TS" (tiled split) operand format shared by the producers of GEMM operands
// (k_aggregate, k_gather_dz, the per-step weight split) and the tcgen05 GEMM.
//
// A logical fp32 matrix X[rows x cols] is stored as bf16 hi/lo halves
// (x = hi + lo, hi = bf16(x), lo = bf16(x - hi)) in blocks of 128 rows x 32
// columns. Block (rt, kc) lives at byte offset (rt * nK + kc) * 16 KB and
// holds [hi 8 KB][lo 8 KB]; inside a half, element (r, k) sits in the UMMA
// canonical no-swizzle core-matrix layout: 8 rows x 16 B core matrices,
//   byte = (r / 8) * 512 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2.
// A block half is therefore directly a K-major tcgen05 operand tile
// (LBO = 128 B between k-cores, SBO = 512 B between 8-row groups), and each
// core matrix read "sideways" is an MN-major core matrix for the transposed
// use (the weight-gradient GEMM), so one stored copy serves both.
// Rows are padded to a multiple of 128 and columns to a multiple of 32 with
// zeros by the producers.
#pragma once

#include <cuda_bf16.h>

#include "hg_common.cuh"

namespace hg {

constexpr int kTsRows = 128;
constexpr int kTsCols = 32;
constexpr int kTsBlock = 16384;      // bytes per (row tile, col chunk): hi + lo
constexpr int kTsHalf = 8192;

__host__ __device__ inline long long ts_bytes(long long rows, int cols) {
  const long long rt = (rows + kTsRows - 1) / kTsRows;
  const long long nk = (cols + kTsCols - 1) / kTsCols;
  return (rt < 1 ? 1 : rt) * (nk < 1 ? 1 : nk) * kTsBlock;
}

__device__ __forceinline__ long long ts_off(int r, int c, int nK) {
  const int rt = r >> 7, rr = r & 127, kc = c >> 5, k = c & 31;
  return (long long)(rt * nK + kc) * kTsBlock + (rr >> 3) * 512 + (k >> 3) * 128 + (rr & 7) * 16 + (k & 7) * 2;
}

// pack 8 consecutive fp32 values (one core-matrix row) into hi/lo 16-byte words
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float a = v[2 * q], b = v[2 * q + 1];
    const __nv_bfloat16 ah = __float2bfloat16_rn(a), bh = __float2bfloat16_rn(b);
    const __nv_bfloat16 al = __float2bfloat16_rn(a - __bfloat162float(ah));
    const __nv_bfloat16 bl = __float2bfloat16_rn(b - __bfloat162float(bh));
    h[q] = (uint32_t)__bfloat16_as_ushort(ah) | ((uint32_t)__bfloat16_as_ushort(bh) << 16);
    l[q] = (uint32_t)__bfloat16_as_ushort(al) | ((uint32_t)__bfloat16_as_ushort(bl) << 16);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// store the 8-column group g (cols 8g..8g+7) of row r from fp32 values
__device__ __forceinline__ void ts_store8(uint8_t* ts, int nK, int r, int g, const float* v8) {
  uint4 hi, lo;
  split8(v8, hi, lo);
  const long long off = ts_off(r, g * 8, nK);
  *reinterpret_cast<uint4*>(ts + off) = hi;
  *reinterpret_cast<uint4*>(ts + off + kTsHalf) = lo;
}

}  // namespace hg
