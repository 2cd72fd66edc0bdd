// "TS" (tiled split) operand format shared by the producers of GEMM operands
// (k_aggregate, k_gather_dz, the per-step weight split) and the tcgen05 GEMM.
//
// A logical fp32 matrix X[rows x cols] is stored as two bf16 planes, hi and lo
// (x = hi + lo, hi = bf16(x), lo = bf16(x - hi)), each in "row-group strip"
// order: rows are grouped by 8 (G = r / 8), columns by 8 (cg = c / 8), and the
// 8 x 8 bf16 core matrix (8 rows x 16 B) of (G, cg) is 128 contiguous bytes:
//   byte(r, c) = ((G * nCG + cg) * 8 + r % 8) * 16 + (c % 8) * 2,
//   lo plane = hi plane + plane_bytes,  plane_bytes = rows_pad * nCG * 16,
// with rows padded to a multiple of 128 and columns to a multiple of 32 (zeros).
// Every tcgen05 operand stage is then ONE 4-D TMA box over
// (core bytes, cg, G, plane), strides increasing:
//   K-major  stage (128 rows x 32 cols): box (64, 4, 16, 2) -> smem [plane][G][cg][core]
//            (SBO = 512 B between row groups, LBO = 128 B between k-cores)
//   MN-major stage (32 rows x M cols):  box (64, M/8, 4, 2) -> smem [plane][G][cg][core]
//            (SBO = 128 B between MN groups, LBO = M/8 * 128 B between k-groups)
// so one stored copy serves the forward / data-gradient GEMMs (K-major) and
// the weight-gradient GEMM (reads the same cores as MN-major operands).
#pragma once

#include <cuda_bf16.h>

#include "hg_common.cuh"

namespace hg {

constexpr int kTsRows = 128;   // row padding granularity
constexpr int kTsCols = 32;    // column padding granularity (one K chunk)

__host__ __device__ inline long long ts_rows_pad(long long rows) {
  long long p = (rows + kTsRows - 1) / kTsRows * kTsRows;
  return p < kTsRows ? kTsRows : p;
}
__host__ __device__ inline int ts_ncg(int cols) {
  int nk = (cols + kTsCols - 1) / kTsCols;
  return (nk < 1 ? 1 : nk) * 4;
}
__host__ __device__ inline long long ts_plane_bytes(long long rows, int cols) {
  return ts_rows_pad(rows) * ts_ncg(cols) * 16;
}
__host__ __device__ inline long long ts_bytes(long long rows, int cols) { return 2 * ts_plane_bytes(rows, cols); }

__device__ __forceinline__ long long ts_off(int r, int c, int nCG) {
  return ((long long)(r >> 3) * nCG + (c >> 3)) * 128 + (r & 7) * 16 + (c & 7) * 2;
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

// store column group g (cols 8g..8g+7) of row r
__device__ __forceinline__ void ts_store8(uint8_t* ts, int nCG, long long plane, int r, int g, const float* v8) {
  uint4 hi, lo;
  split8(v8, hi, lo);
  const long long off = ts_off(r, g * 8, nCG);
  *reinterpret_cast<uint4*>(ts + off) = hi;
  *reinterpret_cast<uint4*>(ts + plane + off) = lo;
}

// A warp's staging row for TS emission (aggregation / transposed aggregation):
// logical float4 chunk j lives at j ^ ((j >> 3) & 1). The emission reads a
// 32-byte column group per lane (chunks 2g, 2g + 1); unswizzled, the 8 lanes
// of an LDS.128 phase hit every bank pair twice (ncu: 3.6M shared-load bank
// conflicts, 7.4 wavefronts per load in the C2 layer-0 aggregation); the
// swizzle spreads them over all banks, and lane-per-chunk writes stay
// conflict-free (the XOR stays inside each aligned group of 8 chunks).
__device__ __forceinline__ int stage_chunk(int j) { return j ^ ((j >> 3) & 1); }
__device__ __forceinline__ void stage_put4(float* row, int j, float4 v) {
  reinterpret_cast<float4*>(row)[stage_chunk(j)] = v;
}
__device__ __forceinline__ float4 stage_get4(const float* row, int j) {
  return reinterpret_cast<const float4*>(row)[stage_chunk(j)];
}
__device__ __forceinline__ void stage_put1(float* row, int c, float x) { row[stage_chunk(c >> 2) * 4 + (c & 3)] = x; }
// emit column group g (logical columns 8g .. 8g + 7) of a staged row
__device__ __forceinline__ void ts_store8_staged(uint8_t* ts, int nCG, long long plane, int r, int g,
                                                 const float* row) {
  const float4 a = stage_get4(row, 2 * g), b = stage_get4(row, 2 * g + 1);
  const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  ts_store8(ts, nCG, plane, r, g, v);
}

}  // namespace hg
