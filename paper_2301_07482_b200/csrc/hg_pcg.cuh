// PCG64 (numpy's XSL-RR 128/64 generator) with O(log k) jump-ahead on device.
//
// Stream contract restated from numpy (see oracle/rng.py):
//   step:   s <- s * MULT + inc  (mod 2^128)   (step happens before output)
//   output: x = rotr64(hi(s) ^ lo(s), hi(s) >> 58)
//   Generator.random() = (x >> 11) * 2^-53  -> the sampler compares x >> 11.
// Stream index k (0-based) is the output after k+1 steps from the seeded state.
//
// Jump tables: kJumpA[w][d] = MULT^(d*16^w), kJumpS[w][d] = sum_{i<m} MULT^i
// for m = d*16^w, so that  s_{k+m} = A*s_k + inc*S. Independent of inc, built
// once per process (host unsigned __int128) and kept in __device__ memory.
#pragma once

#include "hg_common.cuh"

namespace hg {

struct u128 {
  unsigned long long hi, lo;
};

__host__ __device__ __forceinline__ u128 mul128(u128 a, u128 b) {
  u128 r;
#ifdef __CUDA_ARCH__
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
#else
  unsigned __int128 p = (unsigned __int128)a.lo * b.lo;
  r.lo = (unsigned long long)p;
  r.hi = (unsigned long long)(p >> 64) + a.hi * b.lo + a.lo * b.hi;
#endif
  return r;
}

__host__ __device__ __forceinline__ u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}

// a*x + c
__host__ __device__ __forceinline__ u128 fma128(u128 a, u128 x, u128 c) { return add128(mul128(a, x), c); }

__host__ __device__ __forceinline__ unsigned long long pcg_key53(u128 s) {
  unsigned long long x = s.hi ^ s.lo;
  unsigned r = (unsigned)(s.hi >> 58);
  unsigned long long out = (x >> r) | (x << ((64 - r) & 63));
  return out >> 11;
}

constexpr unsigned long long kMultHi = 0x2360ED051FC65DA4ull;
constexpr unsigned long long kMultLo = 0x4385DF649FCCF645ull;

// 16 nibble windows x 16 digits
struct JumpTable {
  u128 A[16][16];
  u128 S[16][16];
};


int ensure_jump_table();  // uploads g_jump once per device

// state after k steps from s (inc supplied per batch); tab in shared or global memory
__device__ __forceinline__ u128 pcg_jump(const JumpTable& tab, u128 s, u128 inc, unsigned long long k) {
  int w = 0;
  while (k) {
    unsigned d = (unsigned)(k & 15ull);
    if (d) s = add128(mul128(tab.A[w][d], s), mul128(inc, tab.S[w][d]));
    k >>= 4;
    ++w;
  }
  return s;
}

}  // namespace hg
