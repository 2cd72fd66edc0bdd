// Native synthetic-graph generator for the benchmark shapes.
//
// Bit-identical to histgnn/data.py:243-270 (`synth_power_law`): node v links
// to the previous step's targets, appends them and v to the endpoint pool,
// then draws `pool[rng.integers(len(pool))]` until m distinct targets are
// chosen, sorted ascending. The caller passes the numpy Generator's PCG64
// state (bit_generator.state: 128-bit state and increment, the buffered
// 32-bit half `has_uint32`/`uinteger`), and gets the advanced state back so
// numpy continues the same stream for the features / labels / split draws.
//
// `Generator.integers(high)` for a scalar high (numpy/random/_bounded_integers
// `_rand_int64` -> random_bounded_uint64_fill) is reproduced exactly:
//   range = high - 1 < 2^32 : Lemire's multiply-shift on next_uint32 (which
//                             serves the stored upper half of the previous
//                             64-bit output first), rejection below
//                             (2^32 - high) % high;
//   range == 2^32 - 1       : next_uint32 itself;
//   larger ranges           : Lemire on next_uint64 with a 128-bit product.
// Host code, single thread (the process is sequential); ~40 M draws/s.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "hgb200.h"

namespace {

typedef unsigned __int128 u128;

struct NumpyPCG64 {
  u128 state, inc;
  int has32;
  uint32_t half;

  uint64_t next64() {
    const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has32) {
      has32 = 0;
      return half;
    }
    const uint64_t n = next64();
    has32 = 1;
    half = (uint32_t)(n >> 32);
    return (uint32_t)n;
  }
  // Generator.integers(high), high >= 1
  uint64_t integers(uint64_t high) {
    const uint64_t rng = high - 1;
    if (rng == 0) return 0;
    if (rng < 0xFFFFFFFFull) {
      const uint32_t excl = (uint32_t)high;
      uint64_t m = (uint64_t)next32() * excl;
      uint32_t left = (uint32_t)m;
      if (left < excl) {
        const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
        while (left < thr) {
          m = (uint64_t)next32() * excl;
          left = (uint32_t)m;
        }
      }
      return m >> 32;
    }
    if (rng == 0xFFFFFFFFull) return next32();
    u128 m = (u128)next64() * high;
    uint64_t left = (uint64_t)m;
    if (left < high) {
      const uint64_t thr = (0xFFFFFFFFFFFFFFFFull - rng) % high;
      while (left < thr) {
        m = (u128)next64() * high;
        left = (uint64_t)m;
      }
    }
    return (uint64_t)(m >> 64);
  }
};

}  // namespace

extern "C" {

// pcg[6] in/out: state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger.
// Writes 2*m*(n-m) directed edges (forward half, then the reversed half, as
// data.py:262-266) into src_out/dst_out (host int32). Returns the count, or -1
// for invalid (n, m) (data.py:247-248 raises ValueError).
long long hg_synth_power_law(long long n, int m, unsigned long long* pcg, int32_t* src_out, int32_t* dst_out) {
  if (m < 1 || n < m + 1) return -1;
  NumpyPCG64 g;
  g.state = ((u128)pcg[0] << 64) | pcg[1];
  g.inc = ((u128)pcg[2] << 64) | pcg[3];
  g.has32 = pcg[4] ? 1 : 0;
  g.half = (uint32_t)pcg[5];
  const long long fwd = (long long)m * (n - m);
  std::vector<int32_t> pool((size_t)(2 * fwd));
  long long plen = 0, e = 0;
  std::vector<int32_t> tgt(m), nxt;
  nxt.reserve(m);
  for (int i = 0; i < m; ++i) tgt[i] = i;
  for (long long v = m; v < n; ++v) {
    for (int i = 0; i < m; ++i) {
      src_out[e] = (int32_t)v;
      dst_out[e] = tgt[i];
      ++e;
      pool[plen + i] = tgt[i];
      pool[plen + m + i] = (int32_t)v;
    }
    plen += 2 * m;
    nxt.clear();
    while ((int)nxt.size() < m) {
      const int32_t c = pool[g.integers((uint64_t)plen)];
      if (std::find(nxt.begin(), nxt.end(), c) == nxt.end()) nxt.push_back(c);
    }
    std::sort(nxt.begin(), nxt.end());
    tgt.assign(nxt.begin(), nxt.end());
  }
  memcpy(src_out + fwd, dst_out, sizeof(int32_t) * fwd);
  memcpy(dst_out + fwd, src_out, sizeof(int32_t) * fwd);
  pcg[0] = (unsigned long long)(g.state >> 64);
  pcg[1] = (unsigned long long)g.state;
  pcg[2] = (unsigned long long)(g.inc >> 64);
  pcg[3] = (unsigned long long)g.inc;
  pcg[4] = (unsigned long long)g.has32;
  pcg[5] = (unsigned long long)g.half;
  return 2 * fwd;
}

}  // extern "C"
