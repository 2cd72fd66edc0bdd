// Native synthetic-graph generator for the benchmark shapes.
//
// Same process as histgnn/data.py:243-270 (preferential attachment: node v
// links to the previous step's m targets, the next targets are m distinct
// draws from the endpoint pool, i.e. degree-proportional), but with its own
// PRNG (splitmix64-seeded xoshiro256**), so it is NOT bit-identical to the
// numpy generator — the products / papers shapes are synthetic workloads, not
// parity fixtures (parity uses the reference generator restated in
// oracle/datagen.py). Host code; ~30 M pool draws per second.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "hgb200.h"

namespace {

struct Xoshiro {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  explicit Xoshiro(uint64_t seed) {
    for (auto& v : s) v = splitmix(seed);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  uint64_t below(uint64_t n) { return (uint64_t)(((unsigned __int128)next() * n) >> 64); }
};

}  // namespace

extern "C" {

// Writes 2*m*(n-m) directed edges (forward then reverse, like the reference)
// into src_out/dst_out (host int32 arrays of that length). Returns the count.
long long hg_synth_power_law(long long n, int m, unsigned long long seed, int32_t* src_out, int32_t* dst_out) {
  if (m < 1 || n < m + 1) return -1;
  const long long fwd = (long long)m * (n - m);
  std::vector<int32_t> pool((size_t)(2 * fwd));
  long long plen = 0, e = 0;
  std::vector<int32_t> tgt(m), nxt;
  nxt.reserve(m);
  for (int i = 0; i < m; ++i) tgt[i] = i;
  Xoshiro rng(seed);
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
      const int32_t c = pool[rng.below((uint64_t)plen)];
      if (std::find(nxt.begin(), nxt.end(), c) == nxt.end()) nxt.push_back(c);
    }
    std::sort(nxt.begin(), nxt.end());
    tgt.assign(nxt.begin(), nxt.end());
  }
  memcpy(src_out + fwd, dst_out, sizeof(int32_t) * fwd);
  memcpy(dst_out + fwd, src_out, sizeof(int32_t) * fwd);
  return 2 * fwd;
}

}  // extern "C"
