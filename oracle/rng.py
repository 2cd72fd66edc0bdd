"""PCG64 stream arithmetic behind the sampler's uniform keys (oracle).

The reference draws one uniform key per candidate in-edge with
`rng.random(total)` on a per-batch `default_rng(SeedSequence((seed, idx)))`
(histgnn/sampler.py:104-106,133). The arithmetic lives in numpy (a third-party
dependency absent from /root/reference; numpy 2.3.x here, PCG64 stream stable
since numpy 1.17, NEP-19). Its published algorithm, restated:

    step:    s <- s * PCG_MULT + inc              (mod 2**128), before output
    output:  x = rotr64(hi(s) ^ lo(s), s >> 122)  (XSL-RR 128/64)
    random() = (x >> 11) * 2**-53

so a key is the 53-bit integer `x >> 11` and stream index k (0-based) is the
output after k+1 steps — the GPU kernel jumps straight to any k. This module
is pure Python big-int arithmetic and is pinned against numpy itself in
tests/test_oracle_golden.py.
"""

from __future__ import annotations

import numpy as np

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
M128 = (1 << 128) - 1
M64 = (1 << 64) - 1


def pcg64_seed_state(seed: int, batch_index: int) -> tuple[int, int]:
    """(state, inc) of default_rng(SeedSequence((seed, batch_index))) before
    any draw — the host-side seeding the GPU sampler starts from."""
    bg = np.random.PCG64(np.random.SeedSequence((int(seed), int(batch_index))))
    st = bg.state["state"]
    return int(st["state"]), int(st["inc"])


def jump(state: int, inc: int, k: int) -> int:
    """State after k LCG steps (square-and-multiply on the affine map)."""
    a, c = 1, 0          # accumulated map x -> a*x + c
    ma, mc = PCG_MULT, inc
    while k:
        if k & 1:
            a, c = (a * ma) & M128, (c * ma + mc) & M128
        ma, mc = (ma * ma) & M128, (mc * ma + mc) & M128
        k >>= 1
    return (a * state + c) & M128


def _xsl_rr(s: int) -> int:
    x = ((s >> 64) ^ s) & M64
    r = s >> 122
    return ((x >> r) | (x << ((64 - r) & 63))) & M64


def pcg64_keys53(state: int, inc: int, offset: int, count: int) -> np.ndarray:
    """Keys (53-bit ints) at stream indices offset .. offset+count-1."""
    s = jump(state, inc, offset)
    out = np.empty(count, dtype=np.uint64)
    for i in range(count):
        s = (s * PCG_MULT + inc) & M128
        out[i] = _xsl_rr(s) >> 11
    return out
