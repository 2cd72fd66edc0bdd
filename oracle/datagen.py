"""Synthetic inputs and the full-graph CSR2 build (oracle restatement).

Restates the reference's input fixtures so the same graphs can be rebuilt on
a box where /root/reference does not exist:
- power-law preferential attachment: histgnn/data.py:243-270
- stochastic block model:             histgnn/data.py:185-240
- 60/20/20 id split:                  histgnn/data.py:173-182
- in-neighbour CSR2, stable per row:  histgnn/graphs.py:161-172

The numpy Generator calls are issued in exactly the reference's order, so the
outputs are bit-identical for the same seed (pinned by tests/golden).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Dataset:
    src: np.ndarray          # int64[E]  edge sources
    dst: np.ndarray          # int64[E]  edge destinations
    num_nodes: int
    features: np.ndarray     # [N, d]
    labels: np.ndarray       # int64[N]
    train_ids: np.ndarray
    val_ids: np.ndarray
    test_ids: np.ndarray

    @property
    def num_classes(self) -> int:
        return int(self.labels.max()) + 1 if len(self.labels) else 0


def _three_way_split(n: int, rng: np.random.Generator):
    """data.py:173-182 — one permutation, 60% / 20% / rest, each sorted."""
    p = rng.permutation(n)
    a, b = int(0.6 * n), int(0.2 * n)
    return np.sort(p[:a]), np.sort(p[a:a + b]), np.sort(p[a + b:])


def power_law_dataset(n: int, rng: np.random.Generator, m: int = 3,
                      feature_dim: int = 32, classes: int = 8) -> Dataset:
    """data.py:243-270. Node v >= m links to the previous step's target set;
    the next target set is m distinct draws from the endpoint pool (uniform
    pool index = degree-proportional choice), sorted ascending."""
    if m < 1 or n < m + 1:
        raise ValueError(f"need n >= m + 1 >= 2, got n={n} m={m}")
    # endpoint pool grows by 2*m per node; preallocate instead of list appends
    pool = np.empty(2 * m * (n - m), dtype=np.int64)
    plen = 0
    fwd_src = np.empty(m * (n - m), dtype=np.int64)
    fwd_dst = np.empty(m * (n - m), dtype=np.int64)
    ecount = 0
    tgt = list(range(m))
    draw = rng.integers
    for v in range(m, n):
        k = len(tgt)
        fwd_src[ecount:ecount + k] = v
        fwd_dst[ecount:ecount + k] = tgt
        ecount += k
        pool[plen:plen + k] = tgt
        pool[plen + k:plen + 2 * k] = v
        plen += 2 * k
        picked = set()
        while len(picked) < m:
            picked.add(int(pool[draw(plen)]))
        tgt = sorted(picked)
    fwd_src, fwd_dst = fwd_src[:ecount], fwd_dst[:ecount]
    src = np.concatenate([fwd_src, fwd_dst])
    dst = np.concatenate([fwd_dst, fwd_src])
    feats = rng.standard_normal((n, feature_dim)).astype(np.float32)
    labels = rng.integers(0, classes, size=n)
    tr, va, te = _three_way_split(n, rng)
    return Dataset(src, dst, n, feats, np.asarray(labels, np.int64), tr, va, te)


def sbm_dataset(n, rng, blocks=8, p_in=None, p_out=None, feature_dim=32, noise=1.0):
    """data.py:185-240 — block-structured graph, label = block id."""
    if n < 2 or blocks < 1 or blocks > n:
        raise ValueError(f"need 2 <= blocks <= n, got n={n} blocks={blocks}")
    p_in = min(1.0, 10.0 * blocks / n) if p_in is None else p_in
    p_out = p_in / 20.0 if p_out is None else p_out
    sizes = np.full(blocks, n // blocks)
    sizes[: n % blocks] += 1
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    labels = np.repeat(np.arange(blocks), sizes)
    us, vs = [], []
    for i in range(blocks):
        for j in range(i, blocks):
            p = p_in if i == j else p_out
            if p <= 0:
                continue
            if i == j:
                u, v = np.triu_indices(sizes[i], k=1)
                u, v = u + bounds[i], v + bounds[i]
            else:
                u = np.repeat(np.arange(bounds[i], bounds[i + 1]), sizes[j])
                v = np.tile(np.arange(bounds[j], bounds[j + 1]), sizes[i])
            sel = rng.random(u.size) < p
            us.append(u[sel])
            vs.append(v[sel])
    hu = np.concatenate(us) if us else np.empty(0, np.int64)
    hv = np.concatenate(vs) if vs else np.empty(0, np.int64)
    centers = rng.standard_normal((blocks, feature_dim))
    feats = (centers[labels] + noise * rng.standard_normal((n, feature_dim))).astype(np.float32)
    tr, va, te = _three_way_split(n, rng)
    return Dataset(np.concatenate([hu, hv]).astype(np.int64),
                   np.concatenate([hv, hu]).astype(np.int64), n, feats,
                   labels.astype(np.int64), tr, va, te)


def csr2_from_edges(src, dst, num_nodes):
    """graphs.py:161-172 — in-neighbour rows (row v lists sources of edges into
    v), edges within a row kept in input order. Returns (start, end, col)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    ptr = np.zeros(num_nodes + 1, dtype=np.int64)
    np.cumsum(np.bincount(dst, minlength=num_nodes), out=ptr[1:])
    perm = np.argsort(dst, kind="stable")
    return ptr[:-1].copy(), ptr[1:].copy(), src[perm]
