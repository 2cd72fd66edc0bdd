"""Layered fan-out sampler (oracle restatement of histgnn/sampler.py).

Semantics restated (all integer, bit-exact targets for the GPU sampler):
- `split_batches`  sampler.py:95-101 — one permutation, cut into batches.
- `batch_rng`      sampler.py:104-106 — PCG64 on SeedSequence((seed, idx)).
- `_pick`          sampler.py:118-138 — one uniform key per candidate in-edge,
  consumed in frontier order; per row keep the min(deg, fanout) smallest by
  (key, position-in-row); emit the chosen global sources in ascending key order.
- `_relabel`       sampler.py:141-163 — new = sorted unique sources not already
  in the frontier; src = frontier ++ new; local column ids; dst_deg = counts.
- `sample_layered` sampler.py:166-190 — outermost first, blocks reversed to
  innermost-first, src_deg chained (block 0 gets zeros).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class OBlock:
    dst_nodes: np.ndarray   # int64[n_dst] == src_nodes[:n_dst]
    src_nodes: np.ndarray   # int64[n_src]
    start: np.ndarray       # int64[n_dst] local CSR2 row starts
    end: np.ndarray         # int64[n_dst] local CSR2 row ends (pruning sets end=start)
    col: np.ndarray         # int64[E]     local source positions
    dst_deg: np.ndarray     # int64[n_dst] build-time sampled in-degree
    src_deg: np.ndarray | None = None
    prune_writes: int = 0

    @property
    def num_dst(self):
        return len(self.dst_nodes)

    @property
    def num_src(self):
        return len(self.src_nodes)

    def copy(self):
        return OBlock(self.dst_nodes, self.src_nodes, self.start.copy(), self.end.copy(),
                      self.col, self.dst_deg, self.src_deg, 0)


@dataclass
class OSubgraph:
    seeds: np.ndarray
    layers: list  # innermost first

    @property
    def num_layers(self):
        return len(self.layers)

    @property
    def input_nodes(self):
        return self.layers[0].src_nodes

    def copy(self):
        return OSubgraph(self.seeds, [b.copy() for b in self.layers])


def split_batches(ids, batch_size, rng):
    ids = np.asarray(ids, dtype=np.int64)
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    p = rng.permutation(ids)
    return [p[o:o + batch_size] for o in range(0, len(p), batch_size)]


def batch_rng(seed, idx):
    return np.random.default_rng(np.random.SeedSequence((int(seed), int(idx))))


def _segment_positions(lengths):
    """0..l0-1, 0..l1-1, ... for int64 lengths."""
    n = int(lengths.sum())
    if n == 0:
        return np.empty(0, np.int64)
    heads = np.cumsum(lengths) - lengths
    return np.arange(n, dtype=np.int64) - np.repeat(heads, lengths)


def _pick(start, end, col, frontier, fanout, rng):
    """sampler.py:118-138. Returns (counts int64[F], chosen global ids)."""
    row_lo = start[frontier]
    deg = (end[frontier] - row_lo).astype(np.int64)
    counts = np.minimum(deg, fanout)
    total = int(deg.sum())
    if total == 0:
        return counts, np.empty(0, np.int64)
    u = rng.random(total)                       # stream consumed in frontier order
    owner = np.repeat(np.arange(len(frontier), dtype=np.int64), deg)
    # stable: within a row ties on the key fall back to candidate position
    perm = np.lexsort((u, owner))
    heads = np.repeat(np.cumsum(deg) - deg, deg)
    j = perm - heads                            # candidate position within its row
    rank = _segment_positions(deg)              # rank of perm[i] inside its row
    sel = rank < fanout
    edge = np.repeat(row_lo, deg) + j
    return counts, col[edge[sel]]


def _relabel(frontier, counts, chosen):
    """sampler.py:141-163 without the O(N) scratch: membership via sorted search."""
    uniq = np.unique(chosen)
    new = np.setdiff1d(uniq, frontier, assume_unique=True)   # sorted ascending
    src = np.concatenate([frontier, new]).astype(np.int64)
    order = np.argsort(src, kind="stable")
    local = order[np.searchsorted(src[order], chosen)]
    ptr = np.zeros(len(frontier) + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    return OBlock(frontier, src, ptr[:-1].copy(), ptr[1:].copy(),
                  local.astype(np.int64), counts.astype(np.int64))


def sample_layered(start, end, col, num_nodes, seeds, fanouts, rng) -> OSubgraph:
    seeds = np.asarray(seeds, dtype=np.int64)
    if len(seeds) == 0:
        raise ValueError("empty seed set")
    if len(np.unique(seeds)) != len(seeds):
        raise ValueError("seed ids must be unique")
    if seeds.min() < 0 or seeds.max() >= num_nodes:
        raise ValueError("seed id out of range")
    blocks, frontier = [], seeds
    for f in fanouts:
        counts, chosen = _pick(start, end, col, frontier, int(f), rng)
        blk = _relabel(frontier, counts, chosen)
        blocks.append(blk)
        frontier = blk.src_nodes
    blocks = blocks[::-1]
    for i, b in enumerate(blocks):
        b.src_deg = np.zeros(b.num_src, np.int64) if i == 0 else blocks[i - 1].dst_deg
    return OSubgraph(seeds, blocks)
