"""Owner-sharded historical cache (TEST INFRASTRUCTURE ONLY) — SURVEY §8(e).

The reference's cache (histgnn/cache.py:226-369) is one process's state; it
defines no multi-GPU semantics. This restatement fixes them for P data-
parallel ranks, rank r training global batch P*s + r at step s, and is the
oracle the GPU's sharded cache (paper_2301_07482_b200/shardcache.py) is
bit-exact against:

- Ownership: node v belongs to owner o with bounds[o] <= v < bounds[o+1],
  the contiguous partition of comms.py:329-337 (distributed.owner_ranges).
  Owner o keeps, per cache layer, the reference's ring state for its own ids
  (row_of / admit_iter / row_owner / table / header / window), with the
  capacity rule of cache.py:79-101 applied to its own node count and, when a
  fixed capacity is given, ceil(capacity / P) rows.
- Lookups of step s are pure reads of the state after step s-1 (every rank
  at its own iteration number): fresh iff held and it - admit_iter <= t_stale
  (cache.py:103-129); an expired entry is a miss and is reported, not
  invalidated, so no rank's lookup can change another rank's answer. Hits and
  misses are counted by the rank that looked up.
- Commit, after the gradient exchange of step s, per owner: first every
  reported expiry (all ranks) is applied, counted once per entry still held
  (the eager invalidation of cache.py:106-115); then, for r = 0..P-1 (batch
  index order), rank r's update request is applied -- the admission rank is
  the whole batch's (k = floor(p_grad * n), norm ascending, ties by id,
  cache.py:188-204), the evictions / ring writes / retained refreshes touch
  only the owner's ids -- followed by end_iteration(P*s + r) (cache.py:330-334).
  Eviction and admission counters belong to the owner.

With P = 1 this is exactly histgnn's sequential cache: lookups precede the
update inside an iteration, so deferring the expiries to the commit changes
nothing (OTrainer with OHistCache).
"""

from __future__ import annotations

import math

import numpy as np

from .histcache import COUNTERS, OCachePolicy, _Ring


def owner_ranges(num_nodes: int, world: int) -> np.ndarray:
    """comms.py:329-337: the first num_nodes % world owners get one extra id."""
    base, extra = divmod(num_nodes, world)
    sizes = np.full(world, base, dtype=np.int64)
    sizes[:extra] += 1
    return np.concatenate([[0], np.cumsum(sizes)])


class OShardedCache:
    def __init__(self, num_nodes, layer_dims, policy: OCachePolicy, world, feature_rows=0,
                 refresh_retained=False, dtype=np.float32):
        self.num_nodes, self.world, self.policy = num_nodes, world, policy
        self.refresh_retained = refresh_retained
        self.bounds = owner_ranges(num_nodes, world)
        cap = None if policy.capacity is None else -(-policy.capacity // world)
        opol = OCachePolicy(policy.p_grad, policy.t_stale, cap)
        self.owners = []
        for o in range(world):
            n_o = int(self.bounds[o + 1] - self.bounds[o])
            self.owners.append({l + 1: _Ring(num_nodes, d, opol, dtype, n_cap=n_o) for l, d in enumerate(layer_dims)})
        self.layer_ids = list(range(1, len(layer_dims) + 1))
        self.feature_rows = int(feature_rows)
        self.feature_table = None
        self.feature_dim = None
        self.feature_row_of = np.full(num_nodes, -1, np.int64)

    def owner_of(self, ids):
        return np.searchsorted(self.bounds, np.asarray(ids), side="right") - 1

    def backfill_features(self, features, in_degrees):
        """Static layer-0 region, replicated on every rank (cache.py:338-351)."""
        if self.feature_rows <= 0:
            return
        deg = np.asarray(in_degrees)
        k = min(self.feature_rows, len(deg))
        top = np.lexsort((np.arange(len(deg)), -deg))[:k][::-1]
        self.feature_dim = features.shape[1]
        self.feature_table = features[top].copy()
        self.feature_row_of[top] = np.arange(k, dtype=np.int64)

    def view(self, rank: int) -> "RankView":
        return RankView(self, rank)

    def owner_counters(self, o: int) -> dict:
        tot = dict.fromkeys(COUNTERS, 0)
        for ring in self.owners[o].values():
            for k, v in ring.counters.items():
                tot[k] += v
        return tot

    def owner_valid(self, o: int) -> int:
        return sum(int((ring.row_of >= 0).sum()) for ring in self.owners[o].values())

    def commit(self, views) -> None:
        """Apply one step's expiries and update requests, views in rank order."""
        t = self.policy.t_stale
        for o, rings in enumerate(self.owners):
            lo, hi = self.bounds[o], self.bounds[o + 1]
            for l, ring in rings.items():
                exp = np.concatenate([v.expired.get(l, np.empty(0, np.int64)) for v in views])
                ring.invalidate(exp[(exp >= lo) & (exp < hi)])
            for v in views:
                for (l, nodes, computed, emb, norms, it) in v.requests:
                    owned = (nodes >= lo) & (nodes < hi)
                    rings[l].apply(nodes, computed, emb, norms, it, self.refresh_retained, owned)
                if v.iteration is not None and not math.isinf(t) and t >= 1 and (v.iteration + 1) % int(t) == 0:
                    for ring in rings.values():
                        ring.sweep()


class RankView:
    """What rank r's trainer sees during a step (OTrainer's `cache`): pure-read
    lookups against every owner, recorded expiries and update requests."""

    def __init__(self, shared: OShardedCache, rank: int):
        self.shared, self.rank = shared, rank
        self.num_nodes = shared.num_nodes
        self.refresh_retained = shared.refresh_retained
        self.policy = shared.policy
        self.counts = dict.fromkeys(COUNTERS, 0)
        self.expired = {}
        self.requests = []
        self.iteration = None

    def lookup(self, layer, ids, it):
        sh = self.shared
        ids = np.asarray(ids, np.int64)
        if layer == 0:
            r = sh.feature_row_of[ids]
            ok = r >= 0
            vals = (sh.feature_table[r[ok]].copy() if sh.feature_table is not None and ok.any()
                    else np.empty((0, sh.feature_dim or 0)))
            self.counts["feature_hits"] += int(ok.sum())
            self.counts["feature_misses"] += int((~ok).sum())
            return ids[ok], vals, ids[~ok]
        if layer not in sh.layer_ids:
            raise ValueError(f"no cache table for layer {layer}")
        own = sh.owner_of(ids)
        fresh = np.zeros(len(ids), bool)
        expired = np.zeros(len(ids), bool)
        dim = sh.owners[0][layer].dim
        vals = np.zeros((len(ids), dim), sh.owners[0][layer].dtype)
        for o in np.unique(own):
            m = own == o
            ok, v, ex = sh.owners[o][layer].peek(ids[m], it)
            fresh[m], expired[m] = ok, ex
            idx = np.flatnonzero(m)[ok]
            vals[idx] = v
        self.expired[layer] = np.concatenate([self.expired.get(layer, np.empty(0, np.int64)), ids[expired]])
        self.counts["hits"] += int(fresh.sum())
        self.counts["misses"] += int((~fresh).sum())
        return ids[fresh], vals[fresh], ids[~fresh]

    def update_cache(self, layer, batch_nodes, normal_nodes, embeddings, grad_norms, it):
        batch_nodes = np.asarray(batch_nodes, np.int64)
        if len(batch_nodes) == 0:
            return
        computed = np.isin(batch_nodes, np.asarray(normal_nodes, np.int64))
        self.requests.append((layer, batch_nodes, computed, np.asarray(embeddings),
                              np.asarray(grad_norms, np.float64), it))

    def end_iteration(self, it):
        self.iteration = it

    def counters(self):
        return dict(self.counts)

    def valid_entries(self):
        return 0
