"""Historical-embedding cache (oracle restatement of histgnn/cache.py).

Per hidden layer: a ring-buffer table plus node->row / row->node maps and an
admission-iteration stamp; plus a static layer-0 raw-feature region.
Restated behaviour (integer decisions are bit-exact targets for the GPU cache):
- lookup          cache.py:103-129  inclusive staleness, expired entries are
                                    invalidated on the spot, hits copied in
                                    query order; counters hits/misses/
                                    staleness_evictions/staleness_violations.
- _release        cache.py:131-137
- _write          cache.py:139-173  ring rows (header+i) % cap; the n >= cap
                                    branch keeps only the trailing cap writes.
- _count_overwrites cache.py:175-186 forced iff age < t_stale (all if inf).
- update          cache.py:188-204  k = floor(p*n), rank by (norm, id),
                                    gradient-evict non-admitted cached nodes,
                                    write admitted computed nodes in rank order.
- _allocate/_grow cache.py:79-101; sweep cache.py:206-211;
  end_iteration   cache.py:330-334; backfill_features cache.py:338-351.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

COUNTERS = ("hits", "misses", "admissions", "gradient_evictions",
            "staleness_evictions", "forced_evictions", "staleness_violations",
            "feature_hits", "feature_misses")


@dataclass(frozen=True)
class OCachePolicy:
    p_grad: float
    t_stale: float
    capacity: int | None = None

    def __post_init__(self):
        if not 0.0 <= self.p_grad <= 1.0:
            raise ValueError(f"p_grad must be in [0, 1], got {self.p_grad}")
        if not (self.t_stale >= 0):
            raise ValueError(f"t_stale must be >= 0 or inf, got {self.t_stale}")
        if self.capacity is not None and self.capacity < 1:
            raise ValueError("capacity must be >= 1 when given")


class _Ring:
    """n = id space (row_of is indexed by global id); n_cap = the node count
    the capacity rule clips to and growth stops at (cache.py:79-101): the
    whole graph, or an owner's range in the sharded cache (oracle/shardcache.py)."""

    def __init__(self, n, dim, policy, dtype, min_capacity=64, n_cap=None):
        self.n, self.dim, self.policy, self.dtype = n, dim, policy, dtype
        self.n_cap = n if n_cap is None else n_cap
        self.min_capacity = min_capacity
        self.capacity, self.header = 0, 0
        self.table = None
        self.row_owner = None
        self.row_of = np.full(n, -1, np.int64)
        self.admit_iter = np.zeros(n, np.int64)
        self.counters = dict.fromkeys(COUNTERS, 0)
        self.window_admissions = 0
        self.window_forced = 0

    @property
    def _inf(self):
        return math.isinf(self.policy.t_stale)

    def _first_capacity(self, first_admits):
        p = self.policy
        if p.capacity is not None:
            cap = p.capacity
        elif self._inf:
            cap = self.n_cap
        else:
            cap = 2 * max(1, first_admits) * max(1, int(p.t_stale))
            cap = int(min(max(cap, self.min_capacity), max(self.n_cap, 1)))
        self.capacity = max(1, cap)
        self.table = np.zeros((self.capacity, self.dim), self.dtype)
        self.row_owner = np.full(self.capacity, -1, np.int64)

    def grow(self):
        if self.table is None or self.capacity >= self.n_cap:
            return
        cap = min(2 * self.capacity, max(self.n_cap, 1))
        t = np.zeros((cap, self.dim), self.dtype)
        t[:self.capacity] = self.table
        o = np.full(cap, -1, np.int64)
        o[:self.capacity] = self.row_owner
        self.table, self.row_owner, self.capacity = t, o, cap

    def lookup(self, ids, it):
        r = self.row_of[ids]
        ok = r >= 0
        if not self._inf:
            age = it - self.admit_iter[ids]
            stale = ok & (age > self.policy.t_stale)
            if stale.any():
                self.row_owner[r[stale]] = -1
                self.row_of[ids[stale]] = -1
                self.counters["staleness_evictions"] += int(stale.sum())
            ok = ok & ~stale
        hit = ids[ok]
        vals = (self.table[r[ok]].copy() if self.table is not None and ok.any()
                else np.empty((0, self.dim), self.dtype))
        if not self._inf and ok.any():
            if int((it - self.admit_iter[hit]).max()) > self.policy.t_stale:
                self.counters["staleness_violations"] += 1
        self.counters["hits"] += len(hit)
        self.counters["misses"] += int((~ok).sum())
        return hit, vals, ids[~ok]

    def _drop(self, nodes):
        r = self.row_of[nodes]
        m = r >= 0
        self.row_owner[r[m]] = -1
        self.row_of[nodes[m]] = -1
        return int(m.sum())

    def _overwrite_ages(self, ages):
        forced = len(ages) if self._inf else int((ages < self.policy.t_stale).sum())
        self.counters["forced_evictions"] += forced
        self.window_forced += forced
        self.counters["staleness_evictions"] += len(ages) - forced

    def write(self, nodes, vals, it):
        if len(nodes) == 0:
            return
        if self.table is None:
            self._first_capacity(len(nodes))
        cap = self.capacity
        if len(nodes) >= cap:
            nodes, vals = nodes[-cap:], vals[-cap:]
            self._drop(nodes)
            held = np.flatnonzero(self.row_owner >= 0)
            if len(held):
                owners = self.row_owner[held]
                self._overwrite_ages(it - self.admit_iter[owners])
                self.row_of[owners] = -1
                self.row_owner[held] = -1
            rows = np.arange(len(nodes), dtype=np.int64)
            self.header = len(nodes) % cap
        else:
            self._drop(nodes)
            rows = (self.header + np.arange(len(nodes), dtype=np.int64)) % cap
            prev = self.row_owner[rows]
            prev = prev[prev >= 0]
            if len(prev):
                self._overwrite_ages(it - self.admit_iter[prev])
                self.row_of[prev] = -1
            self.header = (self.header + len(nodes)) % cap
        self.table[rows] = vals.astype(self.dtype, copy=False)
        self.row_owner[rows] = nodes
        self.row_of[nodes] = rows
        self.admit_iter[nodes] = it
        self.counters["admissions"] += len(nodes)
        self.window_admissions += len(nodes)

    def update(self, nodes, computed, emb, norms, it, refresh_retained):
        n = len(nodes)
        k = int(math.floor(self.policy.p_grad * n))
        rank = np.lexsort((nodes, norms))        # norm ascending, ties by node id
        admitted = np.zeros(n, bool)
        admitted[rank[:k]] = True
        losers = ~admitted & (self.row_of[nodes] >= 0)
        if losers.any():
            self.counters["gradient_evictions"] += self._drop(nodes[losers])
        wpos = rank[:k][computed[rank[:k]]]      # admit-rank order
        self.write(nodes[wpos], emb[wpos], it)
        if refresh_retained:
            kept = nodes[admitted & ~computed]
            kept = kept[self.row_of[kept] >= 0]
            self.admit_iter[kept] = it

    # ---- split form for the owner-sharded cache (oracle/shardcache.py) ----
    def peek(self, ids, it):
        """Pure-read lookup: (fresh mask, rows of the fresh ids in input
        order, expired mask). No state or counter changes."""
        r = self.row_of[ids]
        ok = r >= 0
        expired = np.zeros(len(ids), bool)
        if not self._inf:
            expired = ok & (it - self.admit_iter[ids] > self.policy.t_stale)
            ok = ok & ~expired
        vals = (self.table[r[ok]].copy() if self.table is not None and ok.any()
                else np.empty((0, self.dim), self.dtype))
        return ok, vals, expired

    def invalidate(self, ids):
        """Apply expiries found by pure-read lookups (counted once per entry
        still held, as the eager lookup of cache.py:106-115 counts them)."""
        if self.table is not None and len(ids):
            self.counters["staleness_evictions"] += self._drop(np.unique(np.asarray(ids, np.int64)))

    def apply(self, nodes, computed, emb, norms, it, refresh_retained, owned):
        """update() with the batch-wide admission rank, applied only to the
        `owned` members (an owner's share of a peer's request)."""
        n = len(nodes)
        k = int(math.floor(self.policy.p_grad * n))
        rank = np.lexsort((nodes, norms))
        admitted = np.zeros(n, bool)
        admitted[rank[:k]] = True
        losers = ~admitted & owned & (self.row_of[nodes] >= 0)
        if losers.any():
            self.counters["gradient_evictions"] += self._drop(nodes[losers])
        top = rank[:k]
        wpos = top[computed[top] & owned[top]]
        self.write(nodes[wpos], emb[wpos], it)
        if refresh_retained:
            kept = nodes[admitted & ~computed & owned]
            kept = kept[self.row_of[kept] >= 0]
            self.admit_iter[kept] = it

    def sweep(self):
        if self.window_admissions and self.window_forced > 0.01 * self.window_admissions:
            self.grow()
        self.window_admissions = self.window_forced = 0
        self.header = 0


class OHistCache:
    def __init__(self, num_nodes, layer_dims, policy, feature_dim=None,
                 feature_rows=0, refresh_retained=False, dtype=np.float32):
        self.num_nodes = num_nodes
        self.policy = policy
        self.refresh_retained = refresh_retained
        self.layers = {i + 1: _Ring(num_nodes, d, policy, dtype) for i, d in enumerate(layer_dims)}
        self.feature_rows = int(feature_rows)
        self.feature_dim = feature_dim
        self.feature_table = None
        self.feature_row_of = np.full(num_nodes, -1, np.int64)
        self.fcount = {"feature_hits": 0, "feature_misses": 0}

    def _ring(self, layer):
        if layer not in self.layers:
            raise ValueError(f"no cache table for layer {layer}")
        return self.layers[layer]

    def lookup(self, layer, ids, it):
        ids = np.asarray(ids, np.int64)
        if layer == 0:
            r = self.feature_row_of[ids]
            ok = r >= 0
            vals = (self.feature_table[r[ok]].copy() if self.feature_table is not None and ok.any()
                    else np.empty((0, self.feature_dim or 0)))
            self.fcount["feature_hits"] += int(ok.sum())
            self.fcount["feature_misses"] += int((~ok).sum())
            return ids[ok], vals, ids[~ok]
        return self._ring(layer).lookup(ids, it)

    def update_cache(self, layer, batch_nodes, normal_nodes, embeddings, grad_norms, it):
        batch_nodes = np.asarray(batch_nodes, np.int64)
        normal_nodes = np.asarray(normal_nodes, np.int64)
        if len(batch_nodes) == 0:
            return
        if embeddings.shape[0] != len(batch_nodes):
            raise ValueError("embeddings rows must align with batch_nodes")
        if len(grad_norms) != len(batch_nodes):
            raise ValueError("grad_norms must align with batch_nodes")
        computed = np.isin(batch_nodes, normal_nodes)
        self._ring(layer).update(batch_nodes, computed, embeddings,
                                 np.asarray(grad_norms, np.float64), it,
                                 self.refresh_retained)

    def sweep_staleness(self, it=None):
        for r in self.layers.values():
            r.sweep()

    def end_iteration(self, it):
        t = self.policy.t_stale
        if not math.isinf(t) and t >= 1 and (it + 1) % int(t) == 0:
            self.sweep_staleness(it)

    def backfill_features(self, features, in_degrees):
        if self.feature_rows <= 0:
            return
        if self.feature_table is not None:
            raise ValueError("feature region already backfilled")
        deg = np.asarray(in_degrees)
        k = min(self.feature_rows, len(deg))
        top = np.lexsort((np.arange(len(deg)), -deg))[:k][::-1]
        self.feature_dim = features.shape[1]
        self.feature_table = features[top].copy()
        self.feature_row_of[top] = np.arange(k, dtype=np.int64)

    def counters(self):
        tot = dict.fromkeys(COUNTERS, 0)
        for r in self.layers.values():
            for k, v in r.counters.items():
                tot[k] += v
        for k, v in self.fcount.items():
            tot[k] += v
        return tot

    def valid_entries(self):
        return sum(int((r.row_of >= 0).sum()) for r in self.layers.values())
