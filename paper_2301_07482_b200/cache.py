"""Historical-embedding cache in HBM (drop-in for histgnn/cache.py).

Per hidden layer a ring-buffer table plus node->row (`row_of`), row->node
(`row_owner`) and admission stamps (`admit_iter`), all device resident; the
integer policy of the reference (cache.py:60-211) is executed by the
hg_cache_lookup / hg_cache_rank / hg_cache_write kernels. Host code keeps only
the capacity policy (first-use sizing cache.py:79-91, doubling cache.py:93-101,
sweep cadence cache.py:206-211,330-334). Counters live in a small int64
vector per layer on the device (csrc/hg_state.h) and are read back lazily.

Layer 0 is the static raw-feature region (cache.py:338-351): the top
`feature_rows` nodes by in-degree, HBM resident; its hits only save input I/O.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._state import (CTR_ADMISSIONS, CTR_CAPACITY, CTR_FORCED, CTR_GRAD_EVICT, CTR_HEADER, CTR_HITS,
                     CTR_MISSES, CTR_STALE_EVICT, CTR_VALID, CTR_VIOLATIONS, CTR_WIN_ADMIT, CTR_WIN_FORCED,
                     CTR_NWRITE, GCTR_FEATURE_HITS, GCTR_FEATURE_MISSES, GLOBAL_CTR_LEN, LAYER_CTR_LEN)
from .graphs import _np

COUNTER_NAMES = (
    "hits", "misses", "admissions", "gradient_evictions", "staleness_evictions",
    "forced_evictions", "staleness_violations", "feature_hits", "feature_misses",
)
_LAYER_IDX = {"hits": CTR_HITS, "misses": CTR_MISSES, "admissions": CTR_ADMISSIONS,
              "gradient_evictions": CTR_GRAD_EVICT, "staleness_evictions": CTR_STALE_EVICT,
              "forced_evictions": CTR_FORCED, "staleness_violations": CTR_VIOLATIONS}


def _it_dev(it: int, dev) -> torch.Tensor:
    return torch.tensor([int(it)], dtype=torch.int32, device=dev)


@dataclass(frozen=True)
class CachePolicy:
    """p_grad: admitted fraction per batch (smallest gradient norms first).
    t_stale: max age of a served entry in iterations; math.inf disables aging.
    capacity: rows per layer table; None sizes each table on first use.
    max_capacity: growth limit (extension, not in the reference: None = N as in
    cache.py:93-101); bounds HBM use at the papers100M shape, where doubling to
    N rows of 1 KB would need 113 GB per layer."""

    p_grad: float
    t_stale: float
    capacity: int | None = None
    max_capacity: int | None = None

    def __post_init__(self):
        if not 0.0 <= self.p_grad <= 1.0:
            raise ValueError(f"p_grad must be in [0, 1], got {self.p_grad}")
        if not (self.t_stale >= 0):
            raise ValueError(f"t_stale must be >= 0 or inf, got {self.t_stale}")
        if self.capacity is not None and self.capacity < 1:
            raise ValueError("capacity must be >= 1 when given")
        if self.max_capacity is not None and self.max_capacity < 1:
            raise ValueError("max_capacity must be >= 1 when given")
        if self.capacity is not None and self.max_capacity is not None and self.capacity > self.max_capacity:
            raise ValueError(f"capacity {self.capacity} exceeds max_capacity {self.max_capacity}")


class _LayerCache:
    def __init__(self, num_nodes, dim, policy, dtype, device, min_capacity=64):
        self.num_nodes = num_nodes
        self.dim = dim
        self.policy = policy
        self.dtype = dtype
        self.device = device
        self.min_capacity = min_capacity
        self._capacity = 0
        self._cap_on_device = False   # True once sweeps may grow the capacity on the device
        self.rows_alloc = 0
        self.table = None
        self.row_owner_dev = None
        self.row_of_dev = torch.full((num_nodes,), -1, dtype=torch.int32, device=device)
        self.admit_iter_dev = torch.zeros(num_nodes, dtype=torch.int32, device=device)
        self.ctr = torch.zeros(LAYER_CTR_LEN, dtype=torch.int64, device=device)

    @property
    def capacity(self) -> int:
        """Logical ring size (cache.py:79-101). Device-resident once sweeps run
        on the device (then reading it synchronises)."""
        if self._cap_on_device:
            self._capacity = int(self.ctr[CTR_CAPACITY].item())
        return self._capacity

    @capacity.setter
    def capacity(self, v: int):
        self._capacity = int(v)

    def limit(self) -> int:
        """Growth limit: N (cache.py:93-101), or the policy's max_capacity."""
        limit = max(self.num_nodes, 1)
        if self.policy.max_capacity is not None:
            limit = min(limit, self.policy.max_capacity)
        return limit

    # ---- reference-visible state (numpy views) ----
    @property
    def row_of(self):
        return _np(self.row_of_dev).astype(np.int64)

    @property
    def admit_iter(self):
        return _np(self.admit_iter_dev).astype(np.int64)

    @property
    def row_owner(self):
        return (None if self.row_owner_dev is None
                else _np(self.row_owner_dev[: self.capacity]).astype(np.int64))

    @property
    def table_view(self):
        """The logical ring rows [capacity x dim] (the allocation may be larger)."""
        return None if self.table is None else self.table[: self.capacity]

    @property
    def header(self):
        return int(self.ctr[CTR_HEADER].item())

    @property
    def window_admissions(self):
        return int(self.ctr[CTR_WIN_ADMIT].item())

    @property
    def window_forced(self):
        return int(self.ctr[CTR_WIN_FORCED].item())

    @property
    def counters(self):
        c = self.ctr.cpu().tolist()
        return {k: c[i] for k, i in _LAYER_IDX.items()}

    def _t_stale(self):
        return float(self.policy.t_stale)

    def first_capacity(self, first_admits: int) -> int:
        """cache.py:79-91."""
        p = self.policy
        if p.capacity is not None:
            cap = p.capacity
        elif math.isinf(p.t_stale):
            cap = self.num_nodes
        else:
            window = max(1, int(p.t_stale))
            cap = 2 * max(1, first_admits) * window
            cap = int(np.clip(cap, self.min_capacity, max(self.num_nodes, 1)))
        if p.max_capacity is not None:
            cap = min(cap, p.max_capacity)
        return max(1, cap)

    HEADROOM_BYTES = 8 << 30   # ring preallocation budget per layer (growth without reallocation)

    def _rows_for(self, cap: int) -> int:
        """Rows actually allocated for a logical capacity: as many as the
        byte budget allows (never past N, never below 4x cap when N allows),
        so the doublings of cache.py:93-101 only change the device-resident
        capacity, not the table pointer (a captured CUDA graph stays valid).
        Never past the growth limit (max_capacity bounds HBM use)."""
        row_bytes = max(self.dim * torch.tensor([], dtype=self.dtype).element_size(), 1)
        return max(cap, min(self.limit(), max(4 * cap, self.HEADROOM_BYTES // row_bytes)))

    def allocate(self, first_admits: int):
        self.capacity = self.first_capacity(first_admits)
        self.rows_alloc = self._rows_for(self.capacity)
        self.table = torch.zeros((self.rows_alloc, self.dim), dtype=self.dtype, device=self.device)
        self.row_owner_dev = torch.full((self.rows_alloc,), -1, dtype=torch.int32, device=self.device)
        self.ctr[CTR_CAPACITY] = self.capacity

    def _grow(self):
        """cache.py:93-101 — double (up to N), rows kept in place."""
        limit = self.limit()
        if self.table is None or self.capacity >= limit:
            return
        new_cap = min(self.capacity * 2, limit)
        if new_cap > self.rows_alloc:   # out of headroom: reallocate (a captured graph is re-captured)
            rows = self._rows_for(new_cap)
            table = torch.zeros((rows, self.dim), dtype=self.dtype, device=self.device)
            table[: self.capacity] = self.table[: self.capacity]
            owner = torch.full((rows,), -1, dtype=torch.int32, device=self.device)
            owner[: self.capacity] = self.row_owner_dev[: self.capacity]
            self.table, self.row_owner_dev, self.rows_alloc = table, owner, rows
        self.capacity = new_cap
        self.ctr[CTR_CAPACITY] = new_cap

    def sweep(self, stream=None):
        """cache.py:206-211. When the preallocated rows already reach the
        growth limit, no doubling can need a reallocation: the whole sweep
        (grow test, capacity doubling, window/header reset) runs as one device
        kernel, with no host read. Otherwise one host read of the window
        counters decides the growth on the host."""
        if self.table is not None and self.rows_alloc >= self.limit():
            self._cap_on_device = True
            _lib.call("hg_cache_sweep", _lib.ptr(self.ctr), self.limit(), _lib.stream_ptr(stream))
            return
        wa, wf = self.ctr[CTR_WIN_ADMIT:CTR_WIN_FORCED + 1].cpu().tolist()
        if wa and wf > 0.01 * wa:
            self._grow()
        self.ctr[CTR_WIN_ADMIT] = 0
        self.ctr[CTR_WIN_FORCED] = 0
        self.ctr[CTR_HEADER] = 0

    # ---- device ops on (live list, src ids) views ----
    def lookup_dev(self, n_dev, n_max, live, src_nodes, n_src_max, it_dev, hit_flag, hit_row, stream):
        if self.row_owner_dev is None:
            # nothing admitted yet: every probe misses, no state to invalidate
            owner = self._dummy_owner()
        else:
            owner = self.row_owner_dev
        _lib.call("hg_cache_lookup", _lib.ptr(n_dev), n_max, _lib.ptr(live), _lib.ptr(src_nodes), n_src_max,
                  _lib.ptr(self.row_of_dev), _lib.ptr(self.admit_iter_dev), _lib.ptr(owner), _lib.ptr(it_dev),
                  self._t_stale(), _lib.ptr(hit_flag), _lib.ptr(hit_row), _lib.ptr(self.ctr), stream)

    def injection(self, hit_flag, hit_row):
        """The forward's Injection for this layer's hits (None before any admission)."""
        from .nn import Injection
        return None if self.table is None else Injection(hit_flag, hit_row, self.table)

    def _dummy_owner(self):
        if getattr(self, "_dummy", None) is None:
            self._dummy = torch.full((1,), -1, dtype=torch.int32, device=self.device)
        return self._dummy

    def update_dev(self, n_dev, n_max, live, src_nodes, norms, computed_flag, emb, it_dev, refresh_retained,
                   stream, allow_alloc=True, mark=None):
        """cache.py:188-204 for the n_dev[0] live nodes (n_max host bound).
        The ring table is allocated on first use (cache.py:79-91), which reads
        the first write count back to the host (allow_alloc=False forbids it,
        e.g. while a CUDA graph is being captured)."""
        if n_max <= 0:
            return
        sb = _lib.query("hg_cache_update_scratch_bytes", n_max)
        scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        owner = self.row_owner_dev if self.row_owner_dev is not None else self._dummy_owner()
        _lib.call("hg_cache_rank", _lib.ptr(n_dev), n_max, float(self.policy.p_grad), _lib.ptr(live),
                  _lib.ptr(src_nodes), _lib.ptr(norms), _lib.ptr(computed_flag), _lib.ptr(self.row_of_dev),
                  _lib.ptr(owner), _lib.ptr(self.ctr), _lib.ptr(scratch), sb, stream)
        if mark is not None:
            mark("ranked")
        if self.table is None:
            if not allow_alloc:
                raise RuntimeError("cache table must be allocated before graph capture")
            n_write = int(self.ctr[CTR_NWRITE].item())   # first use only: size the ring
            if n_write == 0:
                return
            self.allocate(n_write)
        row_words = self.dim * (self.table.element_size() // 4)   # rows are copied as 4-byte words
        _lib.call("hg_cache_write", n_max, self.rows_alloc, row_words, _lib.ptr(it_dev), self._t_stale(),
                  int(bool(refresh_retained)), _lib.ptr(live), _lib.ptr(emb), _lib.ptr(self.table),
                  _lib.ptr(self.row_of_dev), _lib.ptr(self.row_owner_dev), _lib.ptr(self.admit_iter_dev),
                  _lib.ptr(self.ctr), _lib.ptr(scratch), sb, stream)

    def valid_entries(self) -> int:
        return int(self.ctr[CTR_VALID].item())

    def check_integrity(self):
        row_of = self.row_of
        live = np.flatnonzero(row_of >= 0)
        rows = row_of[live]
        assert len(np.unique(rows)) == len(rows), "two nodes share a row"
        owner = self.row_owner
        if owner is not None:
            np.testing.assert_array_equal(owner[rows], live)
            owned = np.flatnonzero(owner >= 0)
            np.testing.assert_array_equal(row_of[owner[owned]], owned)
        assert self.valid_entries() == len(live), "device valid-entry counter drifted"


class HistCache:
    """Per-layer embedding caches (layers 1..L) plus the layer-0 feature region."""

    def __init__(self, num_nodes: int, layer_dims, policy: CachePolicy, feature_dim: int | None = None,
                 feature_rows: int = 0, refresh_retained: bool = False, dtype=np.float32, device=None):
        _lib.require_cuda()
        self.device = torch.device(device or "cuda")
        self.num_nodes = num_nodes
        self.policy = policy
        self.refresh_retained = refresh_retained
        tdtype = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[np.dtype(dtype)]
        self.np_dtype = np.dtype(dtype)
        self.layers = {l + 1: _LayerCache(num_nodes, dim, policy, tdtype, self.device)
                       for l, dim in enumerate(layer_dims)}
        self.feature_rows = int(feature_rows)
        self.feature_dim = feature_dim
        self.feature_table = None              # device tensor [k, d] (features dtype)
        self.feature_row_of_dev = torch.full((num_nodes,), -1, dtype=torch.int32, device=self.device)
        self.gctr = torch.zeros(GLOBAL_CTR_LEN, dtype=torch.int64, device=self.device)
        self._ops = 0      # numpy-API calls that moved counters (engine metric snapshots re-sync on change)

    sharded = False

    def begin_step(self, it_dev, stream) -> None:
        """Data-parallel hook before a step's lookups (the owner-sharded cache
        waits for its peers' commits there); a process-local cache has none."""

    def commit(self, stream) -> None:
        """Data-parallel hook after a step's updates; nothing to do here."""

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    @property
    def feature_table_dev(self):
        """The device feature region [k x d] (None before backfill)."""
        return self.feature_table

    @property
    def feature_row_of(self):
        return _np(self.feature_row_of_dev).astype(np.int64)

    def _layer(self, layer: int) -> _LayerCache:
        if layer not in self.layers:
            raise ValueError(f"no cache table for layer {layer}")
        return self.layers[layer]

    # ------------------------------------------------------------- lookups

    def lookup(self, layer: int, ids, current_iter: int):
        """Returns (hit_ids, hit_rows, miss_ids) as numpy, like the reference;
        expired entries are invalidated and reported as misses."""
        ids = np.asarray(ids, dtype=np.int64)
        dev = self.device
        self._ops += 1
        if layer == 0:
            idx = torch.as_tensor(ids, device=dev)
            rows = self.feature_row_of_dev[idx]
            ok = rows >= 0
            nh = int(ok.sum().item())
            self.gctr[GCTR_FEATURE_HITS] += nh
            self.gctr[GCTR_FEATURE_MISSES] += len(ids) - nh
            okn = _np(ok)
            ft = self.feature_table_dev
            vals = (_np(ft[rows[ok].long()]) if ft is not None and nh
                    else np.empty((0, self.feature_dim or 0)))
            return ids[okn], vals, ids[~okn]
        lc = self._layer(layer)
        n = len(ids)
        src = torch.as_tensor(ids.astype(np.int32), device=dev)
        live = torch.arange(n, dtype=torch.int32, device=dev)
        n_dev = torch.tensor([n], dtype=torch.int32, device=dev)
        flag = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        hrow = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        if n:
            lc.lookup_dev(n_dev, n, live, src, n, _it_dev(current_iter, dev), flag, hrow, _lib.stream_ptr())
        f = _np(flag[:n]).astype(bool)
        hit_rows = (_np(lc.table[hrow[:n][flag[:n].bool()].long()]) if f.any() and lc.table is not None
                    else np.empty((0, lc.dim), dtype=self.np_dtype))
        return ids[f], hit_rows, ids[~f]

    # ------------------------------------------------------------- updates

    def update_cache(self, layer: int, batch_nodes, normal_nodes, embeddings, grad_norms, current_iter: int) -> None:
        """Admission/eviction for one layer after a finished iteration (cache.py:289-322)."""
        batch_nodes = np.asarray(batch_nodes, dtype=np.int64)
        normal_nodes = np.asarray(normal_nodes, dtype=np.int64)
        self._ops += 1
        if len(batch_nodes) == 0:
            return
        if embeddings.shape[0] != len(batch_nodes):
            raise ValueError("embeddings rows must align with batch_nodes")
        if len(grad_norms) != len(batch_nodes):
            raise ValueError("grad_norms must align with batch_nodes")
        lc = self._layer(layer)
        dev = self.device
        n = len(batch_nodes)
        computed = np.isin(batch_nodes, normal_nodes).astype(np.uint8)
        emb = torch.as_tensor(np.asarray(embeddings), device=dev).to(lc.dtype).contiguous()
        lc.update_dev(torch.tensor([n], dtype=torch.int32, device=dev), n,
                      torch.arange(n, dtype=torch.int32, device=dev),
                      torch.as_tensor(batch_nodes.astype(np.int32), device=dev),
                      torch.as_tensor(np.asarray(grad_norms, dtype=np.float64), device=dev),
                      torch.as_tensor(computed, device=dev), emb, _it_dev(current_iter, dev), self.refresh_retained,
                      _lib.stream_ptr())

    def sweep_staleness(self, current_iter: int | None = None) -> None:
        for lc in self.layers.values():
            lc.sweep()

    def end_iteration(self, current_iter: int) -> None:
        t = self.policy.t_stale
        if not math.isinf(t) and t >= 1 and (current_iter + 1) % int(t) == 0:
            self.sweep_staleness(current_iter)

    # ------------------------------------------------------- feature region

    def backfill_features(self, features, in_degrees=None, graph=None) -> None:
        """Fill the layer-0 region with the highest in-degree nodes' rows,
        ordered so the top-degree node occupies the final row (one-shot).
        `features` may be a host array or a device tensor; degrees come from
        `graph` (device, preferred) or `in_degrees`."""
        if self.feature_rows <= 0:
            return
        if self.feature_table is not None:
            raise ValueError("feature region already backfilled")
        dev = self.device
        if graph is not None:
            start, end, n = graph.start, graph.end, graph.num_nodes
        else:
            deg = torch.as_tensor(np.asarray(in_degrees, dtype=np.int64), device=dev)
            start, end, n = torch.zeros_like(deg), deg, len(deg)
        k = min(self.feature_rows, n)
        chosen = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
        sb = _lib.query("hg_degree_order_scratch_bytes", n)
        scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        _lib.call("hg_feature_region", _lib.ptr(start), _lib.ptr(end), n, k, _lib.ptr(chosen),
                  _lib.ptr(self.feature_row_of_dev), _lib.ptr(scratch), sb, _lib.stream_ptr())
        feats = (features if isinstance(features, torch.Tensor) or hasattr(features, "index_select")
                 else torch.as_tensor(np.asarray(features)))
        self.feature_dim = int(feats.shape[1])
        if feats.device.type == "cuda":
            self.feature_table = feats.index_select(0, chosen[:k].long()).contiguous()
        else:  # host (possibly pinned) source: gather on the host side once
            self.feature_table = feats[chosen[:k].cpu().long()].contiguous().to(dev)

    # -------------------------------------------------------------- metrics

    def counters(self) -> dict:
        total = dict.fromkeys(COUNTER_NAMES, 0)
        for lc in self.layers.values():
            for k, v in lc.counters.items():
                total[k] += v
        g = self.gctr.cpu().tolist()
        total["feature_hits"] += g[GCTR_FEATURE_HITS]
        total["feature_misses"] += g[GCTR_FEATURE_MISSES]
        return total

    def counters_vector(self) -> torch.Tensor:
        """Device snapshot of every counter (for async readback)."""
        return torch.cat([lc.ctr for lc in self.layers.values()] + [self.gctr])

    def valid_entries(self) -> int:
        return sum(lc.valid_entries() for lc in self.layers.values())

    def check_integrity(self) -> None:
        for lc in self.layers.values():
            lc.check_integrity()
