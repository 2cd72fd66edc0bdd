"""Owner-sharded historical cache across the ranks of one box.

Each rank owns, per cache layer, the reference's ring state (cache.py:60-211)
for the node ids of its contiguous range [bounds[r], bounds[r+1])
(comms.py:329-337) in one CUDA-IPC allocation that every peer maps: row_of /
admit_iter indexed by id - bounds[r], row_owner, the ring table, plus this
rank's per-step request area (admission actions, expired ids, header). The
semantics (oracle/shardcache.py, the oracle the tests pin this against):

  lookups   pure reads of the owners' state after the previous step, at the
            rank's own iteration; hits are injected straight from the owner's
            ring (one-sided NVLink reads on a multi-GPU box); expiries are
            reported
  request   the batch-wide admission rank, published in the rank's memory
  commit    after a device barrier: each owner applies every rank's expiries,
            then the P requests in rank (= batch index) order restricted to
            its ids, each followed by that batch's end_iteration sweep; a
            second barrier orders the commit before the next step's lookups

All of it is stream-ordered device work (hg_shard_cache.cu), so the step
stays capturable in a CUDA graph. With P = 1 the trainer is bit-identical to
the per-process cache.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from ._state import CTR_VALID, GLOBAL_CTR_LEN, LAYER_CTR_LEN
from .cache import CachePolicy, HistCache, _LayerCache
from .distributed import owner_ranges
from .graphs import _np
from .sharding import _DevBuf

_HDR_WORDS = 8


class ShardingUnavailable(RuntimeError):
    """Raised on every rank when some rank cannot map its peers' cache shards."""


def _align(n: int, a: int = 256) -> int:
    return (n + a - 1) // a * a


class ShardedLayerCache(_LayerCache):
    """One cache layer: this rank's shard (owner state + request area, views
    into the IPC block) and the peers' pointer tables."""

    def __init__(self, owner: "ShardedHistCache", layer: int, dim: int, n_req: int):
        # no base __init__: the owner state is n_owned (not N) long and lives in IPC memory
        self.owner, self.layer = owner, layer
        self.num_nodes = owner.num_nodes
        self.dim, self.policy, self.dtype, self.device = dim, owner.policy, torch.float32, owner.device
        self.min_capacity = 64
        self._capacity, self._cap_on_device = 0, True
        self.n_req = int(n_req)
        self.lo, self.hi = int(owner.bounds[owner.rank]), int(owner.bounds[owner.rank + 1])
        self.n_owned = self.hi - self.lo
        P = owner.world
        lim = self.n_owned
        if self.policy.max_capacity is not None:
            lim = min(lim, -(-self.policy.max_capacity // P))
        self.limit_rows = max(1, lim)
        self.cap_fixed = -1 if self.policy.capacity is None else min(-(-self.policy.capacity // P), self.limit_rows)
        self.rows_alloc = self.limit_rows
        self.ctr = torch.zeros(LAYER_CTR_LEN, dtype=torch.int64, device=self.device)
        if self.limit_rows >= 1 << 26 or owner.world > 32:
            raise ValueError("the sharded cache encodes hits as owner << 26 | row: rings < 2^26 rows, <= 32 ranks")
        # hits are injected straight from the owners' rings (hg_inject_rows_sharded);
        # `table` is a placeholder so a captured step sees a stable key
        self.table = torch.zeros((1, dim), dtype=torch.float32, device=self.device)

    # section sizes of this layer in the IPC block (bytes)
    def sections(self):
        n_o, lim, q, d = max(1, self.n_owned), self.limit_rows, max(1, self.n_req), self.dim
        return [("row_of", n_o * 4), ("admit_iter", n_o * 4), ("row_owner", lim * 4), ("ring", lim * d * 4),
                ("req_id", q * 4), ("req_act", q), ("req_src", q * 4), ("req_emb", q * d * 4), ("exp_ids", q * 4),
                ("hdr", _HDR_WORDS * 8)]

    def bind(self, base: int, offs: dict, peers: list):
        """Views of this rank's sections; `peers[r]` = rank r's block base."""
        dev, lim, d = self.device, self.limit_rows, self.dim
        n_o, q = max(1, self.n_owned), max(1, self.n_req)

        def view(name, shape, ts):
            return torch.as_tensor(_DevBuf(base + offs[name], shape, ts), device=dev)

        self.row_of_dev = view("row_of", (n_o,), "<i4")
        self.admit_iter_dev = view("admit_iter", (n_o,), "<i4")
        self.row_owner_dev = view("row_owner", (lim,), "<i4")
        self.ring = view("ring", (lim, d), "<f4")
        self.req_id = view("req_id", (q,), "<i4")
        self.req_act = view("req_act", (q,), "|u1")
        self.req_src = view("req_src", (q,), "<i4")
        self.req_emb = view("req_emb", (q, d), "<f4")
        self.exp_ids = view("exp_ids", (q,), "<i4")
        self.hdr = view("hdr", (_HDR_WORDS,), "<i8")
        self.row_of_dev.fill_(-1)
        self.admit_iter_dev.zero_()
        self.row_owner_dev.fill_(-1)
        self.ring.zero_()
        self.hdr.zero_()

        def table(name):
            return torch.tensor([p + offs[name] for p in peers], dtype=torch.int64, device=dev)

        self.peer_row_of, self.peer_admit, self.peer_ring = table("row_of"), table("admit_iter"), table("ring")
        self.peer_exp, self.peer_hdr = table("exp_ids"), table("hdr")
        self.peer_req = [(p + offs["hdr"], p + offs["req_id"], p + offs["req_act"], p + offs["req_emb"])
                         for p in peers]

    # ---- reference-visible state ----
    @property
    def row_of(self):
        out = np.full(self.num_nodes, -1, dtype=np.int64)
        out[self.lo:self.hi] = _np(self.row_of_dev)[:self.n_owned]
        return out

    @property
    def admit_iter(self):
        out = np.zeros(self.num_nodes, dtype=np.int64)
        out[self.lo:self.hi] = _np(self.admit_iter_dev)[:self.n_owned]
        return out

    def limit(self) -> int:
        return self.limit_rows

    def first_capacity(self, first_admits: int) -> int:
        raise RuntimeError("the sharded cache sizes its ring on the device (hg_cache_apply)")

    def _grow(self):
        raise RuntimeError("the sharded cache grows at its device-side sweeps")

    def sweep(self, stream=None):
        raise RuntimeError("the sharded cache sweeps inside its commit (end_iteration per batch)")

    # ---- the step ----
    def reset_dev(self, it_dev, stream):
        _lib.call("hg_cache_request_reset", _lib.ptr(self.hdr), _lib.ptr(it_dev), stream)

    def lookup_dev(self, n_dev, n_max, live, src_nodes, n_src_max, it_dev, hit_flag, hit_row, stream):
        if n_src_max > self.n_req:
            raise ValueError(f"layer {self.layer}: {n_src_max} sources exceed the request area ({self.n_req})")
        o = self.owner
        _lib.call("hg_cache_lookup_sharded", _lib.ptr(n_dev), n_max, _lib.ptr(live), _lib.ptr(src_nodes), n_src_max,
                  o.world, _lib.ptr(o.bounds_dev), _lib.ptr(self.peer_row_of), _lib.ptr(self.peer_admit),
                  _lib.ptr(it_dev), float(self.policy.t_stale), _lib.ptr(hit_flag), _lib.ptr(hit_row),
                  _lib.ptr(self.exp_ids), _lib.ptr(self.hdr), _lib.ptr(self.ctr), stream)

    def injection(self, hit_flag, hit_row):
        from .nn import Injection
        return Injection(hit_flag, hit_row, None, tables=self.peer_ring, dim=self.dim)

    def update_dev(self, n_dev, n_max, live, src_nodes, norms, computed_flag, emb, it_dev, refresh_retained,
                   stream, allow_alloc=True, mark=None):
        """This rank's admission request (no cache state changes here)."""
        if n_max <= 0:
            return
        if n_max > self.n_req:
            raise ValueError(f"layer {self.layer}: {n_max} live nodes exceed the request area ({self.n_req})")
        sb = _lib.query("hg_cache_update_scratch_bytes", n_max)
        scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        _lib.call("hg_cache_request", _lib.ptr(n_dev), n_max, float(self.policy.p_grad), _lib.ptr(live),
                  _lib.ptr(src_nodes), _lib.ptr(norms), _lib.ptr(computed_flag), _lib.ptr(emb), self.dim,
                  _lib.ptr(self.req_id), _lib.ptr(self.req_act), _lib.ptr(self.req_src), _lib.ptr(self.req_emb),
                  _lib.ptr(self.hdr),
                  _lib.ptr(scratch), sb, stream)
        if mark is not None:
            mark("ranked")

    def commit_dev(self, stream):
        """Owner side of the step: every rank's expiries, then the P requests."""
        o = self.owner
        q = max(1, self.n_req)
        _lib.call("hg_cache_invalidate", o.world, _lib.ptr(self.peer_exp), _lib.ptr(self.peer_hdr), q, self.lo,
                  self.hi, _lib.ptr(self.row_of_dev), _lib.ptr(self.row_owner_dev),
                  _lib.ptr(self.ctr), stream)
        sb = _lib.query("hg_cache_apply_scratch_bytes", q)
        scratch = torch.empty(sb, dtype=torch.uint8, device=self.device)
        # the kernels index the owner arrays by (id - lo)
        row_of, admit = _lib.ptr(self.row_of_dev), _lib.ptr(self.admit_iter_dev)
        for hdr, rid, ract, remb in self.peer_req:
            _lib.call("hg_cache_apply", hdr, rid, ract, remb, q, self.dim, self.lo, self.hi, float(self.policy.t_stale),
                      int(bool(o.refresh_retained)), self.cap_fixed, self.n_owned, self.limit_rows,
                      _lib.ptr(self.ring), row_of, _lib.ptr(self.row_owner_dev), admit, _lib.ptr(self.ctr),
                      _lib.ptr(scratch), sb, stream)

    def check_integrity(self):
        row_of = self.row_of
        live = np.flatnonzero(row_of >= 0)
        assert np.all((live >= self.lo) & (live < self.hi)), "a shard holds a node it does not own"
        super().check_integrity()


class ShardedHistCache(HistCache):
    """HistCache whose layer caches are owner-sharded over a process group.

    A collective constructor: every rank of `group` calls it with the same
    arguments. `n_req[l-1]` bounds the live nodes of cache layer l in one
    batch (the engine's upper bound, sampler.layer_bounds). The layer-0
    feature region stays replicated (HistCache.backfill_features)."""

    def __init__(self, num_nodes: int, layer_dims, policy: CachePolicy, n_req, rank: int, world: int,
                 feature_rows: int = 0, refresh_retained: bool = False, dtype=np.float32, device=None, group=None,
                 timeout_s: float = 120.0):
        import torch.distributed as dist
        _lib.require_cuda()
        if np.dtype(dtype) != np.float32:
            raise ValueError("the sharded cache stores fp32 rows")
        if world > 64:
            raise ValueError("at most 64 ranks")
        self.device = torch.device(device or "cuda")
        self.num_nodes = int(num_nodes)
        self.policy = policy
        self.refresh_retained = refresh_retained
        self.np_dtype = np.dtype(np.float32)
        self.rank, self.world = int(rank), int(world)
        self.bounds = owner_ranges(self.num_nodes, self.world)
        self.bounds_dev = torch.from_numpy(self.bounds.copy()).to(self.device)
        self.layers = {l + 1: ShardedLayerCache(self, l + 1, int(d), int(n_req[l])) for l, d in enumerate(layer_dims)}
        self.feature_rows = int(feature_rows)
        self.feature_dim = None
        self.feature_table = None
        self.feature_row_of_dev = torch.full((self.num_nodes,), -1, dtype=torch.int32, device=self.device)
        self.gctr = torch.zeros(GLOBAL_CTR_LEN, dtype=torch.int64, device=self.device)
        self._ops = 0
        # one IPC block per rank: every layer's sections + the barrier flag
        offs, o = [], 0
        for lc in self.layers.values():
            d = {}
            for name, nbytes in lc.sections():
                d[name] = o
                o += _align(nbytes)
            offs.append(d)
        flag_off = o
        total = o + 256
        p = ctypes.c_void_p()
        _lib.call("hg_device_alloc", total, ctypes.byref(p))
        self._owned = p.value
        torch.as_tensor(_DevBuf(p.value + flag_off, (32,), "<i8"), device=self.device).zero_()
        lib = _lib.load()
        hb = int(lib.hg_ipc_handle_bytes())
        h = ctypes.create_string_buffer(hb)
        _lib.call("hg_ipc_export", p, h)
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h.raw), group=group)
        bases, self._opened = [], []
        err = None
        for r in range(self.world):
            if r == self.rank:
                bases.append(p.value)
                continue
            q = ctypes.c_void_p()
            try:
                _lib.call("hg_ipc_open", ctypes.create_string_buffer(handles[r], hb), ctypes.byref(q))
            except _lib.HgError as e:       # e.g. no peer access between these GPUs
                err = e
                break
            bases.append(q.value)
            self._opened.append(q.value)
        # every rank learns whether every rank mapped every peer, so all fall back together
        ok = torch.tensor([0 if err is not None else 1], dtype=torch.int32,
                          device=self.device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            for q in self._opened:
                _lib.call("hg_ipc_close", ctypes.c_void_p(q))
            self._opened = []
            dist.barrier(group=group)
            _lib.call("hg_device_free", ctypes.c_void_p(self._owned))
            self._owned = None
            raise ShardingUnavailable(f"owner-sharded cache needs CUDA IPC peer mappings on every rank "
                                      f"({err if err is not None else 'failed on a peer rank'})")
        for lc, d in zip(self.layers.values(), offs):
            lc.bind(p.value, d, bases)
        self.my_flag = p.value + flag_off
        self.flags_dev = torch.tensor([b + flag_off for b in bases], dtype=torch.int64, device=self.device)
        self.bstate = torch.zeros(4, dtype=torch.int64, device=self.device)
        self.bstate[2] = int(timeout_s * 1e9)
        self._streams = None
        torch.cuda.synchronize(self.device)
        dist.barrier(group=group)

    sharded = True

    # ---- the step (called by Trainer._step and engine.StepEngine.run) ----
    def begin_step(self, it_dev, stream) -> None:
        """Open this step's request areas at iteration it_dev (every peer
        finished reading them: commit() ends with a barrier)."""
        for lc in self.layers.values():
            lc.reset_dev(it_dev, stream)

    def _barrier(self, stream) -> None:
        _lib.call("hg_peer_signal", self.my_flag, _lib.ptr(self.bstate), stream)
        _lib.call("hg_peer_wait", _lib.ptr(self.flags_dev), self.world, _lib.ptr(self.bstate), stream)

    def commit(self, stream) -> None:
        """Barrier (every rank's lookups and requests are done), the owner
        side of every layer, barrier (every owner is done with the peers'
        requests and embedding rows, which the next step may overwrite, and
        the next lookups see the committed state)."""
        self._barrier(stream)
        # the layers' caches share no state: their apply chains run side by side
        cur = torch.cuda.current_stream(self.device)
        if self._streams is None:
            self._streams = [torch.cuda.Stream(self.device) for _ in self.layers]
        for cs, lc in zip(self._streams, self.layers.values()):
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                lc.commit_dev(_lib.stream_ptr(cs))
        for cs in self._streams:
            cur.wait_stream(cs)
        self._barrier(stream)

    @property
    def timed_out(self) -> bool:
        return bool(int(self.bstate[1].item()))

    def check(self) -> None:
        if self.timed_out:
            raise RuntimeError("sharded cache barrier timed out waiting for a peer rank")

    def end_iteration(self, current_iter: int) -> None:
        """Sweeps run inside the commit, after each batch's request (cache.py:330-334)."""

    def sweep_staleness(self, current_iter=None) -> None:
        raise RuntimeError("the sharded cache sweeps inside its commit")

    def lookup(self, layer, ids, current_iter):
        raise NotImplementedError("the owner-sharded cache is driven by the data-parallel step (Trainer)")

    def update_cache(self, *a, **k):
        raise NotImplementedError("the owner-sharded cache is driven by the data-parallel step (Trainer)")

    def close(self, group=None) -> None:
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        dist.barrier(group=group)
        for q in self._opened:
            _lib.call("hg_ipc_close", ctypes.c_void_p(q))
        self._opened = []
        dist.barrier(group=group)
        if self._owned is not None:
            _lib.call("hg_device_free", ctypes.c_void_p(self._owned))
            self._owned = None
