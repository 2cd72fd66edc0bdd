"""Feature table sharded over the GPUs of one box.

The reference models multi-GPU feature placement only as accounting:
`partition_features` (histgnn/comms.py:329-337) gives GPU r the contiguous
node range [bounds[r], bounds[r+1]) (the first N % P GPUs one extra row), and
the paper's loader reads remote rows one-sided. Here each
rank keeps ONLY its own range in HBM; the other ranks' shards are mapped into
its address space with CUDA IPC, so `hg_load_features_sharded` reads a miss
row straight from the owner's HBM over NVLink (no all-to-all, no staging).
The static feature region (the top N/10 in-degree rows, cache.py:338-351) is
replicated on every rank, so region hits stay local.

`ShardedFeatures.virtual` puts all P shards on one device (pointer tables of
local memory): the same kernel path, used by the 1-GPU tests and for
checking that sharding is bit-transparent.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .distributed import owner_ranges

_DT = {torch.float32: (0, "<f4"), torch.float16: (1, "<f2")}


class _DevBuf:
    """__cuda_array_interface__ view of a raw device allocation."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class ShardedFeatures:
    """A [num_nodes x dim] feature table split by contiguous owner ranges.

    Attributes used by the trainer: shape, dtype, device, element_size(),
    dtype_code, ptrs_dev (int64[P] shard base pointers), bounds_dev
    (int64[P+1]), num_shards, local_shard."""

    def __init__(self, num_nodes: int, dim: int, dtype, device, bounds: np.ndarray, ptrs: list, local: int,
                 keepalive=(), owned=None, opened=()):
        if dtype not in _DT:
            raise ValueError(f"unsupported feature dtype {dtype} (fp32 / fp16)")
        if len(ptrs) > 16:
            raise ValueError("at most 16 shards")
        self.num_nodes = int(num_nodes)
        self.dim = int(dim)
        self.dtype = dtype
        self.device = torch.device(device)
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.num_shards = len(ptrs)
        self.local_shard = int(local)
        self.ptrs_dev = torch.tensor([int(p) for p in ptrs], dtype=torch.int64, device=self.device)
        self.bounds_dev = torch.from_numpy(self.bounds.copy()).to(self.device)
        self._keepalive = list(keepalive)
        self._owned = owned          # hg_device_alloc pointer of the local shard (IPC mode)
        self._opened = list(opened)  # IPC mappings of peer shards
        self.local_rows = None       # tensor view of this rank's own shard
        # rows read per owner shard (cumulative; the real transfer sizes behind
        # distributed.transfer_accounting, comms.py:283-337)
        self.owner_rows = torch.zeros(self.num_shards, dtype=torch.int64, device=self.device)

    # ---- tensor-like surface used by Trainer / cache.backfill_features ----
    @property
    def shape(self):
        return (self.num_nodes, self.dim)

    def element_size(self) -> int:
        return torch.tensor([], dtype=self.dtype).element_size()

    @property
    def dtype_code(self) -> int:
        return _DT[self.dtype][0]

    # ---- construction ----
    @classmethod
    def virtual(cls, features, num_shards: int, device="cuda"):
        """All shards on `device` (single process): bit-identical results to
        the unsharded table, the kernel path of the multi-GPU layout."""
        _lib.require_cuda()
        feats = features if isinstance(features, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(features))
        n, d = int(feats.shape[0]), int(feats.shape[1])
        bounds = owner_ranges(n, num_shards)
        shards = [feats[bounds[o]:bounds[o + 1]].to(device).contiguous() for o in range(num_shards)]
        out = cls(n, d, feats.dtype, device, bounds, [s.data_ptr() for s in shards], 0, keepalive=shards)
        out.local_rows = shards[0]
        return out

    @classmethod
    def from_process_group(cls, local_rows, num_nodes: int, rank: int, world: int, device, group=None):
        """Collective over `group` (every rank calls it with its own range
        [bounds[rank], bounds[rank+1]) of rows): allocate the local shard,
        exchange CUDA IPC handles, map every peer shard."""
        import torch.distributed as dist
        _lib.require_cuda()
        bounds = owner_ranges(num_nodes, world)
        rows = local_rows if isinstance(local_rows, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(local_rows))
        if rows.shape[0] != bounds[rank + 1] - bounds[rank]:
            raise ValueError(f"rank {rank} must pass rows [{bounds[rank]}, {bounds[rank + 1]})")
        d = int(rows.shape[1])
        lib = _lib.load()
        nbytes = max(1, int(rows.shape[0]) * d * rows.element_size())
        p = ctypes.c_void_p()
        _lib.call("hg_device_alloc", nbytes, ctypes.byref(p))
        local = torch.as_tensor(_DevBuf(p.value, (int(rows.shape[0]), d), _DT[rows.dtype][1]), device=device)
        local.copy_(rows)
        torch.cuda.synchronize(device)
        hb = int(lib.hg_ipc_handle_bytes())
        h = ctypes.create_string_buffer(hb)
        _lib.call("hg_ipc_export", p, h)
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h.raw), group=group)
        ptrs, opened = [], []
        for o in range(world):
            if o == rank:
                ptrs.append(p.value)
                continue
            q = ctypes.c_void_p()
            _lib.call("hg_ipc_open", ctypes.create_string_buffer(handles[o], hb), ctypes.byref(q))
            ptrs.append(q.value)
            opened.append(q.value)
        out = cls(num_nodes, d, rows.dtype, device, bounds, ptrs, rank, keepalive=[local], owned=p.value,
                  opened=opened)
        out.local_rows = local
        return out

    def close(self):
        """Unmap peer shards and free the local one (after every peer is done:
        callers barrier first)."""
        for q in self._opened:
            _lib.call("hg_ipc_close", ctypes.c_void_p(q))
        self._opened = []
        self._keepalive = []
        self.local_rows = None
        if self._owned is not None:
            torch.cuda.synchronize(self.device)
            _lib.call("hg_device_free", ctypes.c_void_p(self._owned))
            self._owned = None

    # ---- row access ----
    def load_rows(self, n_live_dev, n_max: int, live, src_nodes, feature_row_of, region, out, gctr, stream,
                  count: bool = True):
        """hg_load_features_sharded: out[live[i]] = fp32(row of src_nodes[live[i]])."""
        _lib.call("hg_load_features_sharded", _lib.ptr(n_live_dev), int(n_max), _lib.ptr(live), _lib.ptr(src_nodes),
                  _lib.ptr(feature_row_of), _lib.ptr(region), _lib.ptr(self.ptrs_dev), _lib.ptr(self.bounds_dev),
                  self.num_shards, self.local_shard, self.dim, self.dtype_code, _lib.ptr(out), _lib.ptr(gctr),
                  _lib.ptr(self.owner_rows) if count else None, stream)

    def index_select(self, dim: int, ids: torch.Tensor, chunk: int = 1 << 22) -> torch.Tensor:
        """rows[ids] in the table's dtype (device), read through the shards
        (used once, to build the replicated static feature region)."""
        if dim != 0:
            raise ValueError("rows only")
        ids = ids.to(self.device).to(torch.int32)
        k = int(ids.numel())
        out = torch.empty((k, self.dim), dtype=self.dtype, device=self.device)
        gctr = torch.zeros(8, dtype=torch.int64, device=self.device)
        sp = _lib.stream_ptr()
        for a in range(0, k, chunk):
            b = min(k, a + chunk)
            n = b - a
            tmp = torch.empty((n, self.dim), dtype=torch.float32, device=self.device)
            live = torch.arange(n, dtype=torch.int32, device=self.device)
            cnt = torch.tensor([n], dtype=torch.int32, device=self.device)
            self.load_rows(cnt, n, live, ids[a:b].contiguous(), None, None, tmp, gctr, sp, count=False)
            out[a:b] = tmp.to(self.dtype)      # fp16 -> fp32 -> fp16 is exact
        return out
