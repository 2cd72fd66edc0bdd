"""Graph containers, device resident (drop-in for histgnn/graphs.py).

`Csr2Graph` keeps the reference's dual-offset CSR (graphs.py:77-150): `start`
and `end` per row into a shared column array, so a row is emptied in O(1) by
`end[v] = start[v]`. On the device the full graph is stored as int64 offsets
(`start`, `end`) and int32 columns (N < 2^31), in HBM, built once by
`build_csr2` with the reference's stable in-row order (graphs.py:161-172).
Sampled blocks use the same container with int32 local offsets.
"""

from __future__ import annotations

import zlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib


def _as_id_array(x) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.int64)
    if a.ndim != 1:
        raise ValueError(f"expected a 1-d id array, got shape {a.shape}")
    return a


def _check_ids(a: np.ndarray, num_nodes: int, what: str) -> None:
    if len(a) == 0:
        return
    lo, hi = int(a.min()), int(a.max())
    if lo < 0 or hi >= num_nodes:
        raise ValueError(f"{what} id out of range: saw {lo if lo < 0 else hi} "
                         f"for a graph with {num_nodes} nodes")


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@dataclass
class CooGraph:
    """Directed multigraph; (src[i], dst[i]) is src -> dst (graphs.py:37-62)."""

    src: np.ndarray
    dst: np.ndarray
    num_nodes: int

    def __post_init__(self):
        self.src = _as_id_array(self.src)
        self.dst = _as_id_array(self.dst)
        if len(self.src) != len(self.dst):
            raise ValueError(f"src/dst length mismatch: {len(self.src)} vs {len(self.dst)}")
        if self.num_nodes < 0:
            raise ValueError("num_nodes must be non-negative")
        _check_ids(self.src, self.num_nodes, "src")
        _check_ids(self.dst, self.num_nodes, "dst")

    @property
    def num_edges(self) -> int:
        return len(self.src)


@dataclass
class Csr2Graph:
    """Dual-offset CSR over in-neighbours; tensors live on the GPU.

    start/end: int64 (full graph) or int32 (sampled block) device tensors,
    col_indices: int32 device tensor. Numpy views are available through
    `.numpy()` style properties for parity checks.
    """

    start: torch.Tensor
    end: torch.Tensor
    col_indices: torch.Tensor
    num_nodes: int
    prune_writes: int = field(default=0, compare=False)
    # device-side prune-write counter for sampled blocks (resolved lazily)
    _prune_dev: object = field(default=None, compare=False, repr=False)

    @property
    def num_edges(self) -> int:
        return int((self.end.long() - self.start.long()).sum().item())

    def neighbors(self, v: int) -> np.ndarray:
        if not 0 <= v < self.num_nodes:
            raise ValueError(f"node {v} out of range for {self.num_nodes} nodes")
        s, e = int(self.start[v]), int(self.end[v])
        return _np(self.col_indices[s:e]).astype(np.int64)

    def prune_in_neighbors(self, v: int) -> None:
        if not 0 <= v < self.num_nodes:
            raise ValueError(f"node {v} out of range for {self.num_nodes} nodes")
        self.end[v] = self.start[v]
        self.prune_writes += 1

    def prune_many(self, nodes) -> None:
        nodes = _as_id_array(nodes)
        _check_ids(nodes, self.num_nodes, "prune")
        idx = torch.as_tensor(nodes, device=self.start.device)
        self.end[idx] = self.start[idx]
        self.prune_writes += len(nodes)

    def in_degrees(self) -> np.ndarray:
        return _np(self.end.long() - self.start.long())

    def copy(self) -> "Csr2Graph":
        return Csr2Graph(self.start.clone(), self.end.clone(), self.col_indices, self.num_nodes)

    def col_checksum(self) -> int:
        return zlib.crc32(np.ascontiguousarray(_np(self.col_indices).astype(np.int64)).tobytes())

    # numpy views (int64 like the reference)
    @property
    def start_np(self):
        return _np(self.start).astype(np.int64)

    @property
    def end_np(self):
        return _np(self.end).astype(np.int64)

    @property
    def col_np(self):
        return _np(self.col_indices).astype(np.int64)


def build_csr2(edges: CooGraph, device=None) -> Csr2Graph:
    """graphs.py:161-172 — group edges by destination, stable within a row,
    built on the GPU (hg_build_csr2: counts, scan, placement, per-row sort)."""
    _lib.require_cuda()
    n = edges.num_nodes
    if n >= 2**31:
        raise ValueError("node ids must fit int32 on the device")
    from .data import csr2_from_edges_device
    return csr2_from_edges_device(edges.src, edges.dst, n, torch.device(device or "cuda"))


def csr2_from_arrays(start, end, col, device=None) -> Csr2Graph:
    """Upload an existing host CSR2 (e.g. a reference Csr2Graph's arrays)."""
    _lib.require_cuda()
    dev = torch.device(device or "cuda")
    s = torch.as_tensor(np.asarray(start, np.int64), device=dev)
    e = torch.as_tensor(np.asarray(end, np.int64), device=dev)
    c = torch.as_tensor(np.asarray(col, np.int64).astype(np.int32), device=dev)
    return Csr2Graph(s, e, c, len(start))
