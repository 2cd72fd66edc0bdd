"""histgnn.graphs conventions (graphs.py:37-172) on top of the device graph.

`Csr2Graph` here is the host-side, int64 numpy form a reference caller
holds: `start` / `end` per row into a shared `col_indices`, rows emptied in
O(1) by `end[v] = start[v]` and every such write counted in `prune_writes`.
`build_csr2` runs on the GPU (`graphs.build_csr2`: bincount + stable sort by
destination, so a row keeps the input edge order, graphs.py:161-172) and
returns the host form. The first GPU call on a host graph uploads it once
(`device_graph`); the mirror is rebuilt after any in-place prune.
"""

from __future__ import annotations

import zlib

import numpy as np

from .. import graphs as _dg
from ..graphs import CooGraph, _as_id_array, _check_ids, _np

__all__ = ["CooGraph", "Csr2Graph", "build_csr2", "device_graph"]


class Csr2Graph:
    """Dual-offset CSR over in-neighbours, host int64 arrays (graphs.py:77-150)."""

    def __init__(self, start, end, col_indices, num_nodes: int, prune_writes: int = 0):
        self.start = _as_id_array(start)
        self.end = _as_id_array(end)
        self.col_indices = _as_id_array(col_indices)
        self.num_nodes = int(num_nodes)
        self.prune_writes = int(prune_writes)
        self._mirror = None          # (version, device Csr2Graph)
        self._version = 0
        if self.start.shape[0] != self.num_nodes or self.end.shape[0] != self.num_nodes:
            raise ValueError(f"start/end must hold {self.num_nodes} offsets each")
        if self.num_nodes:
            if (self.end < self.start).any():
                raise ValueError("a row ends before it starts")
            if self.start.min() < 0 or self.end.max() > self.col_indices.shape[0]:
                raise ValueError("row offsets point outside col_indices")

    def __repr__(self):
        return f"Csr2Graph(num_nodes={self.num_nodes}, num_edges={self.num_edges}, prune_writes={self.prune_writes})"

    @property
    def num_edges(self) -> int:
        return int((self.end - self.start).sum())

    def _node(self, v) -> int:
        v = int(v)
        if v < 0 or v >= self.num_nodes:
            raise ValueError(f"node {v} out of range for {self.num_nodes} nodes")
        return v

    def neighbors(self, v: int) -> np.ndarray:
        v = self._node(v)
        return self.col_indices[self.start[v]:self.end[v]]

    def prune_in_neighbors(self, v: int) -> None:
        v = self._node(v)
        self.end[v] = self.start[v]
        self.prune_writes += 1
        self._version += 1

    def prune_many(self, nodes) -> None:
        nodes = _as_id_array(nodes)
        _check_ids(nodes, self.num_nodes, "prune")
        self.end[nodes] = self.start[nodes]
        self.prune_writes += nodes.shape[0]
        self._version += 1

    def in_degrees(self) -> np.ndarray:
        return self.end - self.start

    def to_coo(self) -> CooGraph:
        """Surviving edges only (graphs.py:127-136), destination-major."""
        deg = self.in_degrees()
        total = int(deg.sum())
        dst = np.repeat(np.arange(self.num_nodes, dtype=np.int64), deg)
        first = np.repeat(self.start, deg)
        within = np.arange(total, dtype=np.int64) - np.repeat(np.cumsum(deg) - deg, deg)
        return CooGraph(self.col_indices[first + within], dst, self.num_nodes)

    def copy(self) -> "Csr2Graph":
        """Own offsets, shared columns (pruning never writes col_indices)."""
        return Csr2Graph(self.start.copy(), self.end.copy(), self.col_indices, self.num_nodes)

    def col_checksum(self) -> int:
        return zlib.crc32(np.ascontiguousarray(self.col_indices).tobytes())


def device_graph(g, device=None):
    """The device Csr2Graph for a host (compat or reference-typed) graph,
    uploaded once and kept while the host offsets are unchanged."""
    if isinstance(g, _dg.Csr2Graph):
        return g
    ver = getattr(g, "_version", None)
    if ver is None:    # a foreign (e.g. reference) graph: key on its offsets' content
        ver = ("crc", id(g.col_indices), zlib.crc32(np.ascontiguousarray(g.start).tobytes()),
               zlib.crc32(np.ascontiguousarray(g.end).tobytes()))
    mirror = getattr(g, "_mirror", None)
    if mirror is not None and mirror[0] == ver:
        return mirror[1]
    d = _dg.csr2_from_arrays(g.start, g.end, g.col_indices, device=device)
    try:
        g._mirror = (ver, d)
    except AttributeError:
        pass
    return d


def build_csr2(edges) -> Csr2Graph:
    """graphs.py:161-172 on the GPU; accepts any (src, dst, num_nodes) edge list."""
    coo = edges if isinstance(edges, CooGraph) else CooGraph(edges.src, edges.dst, edges.num_nodes)
    d = _dg.build_csr2(coo)
    g = Csr2Graph(_np(d.start), _np(d.end), _np(d.col_indices).astype(np.int64), coo.num_nodes)
    g._mirror = (g._version, d)
    return g
