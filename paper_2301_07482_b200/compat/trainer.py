"""histgnn.trainer conventions (trainer.py:59-506) over the device trainer.

`prune_with_cache` takes the reference's host LayeredSubgraph, runs the
walk on the GPU (`hg_prune_block` + `hg_cache_lookup` per block), writes the
pruned row ends back into the caller's numpy offsets (counting them in
`adj.prune_writes`, as `Csr2Graph.prune_many` does) and returns int64 numpy
`compute_rows` / `layer_live` and `(local rows, values)` injections.
`Trainer` accepts host graphs and host subgraphs and exposes the
reference's `source` accounting (`row_bytes`, `fetched_bytes`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .. import trainer as _dt
from ..graphs import Csr2Graph as _DevCsr2, _np
from ..sampler import LayerBlock as _DevBlock, LayeredSubgraph as _DevSub
from ..trainer import (EmbeddingLog, IterMetrics, TrainConfig, cosine_rows, epoch_mean_estimation_error,  # noqa: F401
                       io_saving, make_batches, write_metrics_csv)
from .graphs import device_graph
from .nn import to_device
from .sampler import LayeredSubgraph

__all__ = ["TrainConfig", "IterMetrics", "PrunedBatch", "prune_with_cache", "Trainer", "run_plain_loop", "evaluate",
           "make_batches", "io_saving", "write_metrics_csv", "epoch_mean_estimation_error", "cosine_rows",
           "EmbeddingLog", "FeatureSource"]


@dataclass
class PrunedBatch:
    """trainer.py:138-150, host form."""

    sub: LayeredSubgraph
    compute_rows: list
    injected: list
    layer_live: list


def _i32(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)


def to_device_sub(sub: LayeredSubgraph, device) -> _DevSub:
    """Upload a host subgraph (current, possibly pruned, row ends included)."""
    blocks = []
    for b in sub.layers:
        src = _i32(b.src_nodes, device)
        E = b.adj.col_indices.shape[0]
        off = np.append(np.asarray(b.adj.start, np.int64), E)
        off_d = _i32(off, device)
        adj = _DevCsr2(off_d[:b.num_dst], _i32(b.adj.end, device), _i32(b.adj.col_indices, device), b.num_dst)
        blocks.append(_DevBlock(src[:b.num_dst], src, adj, _i32(b.dst_deg, device), _i32(b.src_deg, device), off_d))
    return _DevSub(np.asarray(sub.seeds, np.int64), blocks)


def _write_back(sub: LayeredSubgraph, dsub: _DevSub) -> None:
    """Pruned row ends (and the prune-write count) into the host offsets."""
    for hb, db in zip(sub.layers, dsub.layers):
        hb.adj.end[:] = db.adj.end_np
        hb.adj.prune_writes += db.adj.prune_writes
        hb.adj._version = getattr(hb.adj, "_version", 0) + 1


def prune_with_cache(sub: LayeredSubgraph, cache, current_iter: int) -> PrunedBatch:
    """trainer.py:166-207 on the GPU; prunes `sub` in place."""
    dsub = to_device_sub(sub, cache.device)
    p = _dt.prune_with_cache(dsub, cache, current_iter)
    _write_back(sub, dsub)
    L = sub.num_layers
    compute = [_np(p.compute_rows[b]).astype(np.int64) for b in range(L)]
    live = [_np(p.layer_live[b]).astype(np.int64) for b in range(L + 1)]
    injected = []
    for b in range(L):
        inj = p.injected_np(b)
        injected.append(None if inj is None or inj[0].shape[0] == 0 else inj)
    return PrunedBatch(sub, compute, injected, live)


class FeatureSource:
    """trainer.py:213-228 accounting view: the device gather's miss rows."""

    def __init__(self, trainer):
        self._tr = trainer
        self.fetched_bytes = 0
        self.fetched_rows = 0

    @property
    def features(self):
        return self._tr.features

    @property
    def row_bytes(self) -> int:
        return self._tr.row_bytes

    def _account(self, m) -> None:
        self.fetched_rows += m.feature_misses
        self.fetched_bytes += m.fetched_bytes


class Trainer(_dt.Trainer):
    """trainer.py:285-433 on the GPU; host graphs, host subgraphs."""

    def __init__(self, graph, features, labels, train_ids, cfg: TrainConfig, num_classes=None, probe_nodes=None):
        super().__init__(device_graph(graph), features, labels, train_ids, cfg, num_classes, probe_nodes)
        self.host_graph = graph
        self.source = FeatureSource(self)
        self._in_train = False

    def train_iteration(self, iteration: int, epoch: int, sub, probe: bool = False):
        if isinstance(sub, LayeredSubgraph):
            dsub = to_device_sub(sub, self.device)
            m = super().train_iteration(iteration, epoch, dsub, probe)
            _write_back(sub, dsub)
        else:
            m = super().train_iteration(iteration, epoch, sub, probe)
        if not self._in_train:
            self.source._account(m)
        return m

    def train(self) -> list:
        n0 = len(self.metrics)
        self._in_train = True
        try:
            out = super().train()
        finally:
            self._in_train = False
        for m in out[n0:]:
            self.source._account(m)
        return out


def run_plain_loop(graph, features, labels, train_ids, cfg: TrainConfig, num_classes=None, on_step=None):
    """trainer.py:439-469 on the GPU (host graph accepted)."""
    return _dt.run_plain_loop(device_graph(graph), features, labels, train_ids, cfg, num_classes, on_step)


def evaluate(network, graph, features, labels, ids) -> float:
    """trainer.py:485-506 on the GPU (host network / graph accepted)."""
    return _dt.evaluate(to_device(network), device_graph(graph), features, labels, ids)
