"""histgnn.sampler conventions (sampler.py:26-263) over the GPU sampler.

`sample_layered` runs `hg_sample_layer` per fanout on the device (the
caller's Generator is advanced by exactly the reference's draw count) and
returns the reference's host form: int64 numpy blocks, block i's src_nodes
being the very object that is block i-1's dst_nodes (and src_deg / dst_deg
likewise), the outermost dst_nodes being `sub.seeds`. `SubgraphProducer`
samples on its own CUDA stream and worker thread and hands out the host form
in batch order with the reference's bounded run-ahead.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .. import sampler as _ds
from ..graphs import _np
from ..sampler import SamplePlan, batch_rng, split_batches
from .graphs import Csr2Graph, device_graph

__all__ = ["SamplePlan", "LayerBlock", "LayeredSubgraph", "split_batches", "batch_rng", "sample_layered",
           "SubgraphProducer"]


@dataclass
class LayerBlock:
    """sampler.py:44-71. adj rows are local positions into src_nodes."""

    dst_nodes: np.ndarray
    src_nodes: np.ndarray
    adj: Csr2Graph
    dst_deg: np.ndarray
    src_deg: np.ndarray = field(default=None)

    @property
    def num_dst(self) -> int:
        return self.dst_nodes.shape[0]

    @property
    def num_src(self) -> int:
        return self.src_nodes.shape[0]

    def copy(self) -> "LayerBlock":
        return LayerBlock(self.dst_nodes, self.src_nodes, self.adj.copy(), self.dst_deg, self.src_deg)


@dataclass
class LayeredSubgraph:
    """sampler.py:74-92. layers[0] is innermost; layers[-1].dst_nodes is seeds."""

    seeds: np.ndarray
    layers: list

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    @property
    def input_nodes(self) -> np.ndarray:
        return self.layers[0].src_nodes

    def copy(self) -> "LayeredSubgraph":
        return LayeredSubgraph(self.seeds, [b.copy() for b in self.layers])


def to_host(dsub, seeds: np.ndarray) -> LayeredSubgraph:
    """Host form of a device LayeredSubgraph with the reference's object
    sharing (outer block's src_nodes *is* the next block's dst_nodes)."""
    outer_first = list(reversed(dsub.layers))
    frontier = seeds
    blocks = []
    for blk in outer_first:
        src = _np(blk.src_nodes).astype(np.int64)
        src[:frontier.shape[0]] = frontier        # identical values; keeps dst a prefix
        F = blk.num_dst
        off = _np(blk.blk_off).astype(np.int64) if blk.blk_off is not None else None
        start = off[:F].copy() if off is not None else blk.adj.start_np
        adj = Csr2Graph(start, blk.adj.end_np, blk.adj.col_np, F)
        blocks.append(LayerBlock(frontier, src, adj, _np(blk.dst_deg).astype(np.int64)))
        frontier = src
    blocks.reverse()
    for i, b in enumerate(blocks):
        b.src_deg = np.zeros(b.num_src, dtype=np.int64) if i == 0 else blocks[i - 1].dst_deg
    return LayeredSubgraph(seeds, blocks)


def sample_layered(g, seeds, plan: SamplePlan, rng: np.random.Generator) -> LayeredSubgraph:
    """sampler.py:166-190 on the GPU; same errors, same caller-RNG advance."""
    seeds = np.asarray(seeds, dtype=np.int64)
    dsub = _ds.sample_layered(device_graph(g), seeds, plan, rng)
    return to_host(dsub, seeds)


class SubgraphProducer(_ds.SubgraphProducer):
    """sampler.py:193-263: worker-thread sampling (own CUDA stream) into a
    bounded FIFO; yields (batch_index, host LayeredSubgraph) in order."""

    def __init__(self, graph, batches, plan: SamplePlan, queue_capacity: int = 2):
        batches = [np.asarray(b, dtype=np.int64) for b in batches]
        super().__init__(device_graph(graph), batches, plan, queue_capacity)

    def __iter__(self):
        for idx, dsub in super().__iter__():
            yield idx, to_host(dsub, self._batches[idx])
