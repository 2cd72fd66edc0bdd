"""Data-parallel plumbing for the per-iteration path.

One process per GPU. Rank r of P trains global batch indices P*s + r at step
s, so every batch's sampled subgraph is bit-identical to the single-GPU run
(per-batch PCG64 streams, histgnn/sampler.py:104-106). The one exchange step
is the gradient all-reduce of the single flat parameter bucket (all layers in
one contiguous fp32 buffer, nn.Network.flat) before SGD; NCCL over NVLink on
the GPU box, gloo in the CPU tests. Feature / cache ownership follows the
reference's contiguous partition (histgnn/comms.py:329-337).
"""

from __future__ import annotations

import numpy as np


def rank_batch_indices(num_batches: int, rank: int, world: int) -> list:
    """Global batch indices rank `rank` trains, in step order."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    steps = num_batches // world          # every rank takes the same number of steps
    return [world * s + rank for s in range(steps)]


def owner_ranges(num_nodes: int, world: int) -> np.ndarray:
    """Contiguous owner ranges [bounds[r], bounds[r+1]) like
    comms.partition_features: the first num_nodes % world owners get one
    extra row."""
    base, extra = divmod(num_nodes, world)
    sizes = np.full(world, base, dtype=np.int64)
    sizes[:extra] += 1
    return np.concatenate([[0], np.cumsum(sizes)])


def owner_of(ids, bounds: np.ndarray) -> np.ndarray:
    return np.searchsorted(bounds, np.asarray(ids), side="right") - 1


def make_allreduce_hook(world: int, group=None):
    """Trainer.grad_hook that averages the flat gradient bucket over ranks
    (one all-reduce per step, fixed reduction order inside the backend)."""
    import torch.distributed as dist

    def hook(grads):
        flat = grads.flat
        dist.all_reduce(flat, group=group)
        flat.div_(world)

    # NCCL collectives are stream-ordered device work and can be captured in
    # the step's CUDA graph (engine.StepEngine); gloo's host-side all-reduce
    # cannot, so a gloo hook keeps the step eager
    hook.graph_safe = dist.get_backend(group) == "nccl"
    return hook
