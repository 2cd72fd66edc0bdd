"""Data-parallel oracle (TEST INFRASTRUCTURE ONLY) — SURVEY §8(e).

The reference defines no multi-GPU semantics (trainer.py:423-433 is strictly
sequential), so this fixes them and restates them serially on one CPU:
P workers share the weights; at step s worker r takes global batch P*s + r,
runs prune/load/forward/backward on its own cache replica, the P gradient sets
are averaged (the all-reduce), every worker applies the same SGD step, then
each worker updates its own cache with its own norms. With P = 1 this is
exactly OTrainer.train.
"""

from __future__ import annotations

import copy

import numpy as np

from .step import OTrainer, make_batches


def average_grads(grad_sets):
    """Mean of P per-layer gradient lists, summed in rank order (fp32)."""
    P = len(grad_sets)
    out = copy.deepcopy(grad_sets[0])
    for l, g in enumerate(out):
        for name in ("weight", "bias", "weight_neigh"):
            a = getattr(g, name)
            if a is None:
                continue
            acc = a.copy()
            for r in range(1, P):
                acc = acc + getattr(grad_sets[r][l], name)
            setattr(g, name, (acc / np.float32(P)).astype(a.dtype))
    return out


def dp_serial_run(graph, features, labels, train_ids, cfg, num_classes, world, steps, norms_for=None):
    """Returns ([per-rank metrics lists], final network of rank 0).
    norms_for(rank, step) -> {layer: fp64 norms} feeds each worker's cache
    admission with externally computed norms (lockstep, SURVEY §8(c) Mode B)."""
    workers = [OTrainer(graph, features, labels, train_ids, cfg, num_classes) for _ in range(world)]
    batches = make_batches(train_ids, cfg)
    metrics = [[] for _ in range(world)]
    for s in range(steps):
        # phase 1: every worker computes its gradients (captured, not applied)
        captured = [None] * world
        subs = []
        for r, w in enumerate(workers):
            idx = world * s + r
            subs.append((idx, w.sample(idx, batches[idx])))

        # run each worker's iteration with a hook that first collects all
        # ranks' grads: emulate the synchronous all-reduce by two passes
        def collect(r):
            def hook(grads):
                captured[r] = copy.deepcopy(grads)
                raise _Stop()
            return hook

        snaps = [copy.deepcopy(w) for w in workers]
        for r, w in enumerate(workers):
            try:
                w.train_iteration(subs[r][0], 0, copy.deepcopy(subs[r][1]), grad_hook=collect(r))
            except _Stop:
                pass
        mean = average_grads(captured)
        workers = snaps

        def apply_mean(grads):
            for g, m in zip(grads, mean):
                g.weight[...] = m.weight
                g.bias[...] = m.bias
                if g.weight_neigh is not None:
                    g.weight_neigh[...] = m.weight_neigh

        for r, w in enumerate(workers):
            nrm = None if norms_for is None else norms_for(r, s)
            metrics[r].append(w.train_iteration(subs[r][0], 0, subs[r][1], norms_override=nrm, grad_hook=apply_mean))
    return metrics, workers[0].network


class _Stop(Exception):
    pass
