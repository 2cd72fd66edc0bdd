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


def dp_sharded_run(graph, features, labels, train_ids, cfg, num_classes, world, steps, norms_for=None):
    """The data-parallel run with ONE owner-sharded cache (oracle/shardcache.py)
    instead of per-rank caches. Per step: every rank samples its batch, prunes
    with pure-read lookups of the state after the previous step, trains, the
    gradients are averaged and applied; then the owners apply all expiries and
    the P update requests in rank order (each followed by its end_iteration).
    Rank r's metrics: its own lookups (hits / misses / feature) and bytes, and
    owner r's admissions / evictions / valid entries.
    Returns ([per-rank metrics lists], final network, the shared cache)."""
    import dataclasses

    from .histcache import OCachePolicy
    from .shardcache import OShardedCache

    workers = [OTrainer(graph, features, labels, train_ids, cfg, num_classes) for _ in range(world)]
    w0 = workers[0]
    shared = OShardedCache(w0.num_nodes, [cfg.hidden] * (len(cfg.fanouts) - 1),
                           OCachePolicy(cfg.p_grad, cfg.t_stale, cfg.capacity), world,
                           feature_rows=w0.cache.feature_rows, refresh_retained=cfg.refresh_retained, dtype=cfg.dtype)
    if shared.feature_rows > 0:
        shared.backfill_features(features, w0.end - w0.start)
    for w in workers:
        w.cache = None
    batches = make_batches(train_ids, cfg)
    metrics = [[] for _ in range(world)]
    evict_fields = ("admissions", "gradient_evictions", "staleness_evictions", "forced_evictions")
    for s in range(steps):
        subs = [(world * s + r, workers[r].sample(world * s + r, batches[world * s + r])) for r in range(world)]
        captured = [None] * world
        snaps = [copy.deepcopy(w) for w in workers]
        for r, w in enumerate(workers):
            w.cache = shared.view(r)

            def hook(grads, r=r):
                captured[r] = copy.deepcopy(grads)
                raise _Stop()
            try:
                w.train_iteration(subs[r][0], 0, copy.deepcopy(subs[r][1]), grad_hook=hook)
            except _Stop:
                pass
            w.cache = None
        mean = average_grads(captured)
        workers = snaps

        def apply_mean(grads):
            for g, m in zip(grads, mean):
                g.weight[...] = m.weight
                g.bias[...] = m.bias
                if g.weight_neigh is not None:
                    g.weight_neigh[...] = m.weight_neigh

        views, step_ms = [], []
        for r, w in enumerate(workers):
            w.cache = views.append(shared.view(r)) or views[-1]
            nrm = None if norms_for is None else norms_for(r, s)
            step_ms.append(w.train_iteration(subs[r][0], 0, subs[r][1], norms_override=nrm, grad_hook=apply_mean))
            w.cache = None
        before = [shared.owner_counters(o) for o in range(world)]
        shared.commit(views)
        for r in range(world):
            after = shared.owner_counters(r)
            upd = {k: after[k] - before[r][k] for k in evict_fields}
            metrics[r].append(dataclasses.replace(step_ms[r], valid_entries=shared.owner_valid(r), **upd))
    return metrics, workers[0].network, shared
