"""Generate golden vectors by running the REFERENCE (histgnn) in the build container.

Usage (build container only; /root/reference does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes small fixtures next to this script. Each fixture records the numpy and
scipy versions that produced it (`meta_numpy`, `meta_scipy`). The fixtures pin
the oracle (tests/test_oracle_golden.py) and, through the oracle or directly,
the CUDA path (tests/test_gpu_*.py).
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np
import scipy

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from histgnn.cache import CachePolicy, HistCache  # noqa: E402
from histgnn.data import synth_power_law, synth_sbm  # noqa: E402
from histgnn.graphs import CooGraph, build_csr2  # noqa: E402
from histgnn.nn import LayerKind, backward, cross_entropy, forward_pass, init_network  # noqa: E402
from histgnn.sampler import SamplePlan, batch_rng, sample_layered, split_batches  # noqa: E402
from histgnn.trainer import TrainConfig, Trainer, make_batches, prune_with_cache, run_plain_loop  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
META = {"meta_numpy": np.array(np.__version__), "meta_scipy": np.array(scipy.__version__)}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def put_sub(out, tag, sub):
    out[f"{tag}_seeds"] = sub.seeds
    out[f"{tag}_L"] = np.array(sub.num_layers)
    for i, b in enumerate(sub.layers):
        p = f"{tag}_b{i}_"
        out[p + "dst"] = b.dst_nodes
        out[p + "src"] = b.src_nodes
        out[p + "start"] = b.adj.start
        out[p + "end"] = b.adj.end
        out[p + "col"] = b.adj.col_indices
        out[p + "dst_deg"] = b.dst_deg
        out[p + "src_deg"] = b.src_deg
        out[p + "prune_writes"] = np.array(b.adj.prune_writes)


def small_powerlaw():
    ds = synth_power_law(3000, np.random.default_rng(0), m=4, feature_dim=16)
    return ds, build_csr2(ds.graph)


# ------------------------------------------------------------------ sampler


def gen_sampler():
    out = dict(META)
    # frozen path graph (test_sampler.py:85-99)
    g = build_csr2(CooGraph([0, 1], [1, 2], 3))
    sub = sample_layered(g, [2], SamplePlan((1, 1), 1, 0), np.random.default_rng(0))
    put_sub(out, "path", sub)
    # random multigraph with self loops and duplicate edges
    rng = np.random.default_rng(5)
    n = 40
    coo = CooGraph(rng.integers(0, n, 170), rng.integers(0, n, 170), n)
    g = build_csr2(coo)
    out["multi_start"], out["multi_end"], out["multi_col"] = g.start, g.end, g.col_indices
    seeds = np.sort(rng.choice(n, size=6, replace=False))
    sub = sample_layered(g, seeds, SamplePlan((3, 3, 3), 6, 0), batch_rng(17, 3))
    put_sub(out, "multi", sub)
    # one generator reused across two calls: the second call continues the stream
    r = np.random.default_rng(11)
    put_sub(out, "reuse0", sample_layered(g, seeds, SamplePlan((4, 2), 6, 0), r))
    put_sub(out, "reuse1", sample_layered(g, seeds[:3], SamplePlan((4, 2), 6, 0), r))
    # power-law 3000 nodes, fanouts (15,10,5), batch 256
    ds, g = small_powerlaw()
    out["pl_start"], out["pl_end"], out["pl_col"] = g.start, g.end, g.col_indices
    batches = split_batches(ds.train_ids, 256, np.random.default_rng(3))
    for idx in range(3):
        sub = sample_layered(g, batches[idx], SamplePlan((15, 10, 5), 256, 0), batch_rng(0, idx))
        put_sub(out, f"pl{idx}", sub)
    # hub rows wider than a warp and wider than 2048 candidates: a star graph
    hub = 5000
    srcs = np.concatenate([np.arange(1, hub + 1), np.arange(1, 40)])
    dsts = np.concatenate([np.zeros(hub, np.int64), np.full(39, 7)])
    g = build_csr2(CooGraph(srcs, dsts, hub + 1))
    out["star_start"], out["star_end"], out["star_col"] = g.start, g.end, g.col_indices
    sub = sample_layered(g, [0, 7, 3], SamplePlan((20, 40), 3, 0), batch_rng(9, 1))
    put_sub(out, "star", sub)
    np.savez_compressed(os.path.join(HERE, "sampler.npz"), **out)


# ---------------------------------------------------------------- C1 hashes


def gen_c1():
    """Size-independent golden for config C1: sha256 of the generated dataset
    and of the reference's sampled blocks for the first batches, plus the
    reference Trainer's IterMetrics for the first iterations."""
    ds = synth_power_law(100_000, np.random.default_rng(0), m=10, feature_dim=128)
    g = build_csr2(ds.graph)
    res = {
        "numpy": np.__version__,
        "dataset": {k: sha(v) for k, v in [("src", ds.graph.src), ("dst", ds.graph.dst),
                                           ("features", ds.features), ("labels", ds.labels),
                                           ("train", ds.train_ids)]},
        "csr2": {"start": sha(g.start), "end": sha(g.end), "col": sha(g.col_indices)},
    }
    cfg = TrainConfig(fanouts=(15, 10, 5), hidden=256, batch_size=1024, epochs=1,
                      eta=0.01, kind=LayerKind.SAGE_MEAN, p_grad=0.9, t_stale=20, seed=0)
    batches = make_batches(ds.train_ids, cfg)
    plan = SamplePlan(cfg.fanouts, cfg.batch_size, cfg.seed)
    subs = {}
    for idx in (0, 1, 7):
        sub = sample_layered(g, batches[idx], plan, batch_rng(cfg.seed, idx))
        subs[str(idx)] = {f"b{i}_{k}": sha(v) for i, b in enumerate(sub.layers)
                          for k, v in [("src", b.src_nodes), ("col", b.adj.col_indices),
                                       ("start", b.adj.start), ("dst_deg", b.dst_deg)]}
        subs[str(idx)]["sizes"] = [[b.num_dst, b.num_src, len(b.adj.col_indices)] for b in sub.layers]
    res["subgraphs"] = subs
    tr = Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
    mets = []
    for it in range(20):
        sub = sample_layered(g, batches[it], plan, batch_rng(cfg.seed, it))
        m = tr.train_iteration(it, 0, sub)
        mets.append({k: (float(v) if isinstance(v, float) else int(v)) for k, v in m.__dict__.items()
                     if k != "estimation_error"})
    res["trainer_sage_0.9_20"] = mets
    res["trainer_sage_0.9_20_weights"] = {
        f"W{l}": {"fro": float(np.linalg.norm(lp.weight.astype(np.float64))),
                  "sum": float(lp.weight.astype(np.float64).sum()),
                  "first": [float(x) for x in lp.weight.reshape(-1)[:16]]}
        for l, lp in enumerate(tr.network.layers)}
    with open(os.path.join(HERE, "c1.json"), "w") as fh:
        json.dump(res, fh, indent=1)


# -------------------------------------------------------------------- cache


def gen_cache():
    out = dict(META)
    cases = [
        (0.9, 3, None, False), (0.5, 2, 4, False), (1.0, math.inf, 5, False),
        (0.3, 1, 16, True), (1.0, 5, 2, False), (0.7, 4, None, True), (0.0, 2, 8, False),
    ]
    for ci, (p, t, cap, refresh) in enumerate(cases):
        num_nodes, dim = 24, 3
        cache = HistCache(num_nodes, [dim], CachePolicy(p, t, cap), refresh_retained=refresh,
                          dtype=np.float32)
        rng = np.random.default_rng(100 + ci)
        ops = []
        for it in range(25):
            batch = np.sort(rng.choice(num_nodes, size=int(rng.integers(1, num_nodes + 1)),
                                       replace=False))
            hits, rows, miss = cache.lookup(1, batch, it)
            emb = (batch[:, None] * 100.0 + it + np.arange(dim)).astype(np.float32)
            grads = np.floor(rng.random(len(batch)) * 6.0)   # many exact ties
            cache.update_cache(1, batch, miss, emb, grads, it)
            cache.end_iteration(it)
            lc = cache.layers[1]
            pfx = f"c{ci}_i{it}_"
            out[pfx + "batch"] = batch
            out[pfx + "grads"] = grads
            out[pfx + "hits"] = np.asarray(hits, np.int64)
            out[pfx + "hitrows"] = np.asarray(rows, np.float32)
            out[pfx + "miss"] = np.asarray(miss, np.int64)
            out[pfx + "row_of"] = lc.row_of.copy()
            out[pfx + "admit_iter"] = lc.admit_iter.copy()
            out[pfx + "row_owner"] = (lc.row_owner.copy() if lc.row_owner is not None
                                      else np.empty(0, np.int64))
            out[pfx + "table"] = (lc.table.copy() if lc.table is not None
                                  else np.empty((0, dim), np.float32))
            out[pfx + "scalars"] = np.array([lc.header, lc.capacity, lc.window_admissions,
                                             lc.window_forced], np.int64)
            c = cache.counters()
            out[pfx + "counters"] = np.array([c[k] for k in sorted(c)], np.int64)
        out[f"c{ci}_policy"] = np.array([p, t, -1 if cap is None else cap, float(refresh)])
    # feature region backfill with degree ties
    cache = HistCache(10, [2], CachePolicy(1.0, 1), feature_rows=4)
    feats = np.arange(20, dtype=np.float32).reshape(10, 2)
    deg = np.array([3, 7, 7, 1, 0, 7, 2, 3, 3, 9])
    cache.backfill_features(feats, deg)
    out["backfill_row_of"] = cache.feature_row_of
    out["backfill_table"] = cache.feature_table
    np.savez_compressed(os.path.join(HERE, "cache.npz"), **out)


# ------------------------------------------------------- prune + nn + trainer


def preload(cache, layer, ids, dim, it=0):
    ids = np.asarray(sorted(ids), dtype=np.int64)
    emb = (ids[:, None] * 10.0 + layer + np.arange(dim)).astype(np.float32)
    cache.update_cache(layer, ids, ids, emb, np.zeros(len(ids)), it)


def gen_prune_nn():
    out = dict(META)
    ds, g = small_powerlaw()
    hidden = 8
    for case, frac in enumerate((0.0, 0.3, 0.8)):
        rng = np.random.default_rng(40 + case)
        seeds = np.sort(rng.choice(ds.train_ids, size=64, replace=False))
        sub = sample_layered(g, seeds, SamplePlan((6, 4, 3), 64, 0), batch_rng(5, case))
        cache = HistCache(3000, [hidden, hidden], CachePolicy(1.0, math.inf))
        pre = {}
        for layer in (1, 2):
            ids = rng.choice(3000, size=int(frac * 3000), replace=False)
            pre[layer] = np.sort(ids)
            if len(ids):
                preload(cache, layer, ids, hidden)
            out[f"p{case}_pre{layer}"] = pre[layer]
        put_sub(out, f"p{case}_orig", sub.copy())
        pr = prune_with_cache(sub, cache, 1)
        put_sub(out, f"p{case}_pruned", sub)
        for b in range(4):
            out[f"p{case}_live{b}"] = pr.layer_live[b]
        for b in range(3):
            out[f"p{case}_rows{b}"] = pr.compute_rows[b]
            inj = pr.injected[b]
            out[f"p{case}_inj{b}_loc"] = (np.asarray(inj[0], np.int64) if inj is not None
                                         else np.empty(0, np.int64))
            out[f"p{case}_inj{b}_val"] = (np.asarray(inj[1], np.float32) if inj is not None
                                         else np.empty((0, hidden), np.float32))
        c = cache.counters()
        out[f"p{case}_counters"] = np.array([c[k] for k in sorted(c)], np.int64)
        # nn on the pruned batch, both kinds
        for kind in (LayerKind.SAGE_MEAN, LayerKind.GCN):
            net = init_network(kind, [16, hidden, hidden, ds.num_classes],
                               np.random.default_rng(7), np.float32)
            h0 = np.zeros((sub.layers[0].num_src, 16), np.float32)
            live0 = pr.layer_live[0]
            h0[live0] = ds.features[sub.layers[0].src_nodes[live0]]
            tape = forward_pass(net, sub.layers, h0, pr.compute_rows, pr.injected)
            loss, dlog = cross_entropy(tape.logits, ds.labels[sub.seeds])
            grads, ngr, dinp = backward(net, sub.layers, tape, dlog)
            k = f"p{case}_{kind.value}_"
            out[k + "loss"] = np.array(loss)
            for l in range(3):
                out[k + f"h{l}"] = tape.h_layers[l]
                out[k + f"ng{l}"] = ngr[l]
                out[k + f"W{l}"] = net.layers[l].weight
                out[k + f"gW{l}"] = grads[l].weight
                out[k + f"gb{l}"] = grads[l].bias
                if kind is LayerKind.SAGE_MEAN:
                    out[k + f"Wn{l}"] = net.layers[l].weight_neigh
                    out[k + f"gWn{l}"] = grads[l].weight_neigh
            out[k + "dinput"] = dinp
    np.savez_compressed(os.path.join(HERE, "prune_nn.npz"), **out)


def gen_trainer():
    out = dict(META)
    ds, g = small_powerlaw()
    for kind in (LayerKind.SAGE_MEAN, LayerKind.GCN):
        for p, t in ((0.9, 5), (0.0, 0), (0.6, math.inf)):
            cfg = TrainConfig(fanouts=(10, 5, 3), hidden=32, batch_size=128, epochs=2,
                              eta=0.05, kind=kind, p_grad=p, t_stale=t, seed=3)
            tr = Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
            ms = tr.train()
            k = f"{kind.value}_{p}_{t}_"
            names = [f for f in ms[0].__dict__ if f not in ("loss", "estimation_error")]
            out[k + "ints"] = np.array([[getattr(m, f) for f in names] for m in ms], np.int64)
            out[k + "loss"] = np.array([m.loss for m in ms])
            out[k + "weights_sha"] = np.array(hashlib.sha256(tr.network.checksum_bytes()).hexdigest())
            for l, lp in enumerate(tr.network.layers):
                out[k + f"W{l}"] = lp.weight
        out["int_names"] = np.array(names)
        cfg = TrainConfig(fanouts=(10, 5, 3), hidden=32, batch_size=128, epochs=1, eta=0.05,
                          kind=kind, p_grad=0.0, t_stale=0, seed=3)
        net, losses = run_plain_loop(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
        out[f"{kind.value}_plain_sha"] = np.array(hashlib.sha256(net.checksum_bytes()).hexdigest())
        out[f"{kind.value}_plain_loss"] = np.array(losses)
        for l, lp in enumerate(net.layers):
            out[f"{kind.value}_plain_W{l}"] = lp.weight
            out[f"{kind.value}_plain_b{l}"] = lp.bias
    np.savez_compressed(os.path.join(HERE, "trainer.npz"), **out)


def gen_evaluate():
    """trainer.py:473-506: full-graph inference of a briefly trained network."""
    from histgnn.nn import layer_forward
    from histgnn.trainer import evaluate, full_graph_blocks
    out = dict(META)
    ds, g = small_powerlaw()
    for kind in (LayerKind.SAGE_MEAN, LayerKind.GCN):
        cfg = TrainConfig(fanouts=(10, 5, 3), hidden=32, batch_size=128, epochs=1, eta=0.05, kind=kind,
                          p_grad=0.0, t_stale=0, seed=3)
        net, _ = run_plain_loop(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
        k = f"{kind.value}_"
        for l, lp in enumerate(net.layers):
            out[k + f"W{l}"] = lp.weight
            out[k + f"b{l}"] = lp.bias
            if lp.weight_neigh is not None:
                out[k + f"Wn{l}"] = lp.weight_neigh
        h = ds.features.astype(net.dtype)
        for l, blk in enumerate(full_graph_blocks(g, net.num_layers)):
            h = layer_forward(net.kind, net.layers[l], blk, h, activation=l < net.num_layers - 1)
        out[k + "logits"] = h
        out[k + "acc_val"] = np.array(evaluate(net, g, ds.features, ds.labels, ds.val_ids))
        out[k + "acc_test"] = np.array(evaluate(net, g, ds.features, ds.labels, ds.test_ids))
    out["val_ids"] = ds.val_ids
    out["test_ids"] = ds.test_ids
    np.savez_compressed(os.path.join(HERE, "evaluate.npz"), **out)


def gen_probes():
    """trainer.py:231-272,345-358: estimation-error and drift probes of a
    cache-everything run (p_grad 1, t_stale inf): every admission decision is
    independent of the gradient norms, so a free-running GPU trainer follows
    the same integer trajectory and its probes are comparable value for value."""
    out = dict(META)
    ds, g = small_powerlaw()
    for kind in (LayerKind.SAGE_MEAN, LayerKind.GCN):
        cfg = TrainConfig(fanouts=(4, 4), hidden=16, batch_size=64, epochs=2, eta=0.1, kind=kind, p_grad=1.0,
                          t_stale=math.inf, probe_every=1, seed=3)
        tr = Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes,
                     probe_nodes=np.arange(0, ds.features.shape[0], 7))
        ms = tr.train()
        k = f"{kind.value}_"
        names = [f for f in ms[0].__dict__ if f not in ("loss", "estimation_error")]
        out[k + "ints"] = np.array([[getattr(m, f) for f in names] for m in ms], np.int64)
        out[k + "loss"] = np.array([m.loss for m in ms])
        out[k + "est"] = np.array([m.estimation_error for m in ms])
        its = sorted(tr.embedding_log.records)
        pairs = [(t, s) for t in its[-3:] for s in (0, 1, 5, 20) if t - s in tr.embedding_log.records]
        out[k + "sim_pairs"] = np.array(pairs, np.int64)
        out[k + "sim"] = np.array([tr.embedding_log.similarity(t, s) for t, s in pairs])
        out[k + "log_ids_last"] = tr.embedding_log.records[its[-1]][0]
    out["int_names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "probes.npz"), **out)


def gen_datagen():
    out = dict(META)
    ds = synth_power_law(2000, np.random.default_rng(4), m=4, feature_dim=8, classes=5)
    for k, v in [("src", ds.graph.src), ("dst", ds.graph.dst), ("features", ds.features),
                 ("labels", ds.labels), ("train", ds.train_ids), ("val", ds.val_ids),
                 ("test", ds.test_ids)]:
        out["pl_" + k] = v
    ds = synth_sbm(600, np.random.default_rng(2), blocks=4)
    for k, v in [("src", ds.graph.src), ("dst", ds.graph.dst), ("features", ds.features),
                 ("labels", ds.labels), ("train", ds.train_ids)]:
        out["sbm_" + k] = v
    np.savez_compressed(os.path.join(HERE, "datagen.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["datagen", "sampler", "cache", "prune_nn", "trainer", "c1", "evaluate", "probes"]
    for w in which:
        print("generating", w, flush=True)
        globals()["gen_" + w]()
