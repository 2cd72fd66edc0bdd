"""Parity at the benchmark configurations, not only at toy
scale.

* C1 at full size (100K nodes / 2M edges, 128-d, SAGE hidden 256, fanouts
  15,10,5, batch 1024, cache (0.9, 20)): the dataset produced by the native
  generator hashes to the reference's (tests/golden/c1.json); the first
  iteration of the GPU trainer (engine: CUDA graph + lookahead sampler) equals
  the reference Trainer's IterMetrics; then 24 iterations run in lockstep with
  the oracle (Mode B: the oracle's admission ranks the GPU's fp64 norms), every
  integer metric and pruned set bit-exact, loss and weights within 1e-3.
* C2 (the products shape the bench line is measured on, same generator and
  config as bench.py): 4 engine iterations in lockstep with the oracle.
* The cache-free GPU loop against the reference's run_plain_loop goldens.
"""

import math

import numpy as np
import pytest

from oracle.datagen import csr2_from_edges
from oracle.step import GCN, SAGE, OTrainConfig, OTrainer
from tests.goldens import load, load_json, sha

pytestmark = pytest.mark.gpu

INT_FIELDS = ["fetched_bytes", "baseline_bytes", "prune_writes", "hits", "misses", "admissions",
              "gradient_evictions", "staleness_evictions", "forced_evictions", "feature_hits",
              "feature_misses", "valid_entries"]


def _lockstep(tr, otr, batches, iters, first_gold=None):
    """Engine steps (lookahead on) against the oracle with the GPU's norms."""
    for it in range(iters):
        nxt = (it + 1, batches[it + 1]) if it + 1 < len(batches) else None
        m = tr.train_step(it, 0, batches[it], next_batch=nxt)
        norms = {l: tr.last[3][l].cpu().numpy() for l in range(1, 3)}
        om = otr.train_iteration(it, 0, otr.sample(it, batches[it]), norms_override=norms)
        if it == 0 and first_gold is not None:
            # iteration 0 has no cache history: the free-running GPU run must
            # equal the reference's own Trainer (integers exact, loss 1e-3)
            for f in INT_FIELDS:
                assert getattr(m, f) == first_gold[f], (f, getattr(m, f), first_gold[f])
            assert abs(m.loss - first_gold["loss"]) <= 1e-3 * abs(first_gold["loss"])
        for f in INT_FIELDS:
            assert getattr(m, f) == getattr(om, f), (it, f, getattr(m, f), getattr(om, f))
        assert abs(m.loss - om.loss) <= 1e-3 * abs(om.loss), (it, m.loss, om.loss)
        for b in range(3):
            np.testing.assert_array_equal(tr.last.layer_live[b].cpu().numpy(), otr.last[0].layer_live[b])
            np.testing.assert_array_equal(tr.last.compute_rows[b].cpu().numpy(), otr.last[0].compute_rows[b])
    assert any(e.graph is not None for e in tr._engines.values()), "the step graph was never captured"
    tr.cache.check_integrity()
    for l in range(3):
        w = tr.network.layers[l].weight.cpu().numpy()
        ow = otr.network.layers[l].weight
        assert np.linalg.norm(w - ow) <= 1e-3 * np.linalg.norm(ow), l


def test_c1_full_size_engine_lockstep_and_reference_golden():
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.data import synth_power_law_host
    gold = load_json("c1")
    src, dst, feats, labels, train, _, _ = synth_power_law_host(100_000, np.random.default_rng(0), 10, 128, 8)
    for k, v in [("src", src.astype(np.int64)), ("dst", dst.astype(np.int64)), ("features", feats),
                 ("labels", labels), ("train", train)]:
        assert sha(v) == gold["dataset"][k], k
    g = csr2_from_edges(src, dst, 100_000)
    assert sha(g[2]) == gold["csr2"]["col"]
    common = dict(fanouts=(15, 10, 5), hidden=256, batch_size=1024, epochs=1, eta=0.01, p_grad=0.9, t_stale=20,
                  seed=0)
    tr = hg.Trainer(g, feats, labels, train, hg.TrainConfig(kind=hg.LayerKind.SAGE_MEAN, **common), 8)
    otr = OTrainer(g, feats, labels, train, OTrainConfig(kind=SAGE, **common), 8)
    batches = hg.make_batches(train, tr.cfg)
    _lockstep(tr, otr, batches, 24, first_gold=gold["trainer_sage_0.9_20"][0])


def test_c2_products_shape_engine_lockstep():
    """The bench's own dataset and configuration (bench.py CONFIGS['c2'])."""
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.data import synth_power_law_host
    n = 2_400_000
    src, dst, feats, labels, train, _, _ = synth_power_law_host(n, np.random.default_rng(0), 13, 100, 47)
    g = csr2_from_edges(src, dst, n)
    del src, dst
    common = dict(fanouts=(15, 10, 5), hidden=256, batch_size=1024, epochs=1, eta=0.01, p_grad=0.9, t_stale=20,
                  seed=0)
    tr = hg.Trainer(g, feats, labels, train, hg.TrainConfig(kind=hg.LayerKind.SAGE_MEAN, **common), 47)
    otr = OTrainer(g, feats, labels, train, OTrainConfig(kind=SAGE, **common), 47)
    batches = hg.make_batches(train, tr.cfg)
    _lockstep(tr, otr, batches, 4)


@pytest.mark.parametrize("kind", [SAGE, GCN])
def test_plain_loop_matches_reference_golden(kind):
    """run_plain_loop (trainer.py:439-469) on the GPU against the reference's
    own run (tests/golden/trainer.npz): per-iteration losses and final
    weights within 1e-3 relative."""
    import paper_2301_07482_b200 as hg
    from oracle.datagen import power_law_dataset
    z = load("trainer")
    ds = power_law_dataset(3000, np.random.default_rng(0), m=4, feature_dim=16)
    g = csr2_from_edges(ds.src, ds.dst, ds.num_nodes)
    lk = hg.LayerKind.SAGE_MEAN if kind == SAGE else hg.LayerKind.GCN
    cfg = hg.TrainConfig(fanouts=(10, 5, 3), hidden=32, batch_size=128, epochs=1, eta=0.05, kind=lk, p_grad=0.0,
                         t_stale=0, seed=3)
    net, losses = hg.run_plain_loop(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
    np.testing.assert_allclose(losses, z[f"{kind}_plain_loss"], rtol=1e-3)
    for l in range(3):
        w, ref = net.layers[l].weight.cpu().numpy(), z[f"{kind}_plain_W{l}"]
        assert np.linalg.norm(w - ref) <= 1e-3 * np.linalg.norm(ref), l
        b, rb = net.layers[l].bias.cpu().numpy(), z[f"{kind}_plain_b{l}"]
        assert np.linalg.norm(b - rb) <= 1e-3 * max(np.linalg.norm(rb), 1e-6), l
