"""Estimation / drift probes (histgnn/trainer.py:231-272,345-358; the
reference's own tests test_trainer.py:225-310 restated): host bookkeeping on
CPU, the device probes on the GPU."""

import math

import numpy as np
import pytest

from paper_2301_07482_b200.trainer import EmbeddingLog, cosine_rows


def test_embedding_log_records_and_cosine():
    log = EmbeddingLog()
    log.record(0, [1, 2, 3], np.array([[9.0, 9.0], [1.0, 0.0], [1.0, 1.0]]))
    log.record(4, [2, 3, 9], np.array([[1.0, np.sqrt(3.0)], [2.0, 2.0], [5.0, 5.0]]))
    assert log.similarity(4, 4) == pytest.approx(0.75)      # common nodes 2, 3: cos 0.5, 1.0
    assert log.similarity(4, 0) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        log.similarity(4, 5)
    with pytest.raises(ValueError):
        log.similarity(3, 1)


def test_cosine_rows_excludes_zero_rows():
    a = np.array([[1.0, 0.0], [0.0, 0.0], [1.0, 1.0]])
    b = np.array([[0.0, 1.0], [1.0, 0.0], [2.0, 2.0]])
    cos = cosine_rows(a, b)
    assert cos[0] == pytest.approx(0.0)
    assert np.isnan(cos[1])
    assert cos[2] == pytest.approx(1.0)


def _data(n, m, seed):
    from oracle.datagen import csr2_from_edges, power_law_dataset
    ds = power_law_dataset(n, np.random.default_rng(seed), m=m, feature_dim=8)
    return ds, csr2_from_edges(ds.src, ds.dst, ds.num_nodes)


@pytest.mark.gpu
def test_estimation_error_is_exactly_zero_without_cache():
    import paper_2301_07482_b200 as hg
    ds, g = _data(400, 3, 0)
    cfg = hg.TrainConfig(fanouts=(3, 3), hidden=8, batch_size=40, epochs=1, p_grad=0.0, t_stale=0,
                         probe_every=1, seed=0, kind=hg.LayerKind.SAGE_MEAN)
    tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
    metrics = tr.train()
    assert all(m.estimation_error == 0.0 for m in metrics)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["sage", "gcn", "gat"])
def test_stale_everything_cache_builds_up_estimation_error(kind):
    import paper_2301_07482_b200 as hg
    ds, g = _data(600, 4, 1)
    k = {"sage": hg.LayerKind.SAGE_MEAN, "gcn": hg.LayerKind.GCN, "gat": hg.LayerKind.GAT}[kind]
    cfg = hg.TrainConfig(fanouts=(4, 4), hidden=8, batch_size=60, epochs=3, eta=0.1, p_grad=1.0,
                         t_stale=math.inf, probe_every=1, seed=0, kind=k, heads=2)
    tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
    metrics = tr.train()
    assert hg.epoch_mean_estimation_error(metrics, cfg.epochs - 1) > 0.0
    assert not math.isnan(hg.epoch_mean_estimation_error(metrics, 0))
    # the probe changes nothing: the same run without probes trains identically
    cfg2 = hg.TrainConfig(fanouts=(4, 4), hidden=8, batch_size=60, epochs=3, eta=0.1, p_grad=1.0,
                          t_stale=math.inf, probe_every=0, seed=0, kind=k, heads=2)
    tr2 = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg2, ds.num_classes)
    m2 = [tr2.train_iteration(i, 0, tr2.sample(i, s)) for i, s in enumerate(hg.make_batches(ds.train_ids, cfg2))]
    assert [m.loss for m in metrics] == [m.loss for m in m2]
    assert tr.network.checksum_bytes() == tr2.network.checksum_bytes()


@pytest.mark.gpu
def test_trainer_fills_embedding_log_for_probe_nodes():
    import paper_2301_07482_b200 as hg
    ds, g = _data(300, 3, 4)
    cfg = hg.TrainConfig(fanouts=(4, 4), hidden=8, batch_size=30, epochs=2, p_grad=0.5, t_stale=10,
                         probe_every=1, seed=0, kind=hg.LayerKind.SAGE_MEAN)
    tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes, probe_nodes=np.arange(300))
    tr.train()
    assert len(tr.embedding_log.records) > 0
    t = max(tr.embedding_log.records)
    assert tr.embedding_log.similarity(t, 0) == pytest.approx(1.0)


def test_similarity_edge_cases_against_a_set_restatement():
    """Random snapshots (empty, disjoint, zero rows) against a dictionary
    restatement of trainer.py:253-272."""
    rng = np.random.default_rng(0)

    def slow(log, t, s):
        a, b = dict(zip(*map(list, log.records[t]))), dict(zip(*map(list, log.records[t - s])))
        cos = []
        for k in sorted(set(a) & set(b)):
            x, y = np.asarray(a[k], float), np.asarray(b[k], float)
            nx, ny = np.linalg.norm(x), np.linalg.norm(y)
            if nx > 0 and ny > 0:
                cos.append(float(x @ y) / (nx * ny))
        return float(np.mean(cos)) if cos else math.nan

    for _ in range(200):
        log = EmbeddingLog()
        for it in range(4):
            n = int(rng.integers(0, 8))
            rows = rng.standard_normal((n, 3))
            rows[rng.random(n) < 0.2] = 0.0
            log.record(it, rng.choice(12, size=n, replace=False), rows)
        for t in range(4):
            for s in range(t + 1):
                got, want = log.similarity(t, s), slow(log, t, s)
                assert (math.isnan(got) and math.isnan(want)) or got == pytest.approx(want, abs=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["sage_mean", "gcn"])
def test_probes_match_reference_golden(kind):
    """Free-running GPU trainer vs the reference's own probe values
    (tests/golden/probes.npz, make_golden.py gen_probes): a cache-everything
    run (p_grad 1, t_stale inf) whose admissions never depend on the norms,
    so the integer trajectory is identical and the estimation errors
    (trainer.py:345-358) and drift similarities (trainer.py:253-272) agree
    value for value within fp32 tolerance."""
    import os
    import paper_2301_07482_b200 as hg
    from oracle.datagen import csr2_from_edges, power_law_dataset
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "probes.npz"))
    ds = power_law_dataset(3000, np.random.default_rng(0), m=4, feature_dim=16)
    g = csr2_from_edges(ds.src, ds.dst, ds.num_nodes)
    lk = {"sage_mean": hg.LayerKind.SAGE_MEAN, "gcn": hg.LayerKind.GCN}[kind]
    cfg = hg.TrainConfig(fanouts=(4, 4), hidden=16, batch_size=64, epochs=2, eta=0.1, kind=lk, p_grad=1.0,
                         t_stale=math.inf, probe_every=1, seed=3)
    tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes,
                    probe_nodes=np.arange(0, ds.num_nodes, 7))
    ms = tr.train()
    names = list(z["int_names"])
    np.testing.assert_array_equal(np.array([[getattr(m, f) for f in names] for m in ms], np.int64),
                                  z[f"{kind}_ints"])
    np.testing.assert_allclose([m.loss for m in ms], z[f"{kind}_loss"], rtol=1e-3)
    est = np.array([m.estimation_error for m in ms])
    want = z[f"{kind}_est"]
    assert est[0] == 0.0 and want[0] == 0.0
    np.testing.assert_allclose(est, want, rtol=1e-3, atol=1e-6)
    pairs = z[f"{kind}_sim_pairs"]
    sim = np.array([tr.embedding_log.similarity(int(t), int(s)) for t, s in pairs])
    np.testing.assert_allclose(sim, z[f"{kind}_sim"], rtol=1e-4, atol=1e-6, equal_nan=True)
    last = max(tr.embedding_log.records)
    np.testing.assert_array_equal(tr.embedding_log.records[last][0], z[f"{kind}_log_ids_last"])
