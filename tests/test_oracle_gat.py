"""GAT oracle (oracle/gat.py) — no reference implementation exists
(histgnn/nn.py:28-30 has GCN / SAGE_MEAN only), so the restatement is pinned
the way the reference pins its own layers (test_nn.py:27-46,148-160,271-309):
against a dense formulation and by finite differences, in float64."""

import numpy as np
import pytest

from oracle import gat
from oracle.datagen import csr2_from_edges, power_law_dataset
from oracle.sampling import sample_layered
from oracle.step import GAT, OTrainConfig, OTrainer, make_batches


class _Blk:
    def __init__(self, start, end, col, num_src, num_dst):
        self.start, self.end, self.col = start, end, col
        self.num_src, self.num_dst = num_src, num_dst


def _block(rng, n_dst=7, n_src=15, max_deg=5):
    deg = rng.integers(0, max_deg + 1, size=n_dst)
    start = np.concatenate([[0], np.cumsum(deg)[:-1]]).astype(np.int64)
    end = start + deg
    col = rng.integers(0, n_src, size=int(deg.sum())).astype(np.int64)
    return _Blk(start, end, col, n_src, n_dst)


def _params(rng, fi, fo, heads, dt=np.float64):
    p = gat.init_layer(rng, fi, fo, heads, dt)
    p.bias = rng.normal(size=fo).astype(dt) * 0.1
    return p


@pytest.mark.parametrize("heads", [1, 4])
def test_forward_matches_dense(heads):
    rng = np.random.default_rng(0)
    blk = _block(rng)
    p = _params(rng, 6, 8, heads)
    h = rng.normal(size=(blk.num_src, 6))
    rows = np.array([0, 2, 3, 6])
    out, _ = gat.layer_forward(p, blk, h, rows, act=True)
    adj = [blk.col[blk.start[r]:blk.end[r]] for r in rows]
    ref = gat.dense_forward(p, adj, h, rows, act=True)
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("heads", [1, 2])
def test_backward_matches_finite_differences(heads):
    rng = np.random.default_rng(1)
    blk = _block(rng, n_dst=5, n_src=9, max_deg=4)
    p = _params(rng, 4, 6, heads)
    h = rng.normal(size=(blk.num_src, 4))
    rows = np.array([0, 1, 3, 4])
    G = rng.normal(size=(len(rows), 6))

    def loss(pp, hh):
        out, _ = gat.layer_forward(pp, blk, hh, rows, act=False)
        return float((out * G).sum())

    _, t = gat.layer_forward(p, blk, h, rows, act=False)
    g, d_in = gat.layer_backward(p, t, G)
    eps = 1e-6
    for name in ("weight", "bias", "att_src", "att_dst"):
        a = getattr(p, name)
        num = np.zeros_like(a)
        for idx in np.ndindex(a.shape):
            old = a[idx]
            a[idx] = old + eps
            lp = loss(p, h)
            a[idx] = old - eps
            lm = loss(p, h)
            a[idx] = old
            num[idx] = (lp - lm) / (2 * eps)
        np.testing.assert_allclose(getattr(g, name), num, rtol=1e-6, atol=1e-7, err_msg=name)
    num = np.zeros_like(h)
    for idx in np.ndindex(h.shape):
        old = h[idx]
        h[idx] = old + eps
        lp = loss(p, h)
        h[idx] = old - eps
        lm = loss(p, h)
        h[idx] = old
        num[idx] = (lp - lm) / (2 * eps)
    np.testing.assert_allclose(d_in, num, rtol=1e-6, atol=1e-7)


def test_gat_trainer_runs_with_cache():
    ds = power_law_dataset(1200, np.random.default_rng(3), m=3, feature_dim=8)
    g = csr2_from_edges(ds.src, ds.dst, ds.num_nodes)
    cfg = OTrainConfig(fanouts=(5, 4, 3), hidden=16, batch_size=64, eta=0.05, kind=GAT, p_grad=0.9, t_stale=3,
                       seed=1, heads=4)
    tr = OTrainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
    batches = make_batches(ds.train_ids, cfg)
    ms = [tr.train_iteration(i, 0, tr.sample(i, batches[i])) for i in range(6)]
    assert all(np.isfinite(m.loss) for m in ms)
    assert sum(m.hits for m in ms) > 0          # the historical cache is exercised
    assert tr.network.layers[0].heads == 4 and tr.network.layers[-1].heads == 1
