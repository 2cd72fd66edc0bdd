"""GPU prune + lookup bit-exact vs the reference (golden prune_nn.npz), and the
block convolutions / backward within 1e-3 relative of the reference's fp32."""

import math

import numpy as np
import pytest

from oracle.datagen import power_law_dataset
from tests.goldens import golden_sub, load
from tests.gpu_helpers import assert_close, dev_sub_from_golden

pytestmark = pytest.mark.gpu

CNAMES = sorted(("hits", "misses", "admissions", "gradient_evictions", "staleness_evictions",
                 "forced_evictions", "staleness_violations", "feature_hits", "feature_misses"))
_DS = {}


def _pl3000():
    if "ds" not in _DS:
        _DS["ds"] = power_law_dataset(3000, np.random.default_rng(0), m=4, feature_dim=16)
    return _DS["ds"]


def _setup(case, hidden=8):
    import paper_2301_07482_b200 as hg
    z = load("prune_nn")
    seeds, blocks = golden_sub(z, f"p{case}_orig")
    sub = dev_sub_from_golden(seeds, blocks)
    cache = hg.HistCache(3000, [hidden, hidden], hg.CachePolicy(1.0, math.inf))
    for layer in (1, 2):
        ids = z[f"p{case}_pre{layer}"]
        if len(ids):
            emb = (ids[:, None] * 10.0 + layer + np.arange(hidden)).astype(np.float32)
            cache.update_cache(layer, ids, ids, emb, np.zeros(len(ids)), 0)
    return z, sub, cache


@pytest.mark.parametrize("case", range(3))
def test_prune_matches_reference(case):
    import paper_2301_07482_b200 as hg
    z, sub, cache = _setup(case)
    before = cache.counters()
    pr = hg.prune_with_cache(sub, cache, 1)
    for b in range(4):
        np.testing.assert_array_equal(pr.layer_live[b].cpu().numpy(), z[f"p{case}_live{b}"], err_msg=f"live {b}")
    for b in range(3):
        np.testing.assert_array_equal(pr.compute_rows[b].cpu().numpy(), z[f"p{case}_rows{b}"], err_msg=f"rows {b}")
        inj = pr.injected_np(b)
        want_loc = z[f"p{case}_inj{b}_loc"]
        if inj is None:
            assert len(want_loc) == 0
        else:
            np.testing.assert_array_equal(inj[0], want_loc)
            np.testing.assert_array_equal(inj[1], z[f"p{case}_inj{b}_val"])
        assert sub.layers[b].adj.prune_writes == int(z[f"p{case}_pruned_b{b}_prune_writes"])
        np.testing.assert_array_equal(sub.layers[b].adj.end_np, z[f"p{case}_pruned_b{b}_end"])
    after = cache.counters()
    # reference counters include the preload (admissions), compare totals
    np.testing.assert_array_equal([after[k] for k in CNAMES], z[f"p{case}_counters"])
    assert after["admissions"] == before["admissions"]


@pytest.mark.parametrize("case", range(3))
@pytest.mark.parametrize("kind", ["sage_mean", "gcn"])
def test_nn_matches_reference(case, kind):
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.nn import network_from_numpy
    z, sub, cache = _setup(case)
    pr = hg.prune_with_cache(sub, cache, 1)
    k = f"p{case}_{kind}_"
    lk = hg.LayerKind(kind)
    layers = [{"weight": z[k + f"W{l}"], "bias": np.zeros(z[k + f"W{l}"].shape[1], np.float32),
               "weight_neigh": z[k + f"Wn{l}"] if kind == "sage_mean" else None} for l in range(3)]
    net = network_from_numpy(lk, layers)
    ds = _pl3000()
    b0 = sub.layers[0]
    h0 = np.zeros((b0.num_src, 16), np.float32)
    live0 = pr.layer_live[0].cpu().numpy()
    h0[live0] = ds.features[b0.src_nodes.cpu().numpy()[live0]]
    tape = hg.forward_pass(net, sub.layers, h0, pr.compute_rows, pr.injected)
    loss, dl = hg.cross_entropy(tape.logits, ds.labels[sub.seeds])
    grads, ng, dinp = hg.backward(net, sub.layers, tape, dl)
    assert abs(loss - float(z[k + "loss"])) <= 1e-3 * abs(float(z[k + "loss"]))
    for l in range(3):
        assert_close(tape.h_layer_np(l), z[k + f"h{l}"], what=f"h{l}")
        assert_close(ng[l].cpu().numpy(), z[k + f"ng{l}"], what=f"node grad {l}")
        g = grads[l].numpy()
        assert_close(g["weight"], z[k + f"gW{l}"], what=f"dW{l}")
        assert_close(g["bias"], z[k + f"gb{l}"], what=f"db{l}")
        if kind == "sage_mean":
            assert_close(g["weight_neigh"], z[k + f"gWn{l}"], what=f"dWn{l}")
    assert_close(dinp.cpu().numpy(), z[k + "dinput"], what="d_input")


def test_node_grad_norms_and_sgd_exact():
    import paper_2301_07482_b200 as hg
    from oracle.step import node_grad_norms as onorms
    rng = np.random.default_rng(0)
    g = rng.standard_normal((257, 37)).astype(np.float32)
    np.testing.assert_allclose(hg.node_grad_norms(g).cpu().numpy(), onorms(g), rtol=1e-12)
    net = hg.init_network(hg.LayerKind.SAGE_MEAN, [8, 4, 3], np.random.default_rng(1))
    before = net.flat.cpu().numpy().copy()
    grads = net.new_grads()
    grads.flat.copy_(__import__("torch").as_tensor(rng.standard_normal(before.shape).astype(np.float32)))
    hg.sgd_step(net, grads, 0.01)
    want = before - np.float32(0.01) * grads.flat.cpu().numpy()
    np.testing.assert_array_equal(net.flat.cpu().numpy(), want)
