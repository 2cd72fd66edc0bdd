"""GPU sampler parity: blocks bit-identical to the reference's (golden vectors
from tests/golden/make_golden.py) and to the oracle, incl. hubs wider than a
warp / than 2048 candidates, fanout > 32, multigraph self loops, reused RNGs."""

import numpy as np
import pytest
import torch

from oracle.datagen import csr2_from_edges, power_law_dataset
from oracle.sampling import batch_rng as obatch_rng
from oracle.sampling import sample_layered as osample
from tests.goldens import assert_sub_equal, golden_sub, load, load_json, sha

pytestmark = pytest.mark.gpu


def _hg():
    import paper_2301_07482_b200 as hg
    return hg


def _dev_graph(z, tag):
    hg = _hg()
    return hg.csr2_from_arrays(z[f"{tag}_start"], z[f"{tag}_end"], z[f"{tag}_col"])


def _np_blocks(sub):
    return [b.as_numpy() for b in sub.layers]


def test_path_graph():
    hg = _hg()
    z = load("sampler")
    g = hg.build_csr2(hg.CooGraph([0, 1], [1, 2], 3))
    sub = hg.sample_layered(g, [2], hg.SamplePlan((1, 1), 1, 0), np.random.default_rng(0))
    _, blocks = golden_sub(z, "path")
    assert_sub_equal(_np_blocks(sub), blocks)


@pytest.mark.parametrize("tag,graph,fanouts,seed,idx", [
    ("multi", "multi", (3, 3, 3), 17, 3),
    ("star", "star", (20, 40), 9, 1),
    ("pl0", "pl", (15, 10, 5), 0, 0),
    ("pl1", "pl", (15, 10, 5), 0, 1),
    ("pl2", "pl", (15, 10, 5), 0, 2),
])
def test_matches_reference_golden(tag, graph, fanouts, seed, idx):
    hg = _hg()
    z = load("sampler")
    g = _dev_graph(z, graph)
    seeds, blocks = golden_sub(z, tag)
    rng = hg.batch_rng(seed, idx)
    sub = hg.sample_layered(g, seeds, hg.SamplePlan(fanouts, len(seeds), seed), rng)
    assert_sub_equal(_np_blocks(sub), blocks)
    # the caller's generator advanced exactly like rng.random(total) would
    total = 0
    s, e, c = z[f"{graph}_start"], z[f"{graph}_end"], z[f"{graph}_col"]
    fr = seeds
    for i, f in enumerate(fanouts):
        total += int(np.sum(e[fr] - s[fr]))
        fr = blocks[len(blocks) - 1 - i]["src"]
    ref2 = obatch_rng(seed, idx)
    ref2.random(total)
    assert rng.random() == ref2.random()


def test_reused_generator_continues_stream():
    hg = _hg()
    z = load("sampler")
    g = _dev_graph(z, "multi")
    r = np.random.default_rng(11)
    for tag in ("reuse0", "reuse1"):
        seeds, blocks = golden_sub(z, tag)
        sub = hg.sample_layered(g, seeds, hg.SamplePlan((4, 2), 6, 0), r)
        assert_sub_equal(_np_blocks(sub), blocks)


def test_seed_validation_errors():
    hg = _hg()
    g = hg.build_csr2(hg.CooGraph([0, 1], [1, 2], 3))
    plan = hg.SamplePlan((1,), 1, 0)
    for bad in ([], [1, 1], [5], [-1]):
        with pytest.raises(ValueError):
            hg.sample_layered(g, bad, plan, np.random.default_rng(0))
    with pytest.raises(ValueError):
        hg.SamplePlan((), 1)


@pytest.mark.parametrize("fanouts", [(1,), (2, 2), (33, 3), (64,)])
def test_random_multigraph_vs_oracle(fanouts):
    hg = _hg()
    rng = np.random.default_rng(123)
    n, m = 300, 4000
    src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
    s, e, c = csr2_from_edges(src, dst, n)
    g = hg.csr2_from_arrays(s, e, c)
    for idx in range(3):
        seeds = rng.choice(n, size=40, replace=False)
        want = osample(s, e, c, n, seeds, fanouts, obatch_rng(5, idx))
        got = hg.sample_layered(g, seeds, hg.SamplePlan(fanouts, 40, 5), hg.batch_rng(5, idx))
        assert_sub_equal(_np_blocks(got), [
            {"dst": b.dst_nodes, "src": b.src_nodes, "start": b.start, "end": b.end, "col": b.col,
             "dst_deg": b.dst_deg, "src_deg": b.src_deg} for b in want.layers])


def test_zero_degree_rows_and_isolated_seeds():
    hg = _hg()
    s, e, c = csr2_from_edges([0, 1, 2], [1, 2, 3], 6)
    g = hg.csr2_from_arrays(s, e, c)
    want = osample(s, e, c, 6, [5, 0, 3], (2, 2), obatch_rng(1, 1))
    got = hg.sample_layered(g, [5, 0, 3], hg.SamplePlan((2, 2), 3), hg.batch_rng(1, 1))
    assert_sub_equal(_np_blocks(got), [
        {"dst": b.dst_nodes, "src": b.src_nodes, "start": b.start, "end": b.end, "col": b.col,
         "dst_deg": b.dst_deg, "src_deg": b.src_deg} for b in want.layers])


def test_c1_subgraphs_match_reference_hashes():
    """Config C1 (100K nodes / 2M edges, fanout 15,10,5, batch 1024)."""
    hg = _hg()
    gold = load_json("c1")
    ds = power_law_dataset(100_000, np.random.default_rng(0), m=10, feature_dim=128)
    g = hg.build_csr2(hg.CooGraph(ds.src, ds.dst, ds.num_nodes))
    assert sha(g.col_np) == gold["csr2"]["col"]
    cfg = hg.TrainConfig(fanouts=(15, 10, 5), hidden=256, batch_size=1024, kind=hg.LayerKind.SAGE_MEAN)
    batches = hg.make_batches(ds.train_ids, cfg)
    plan = hg.SamplePlan(cfg.fanouts, 1024, 0)
    for idx in ("0", "1", "7"):
        sub = hg.sample_layered(g, batches[int(idx)], plan, hg.batch_rng(0, int(idx)))
        want = gold["subgraphs"][idx]
        for i, b in enumerate(sub.layers):
            nb = b.as_numpy()
            assert sha(nb["src"]) == want[f"b{i}_src"]
            assert sha(nb["col"]) == want[f"b{i}_col"]
            assert sha(nb["start"]) == want[f"b{i}_start"]
            assert sha(nb["dst_deg"]) == want[f"b{i}_dst_deg"]
        assert [[b.num_dst, b.num_src, b.num_edges_built] for b in sub.layers] == want["sizes"]


def test_producer_matches_sequential():
    hg = _hg()
    z = load("sampler")
    g = _dev_graph(z, "pl")
    rng = np.random.default_rng(3)
    batches = [rng.choice(3000, size=64, replace=False) for _ in range(5)]
    plan = hg.SamplePlan((5, 3), 64, 4)
    seq = [hg.sample_layered(g, b, plan, hg.batch_rng(4, i)) for i, b in enumerate(batches)]
    with hg.SubgraphProducer(g, batches, plan, queue_capacity=2) as prod:
        got = list(prod)
    assert [i for i, _ in got] == list(range(5))
    for (_, a), b in zip(got, seq):
        assert_sub_equal(_np_blocks(a), _np_blocks(b))


@pytest.mark.parametrize("fanouts", [(5, 3), (15, 10), (32,)])
def test_hub_rows_split_across_warps_vs_oracle(fanouts):
    """Rows with more than 1024 candidates take the segmented hub path
    (512-candidate segments, merged by the warp finishing a row's last
    segment): several hubs of 4097 .. 30000 in-edges (multi-edges and ties
    included) must sample bit-exactly like the oracle."""
    hg = _hg()
    rng = np.random.default_rng(77)
    n = 40000
    hubs = [0, 1, 2, 3, 7]
    degs = [4097, 6000, 12345, 30000, 8192]
    src = [rng.integers(0, n, d) for d in degs]
    dst = [np.full(d, h) for h, d in zip(hubs, degs)]
    # background edges so the second layer has ordinary rows too
    bs, bd = rng.integers(0, n, 60000), rng.integers(0, n, 60000)
    s, e, c = csr2_from_edges(np.concatenate(src + [bs]), np.concatenate(dst + [bd]), n)
    g = hg.csr2_from_arrays(s, e, c)
    for idx in range(3):
        seeds = np.concatenate([hubs, rng.choice(np.arange(10, n), size=59, replace=False)])
        want = osample(s, e, c, n, seeds, fanouts, obatch_rng(9, idx))
        got = hg.sample_layered(g, seeds, hg.SamplePlan(fanouts, len(seeds), 9), hg.batch_rng(9, idx))
        assert_sub_equal(_np_blocks(got), [
            {"dst": b.dst_nodes, "src": b.src_nodes, "start": b.start, "end": b.end, "col": b.col,
             "dst_deg": b.dst_deg, "src_deg": b.src_deg} for b in want.layers])


@pytest.mark.parametrize("fanout", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17, 31, 32])
def test_every_selection_path_vs_oracle(fanout):
    """In-degrees spread over 0 .. 3000 so one layer mixes rows on every
    selection path of k_select_all -- one row per thread (<= 64 candidates,
    each register-network width kF), one row per warp (65 .. 1024, packed and
    first-chunk paths) and 512-candidate hub segments (> 1024) -- for every
    fanout the templates distinguish; bit-exact with the oracle."""
    hg = _hg()
    rng = np.random.default_rng(1000 + fanout)
    n = 6000
    degs = np.concatenate([rng.integers(0, 70, n - 60), rng.integers(60, 1100, 50), rng.integers(1000, 3000, 10)])
    dst = np.repeat(np.arange(n), degs)
    src = rng.integers(0, n, len(dst))
    s, e, c = csr2_from_edges(src, dst, n)
    g = hg.csr2_from_arrays(s, e, c)
    for idx in range(2):
        seeds = np.concatenate([np.arange(n - 60, n), rng.choice(n - 60, size=200, replace=False)])
        want = osample(s, e, c, n, seeds, (fanout, 2), obatch_rng(3, idx))
        got = hg.sample_layered(g, seeds, hg.SamplePlan((fanout, 2), len(seeds), 3), hg.batch_rng(3, idx))
        assert_sub_equal(_np_blocks(got), [
            {"dst": b.dst_nodes, "src": b.src_nodes, "start": b.start, "end": b.end, "col": b.col,
             "dst_deg": b.dst_deg, "src_deg": b.src_deg} for b in want.layers])
