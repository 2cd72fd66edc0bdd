"""The owner-sharded cache oracle (oracle/shardcache.py, oracle/dp.py
dp_sharded_run) on CPU: with one owner it is the reference's sequential
cache (pinned to the reference through OTrainer, tests/test_oracle_golden.py);
with several, every owner's ring is internally consistent, holds only its own
ids, never serves an entry older than t_stale, and every hit returns the
value of that node's latest admission."""

import math

import numpy as np
import pytest

from oracle.datagen import csr2_from_edges, power_law_dataset
from oracle.dp import dp_sharded_run
from oracle.shardcache import OShardedCache, owner_ranges
from oracle.histcache import OCachePolicy
from oracle.step import INT_METRICS, SAGE, OTrainConfig, OTrainer, make_batches

POLICIES = [dict(p_grad=0.9, t_stale=3), dict(p_grad=0.9, t_stale=math.inf), dict(p_grad=1.0, t_stale=2, capacity=40),
            dict(p_grad=0.6, t_stale=4, refresh_retained=True)]


@pytest.fixture(scope="module")
def data():
    ds = power_law_dataset(1200, np.random.default_rng(2), m=3, feature_dim=8)
    return ds, csr2_from_edges(ds.src, ds.dst, ds.num_nodes)


def _cfg(**pol):
    return OTrainConfig(fanouts=(6, 4, 3), hidden=16, batch_size=48, epochs=1, eta=0.05, kind=SAGE, seed=5, **pol)


@pytest.mark.parametrize("pol", POLICIES)
def test_one_owner_is_the_sequential_cache(data, pol):
    ds, g = data
    cfg = _cfg(**pol)
    ms, _, _ = dp_sharded_run(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes, 1, 10)
    tr = OTrainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
    b = make_batches(ds.train_ids, cfg)
    for it in range(10):
        m = tr.train_iteration(it, 0, tr.sample(it, b[it]))
        assert [getattr(ms[0][it], f) for f in INT_METRICS] == [getattr(m, f) for f in INT_METRICS], it
        assert ms[0][it].loss == m.loss


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("pol", POLICIES)
def test_owner_rings_are_consistent(data, pol, world):
    ds, g = data
    ms, _, sh = dp_sharded_run(g, ds.features, ds.labels, ds.train_ids, _cfg(**pol), ds.num_classes, world, 5)
    assert sum(m.hits for r in ms for m in r) > 0
    for o in range(world):
        lo, hi = sh.bounds[o], sh.bounds[o + 1]
        for ring in sh.owners[o].values():
            held = np.flatnonzero(ring.row_of >= 0)
            assert np.all((held >= lo) & (held < hi))
            rows = ring.row_of[held]
            assert len(np.unique(rows)) == len(rows)
            if ring.row_owner is not None:
                np.testing.assert_array_equal(ring.row_owner[rows], held)
                assert ring.capacity <= hi - lo
        assert ms[o][-1].valid_entries == sh.owner_valid(o)


def test_lookups_are_pure_reads_and_serve_latest_admissions():
    """Scripted: two ranks look up the same ids in one step; an expiry found
    by one rank does not change the other's answer; the commit applies it once."""
    sh = OShardedCache(10, [2], OCachePolicy(1.0, 2), 2)
    ids = np.arange(10)
    v0 = sh.view(0)
    v0.update_cache(1, ids, ids, np.arange(20, dtype=np.float32).reshape(10, 2), np.zeros(10), 0)
    v0.end_iteration(0)
    sh.commit([v0, sh.view(1)])
    # step: rank 0 at it 2 (fresh: age 2 <= 2), rank 1 at it 3 (expired)
    a, b = sh.view(0), sh.view(1)
    h0, vals0, _ = a.lookup(1, ids, 2)
    h1, _, m1 = b.lookup(1, ids, 3)
    assert len(h0) == 10 and len(h1) == 0 and len(m1) == 10
    np.testing.assert_array_equal(vals0, np.arange(20, dtype=np.float32).reshape(10, 2))
    before = sum(sh.owner_counters(o)["staleness_evictions"] for o in range(2))
    sh.commit([a, b])
    after = sum(sh.owner_counters(o)["staleness_evictions"] for o in range(2))
    assert after - before == 10
    assert sum(sh.owner_valid(o) for o in range(2)) == 0


def test_owner_ranges_match_the_product():
    from paper_2301_07482_b200.distributed import owner_ranges as product
    for n, p in [(10, 3), (7, 7), (100, 8), (5, 1)]:
        np.testing.assert_array_equal(owner_ranges(n, p), product(n, p))
