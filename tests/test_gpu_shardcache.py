"""Owner-sharded historical cache (paper_2301_07482_b200/
shardcache.py) against its oracle (oracle/shardcache.py + oracle/dp.py
dp_sharded_run).

- world 1: the sharded trainer is bitwise the per-process trainer (integer
  metrics, losses, weights), eager API path and CUDA-graph engine;
- world 2, two processes sharing one B200 over real CUDA IPC: every rank's
  integer metrics equal the sharded DP oracle's step by step (lockstep: the
  oracle's admission ranks each rank's GPU norms, SURVEY §8(c) Mode B), loss
  within 1e-3, both ranks end with identical weights; once through the eager
  path (gloo all-reduce) and once through the captured engine with the fused
  P2P all-reduce + SGD.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

FIELDS = ["fetched_bytes", "baseline_bytes", "prune_writes", "hits", "misses", "admissions", "gradient_evictions",
          "staleness_evictions", "forced_evictions", "feature_hits", "feature_misses", "valid_entries"]
POLICIES = {"t3": dict(p_grad=0.9, t_stale=3), "inf": dict(p_grad=0.9, t_stale=math.inf),
            "cap": dict(p_grad=1.0, t_stale=2, capacity=60), "refresh": dict(p_grad=0.6, t_stale=4,
                                                                            refresh_retained=True)}


def _data():
    from oracle.datagen import csr2_from_edges, power_law_dataset
    ds = power_law_dataset(1500, np.random.default_rng(2), m=3, feature_dim=8)
    return ds, csr2_from_edges(ds.src, ds.dst, ds.num_nodes)


def _cfg(hg, policy, sharding):
    return hg.TrainConfig(fanouts=(6, 4, 3), hidden=16, batch_size=48, epochs=1, eta=0.05,
                          kind=hg.LayerKind.SAGE_MEAN, seed=5, cache_sharding=sharding, **POLICIES[policy])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ------------------------------------------------------------------ world 1


def _world1_worker(rank, port, out_dir, policy):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    torch.cuda.set_device(0)
    import paper_2301_07482_b200 as hg
    ds, g = _data()
    res = {}
    for sharding in ("local", "owner"):
        for path in ("eager", "engine"):
            cfg = _cfg(hg, policy, sharding)
            tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
            batches = hg.make_batches(ds.train_ids, cfg)
            ms = []
            for i in range(14):
                if path == "eager":
                    m = tr.train_iteration(i, 0, tr.sample(i, batches[i]))
                else:
                    m = tr.train_step(i, 0, batches[i], next_batch=(i + 1, batches[i + 1]))
                ms.append([getattr(m, f) for f in FIELDS] + [m.loss])
            tr.cache.check_integrity()
            res[f"{sharding}_{path}_m"] = np.array(ms, dtype=np.float64)
            res[f"{sharding}_{path}_w"] = np.frombuffer(tr.network.checksum_bytes(), np.uint8)
            if sharding == "owner" and path == "engine":
                res["captures"] = np.array([sum(e.captures for e in tr._engines.values())])
    np.savez(os.path.join(out_dir, "w1.npz"), **res)
    dist.destroy_process_group()


@pytest.mark.parametrize("policy", sorted(POLICIES))
def test_world1_sharded_cache_is_the_local_cache(tmp_path, policy):
    mp.start_processes(_world1_worker, args=(_free_port(), str(tmp_path), policy), nprocs=1, join=True,
                       start_method="spawn")
    r = np.load(tmp_path / "w1.npz")
    for path in ("eager", "engine"):
        np.testing.assert_array_equal(r[f"owner_{path}_m"], r[f"local_{path}_m"], err_msg=path)
        np.testing.assert_array_equal(r[f"owner_{path}_w"], r[f"local_{path}_w"], err_msg=path)
    assert r["local_eager_m"][:, FIELDS.index("hits")].sum() > 0
    assert r["captures"][0] >= 1, "the sharded engine never captured its step graph"


# ------------------------------------------------------------------ world 2

WORLD, STEPS = 2, 6


def _world2_worker(rank, port, out_dir, policy, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.distributed import P2PAllReduce, make_allreduce_hook, rank_batch_indices
    ds, g = _data()
    cfg = _cfg(hg, policy, "owner")
    tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
    if path == "eager":
        tr.grad_hook = make_allreduce_hook(WORLD)
    else:
        tr.grad_hook = P2PAllReduce(tr.network.flat.numel(), rank, WORLD, "cuda", timeout_s=60.0)
    batches = hg.make_batches(ds.train_ids, cfg)
    idx = rank_batch_indices(len(batches), rank, WORLD)[:STEPS]
    ms, norms = [], {}
    for s, i in enumerate(idx):
        if path == "eager":
            m = tr.train_iteration(i, 0, tr.sample(i, batches[i]))
        else:
            nxt = (idx[s + 1], batches[idx[s + 1]]) if s + 1 < len(idx) else None
            m = tr.train_step(i, 0, batches[i], next_batch=nxt)
        ms.append([getattr(m, f) for f in FIELDS] + [m.loss])
        for l in (1, 2):
            norms[f"s{s}_l{l}"] = tr.last[3][l].cpu().numpy()
    tr.cache.check()
    if path != "eager":
        tr.grad_hook.check()
    tr.cache.check_integrity()
    out = dict(m=np.array(ms, dtype=np.float64), w=np.frombuffer(tr.network.checksum_bytes(), np.uint8),
               W=np.concatenate([tr.network.layers[l].weight.cpu().numpy().ravel() for l in range(3)]),
               row_of=np.stack([tr.cache.layers[l].row_of for l in (1, 2)]), **norms)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **out)
    torch.cuda.synchronize()
    dist.barrier()
    tr.cache.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("path", ["eager", "engine"])
@pytest.mark.parametrize("policy", ["t3", "cap", "refresh"])
def test_two_ranks_on_one_gpu_match_the_sharded_oracle(tmp_path, policy, path):
    from oracle.dp import dp_sharded_run
    from oracle.step import SAGE, OTrainConfig
    mp.start_processes(_world2_worker, args=(_free_port(), str(tmp_path), policy, path), nprocs=WORLD, join=True,
                       start_method="spawn")
    res = [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(WORLD)]
    np.testing.assert_array_equal(res[0]["w"], res[1]["w"])
    ds, g = _data()
    ocfg = OTrainConfig(fanouts=(6, 4, 3), hidden=16, batch_size=48, epochs=1, eta=0.05, kind=SAGE, seed=5,
                        **POLICIES[policy])
    metrics, onet, shared = dp_sharded_run(
        g, ds.features, ds.labels, ds.train_ids, ocfg, ds.num_classes, WORLD, STEPS,
        norms_for=lambda r, s: {l: res[r][f"s{s}_l{l}"] for l in (1, 2)})
    for r in range(WORLD):
        for s in range(STEPS):
            m = metrics[r][s]
            np.testing.assert_array_equal(res[r]["m"][s, :len(FIELDS)], [getattr(m, f) for f in FIELDS],
                                          err_msg=f"rank {r} step {s}")
            assert abs(res[r]["m"][s, -1] - m.loss) <= 1e-3 * abs(m.loss), (r, s)
    # the owners' maps together are the oracle's (ids owned elsewhere are -1 on each rank)
    for li, l in enumerate((1, 2)):
        got = np.maximum(res[0]["row_of"][li], res[1]["row_of"][li])
        want = np.full(ds.num_nodes, -1, np.int64)
        for o in range(WORLD):
            lo, hi = shared.bounds[o], shared.bounds[o + 1]
            want[lo:hi] = shared.owners[o][l].row_of[lo:hi]
        np.testing.assert_array_equal(got, want, err_msg=f"layer {l} row_of")
    hits = sum(res[r]["m"][:, FIELDS.index("hits")].sum() for r in range(WORLD))
    assert hits > 0, "the cache never served a hit: the test would be vacuous"
    W = res[0]["W"]
    oW = np.concatenate([onet.layers[l].weight.ravel() for l in range(3)])
    assert np.linalg.norm(W - oW) <= 1e-3 * np.linalg.norm(oW)
