"""Data-parallel GPU path with two ranks sharing one B200 (gloo carries the
CUDA-tensor all-reduce because NCCL refuses duplicate GPUs): both ranks end
with bitwise-identical weights, and step 0 (no cache history yet) matches the
serial DP oracle's loss within 1e-3 and its integer metrics exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD, STEPS = 2, 4


def _data():
    from oracle.datagen import csr2_from_edges, power_law_dataset
    ds = power_law_dataset(1500, np.random.default_rng(2), m=3, feature_dim=8)
    return ds, csr2_from_edges(ds.src, ds.dst, ds.num_nodes)


def _worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.distributed import make_allreduce_hook, rank_batch_indices
    ds, g = _data()
    cfg = hg.TrainConfig(fanouts=(6, 4, 3), hidden=16, batch_size=96, epochs=1, eta=0.05,
                         kind=hg.LayerKind.SAGE_MEAN, p_grad=0.9, t_stale=3, seed=5)
    tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
    tr.grad_hook = make_allreduce_hook(WORLD)
    batches = hg.make_batches(ds.train_ids, cfg)
    ms = []
    for idx in rank_batch_indices(len(batches), rank, WORLD)[:STEPS]:
        m = tr.train_iteration(idx, 0, tr.sample(idx, batches[idx]))
        ms.append([m.hits, m.misses, m.admissions, m.fetched_bytes, m.prune_writes, m.loss])
    np.save(os.path.join(out_dir, f"r{rank}_metrics.npy"), np.array(ms, dtype=np.float64))
    np.save(os.path.join(out_dir, f"r{rank}_w.npy"), np.frombuffer(tr.network.checksum_bytes(), np.uint8))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_dp_on_one_gpu(tmp_path):
    from oracle.dp import dp_serial_run
    from oracle.step import SAGE, OTrainConfig
    mp.start_processes(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True, start_method="spawn")
    w0 = np.load(tmp_path / "r0_w.npy")
    w1 = np.load(tmp_path / "r1_w.npy")
    np.testing.assert_array_equal(w0, w1)
    ds, g = _data()
    ocfg = OTrainConfig(fanouts=(6, 4, 3), hidden=16, batch_size=96, epochs=1, eta=0.05, kind=SAGE,
                        p_grad=0.9, t_stale=3, seed=5)
    metrics, _ = dp_serial_run(g, ds.features, ds.labels, ds.train_ids, ocfg, ds.num_classes, WORLD, 1)
    for r in range(WORLD):
        got = np.load(tmp_path / f"r{r}_metrics.npy")[0]
        m = metrics[r][0]
        np.testing.assert_array_equal(got[:5], [m.hits, m.misses, m.admissions, m.fetched_bytes, m.prune_writes])
        assert abs(got[5] - m.loss) <= 1e-3 * abs(m.loss)


def _nccl_worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.distributed import make_allreduce_hook
    ds, g = _data()
    cfg = hg.TrainConfig(fanouts=(6, 4, 3), hidden=16, batch_size=96, epochs=1, eta=0.05,
                         kind=hg.LayerKind.SAGE_MEAN, p_grad=0.9, t_stale=3, seed=5)
    out = []
    for hooked in (False, True):
        tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
        if hooked:
            tr.grad_hook = make_allreduce_hook(1)
            assert tr.grad_hook.graph_safe
        batches = hg.make_batches(ds.train_ids, cfg)
        losses = [tr.train_step(i, 0, batches[i], next_batch=(i + 1, batches[i + 1])).loss for i in range(8)]
        caps = sum(e.captures for e in tr._engines.values())
        out.append((losses, caps, np.frombuffer(tr.network.checksum_bytes(), np.uint8)))
    np.save(os.path.join(out_dir, "losses.npy"), np.array([o[0] for o in out]))
    np.save(os.path.join(out_dir, "caps.npy"), np.array([o[1] for o in out]))
    np.save(os.path.join(out_dir, "w.npy"), np.stack([o[2] for o in out]))
    dist.destroy_process_group()


def test_nccl_allreduce_is_captured_in_the_step_graph(tmp_path):
    """A single-rank NCCL group: the all-reduce hook is recorded inside the
    step's CUDA graph (the N>1 bench path) and changes nothing numerically."""
    mp.start_processes(_nccl_worker, args=(_free_port(), str(tmp_path)), nprocs=1, join=True, start_method="spawn")
    caps = np.load(tmp_path / "caps.npy")
    assert caps[1] >= 1, "the hooked trainer never captured a CUDA graph"
    losses = np.load(tmp_path / "losses.npy")
    np.testing.assert_array_equal(losses[0], losses[1])
    w = np.load(tmp_path / "w.npy")
    np.testing.assert_array_equal(w[0], w[1])


def _p2p_worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.distributed import P2PAllReduce, make_allreduce_hook, rank_batch_indices
    ds, g = _data()
    cfg = hg.TrainConfig(fanouts=(6, 4, 3), hidden=16, batch_size=96, epochs=1, eta=0.05,
                         kind=hg.LayerKind.SAGE_MEAN, p_grad=0.9, t_stale=3, seed=5)
    out = {}
    for mode in ("gloo", "p2p"):
        tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
        ex = None
        if mode == "gloo":
            tr.grad_hook = make_allreduce_hook(WORLD)
        else:
            ex = P2PAllReduce(tr.network.flat.numel(), rank, WORLD, "cuda:0")
            tr.grad_hook = ex
        batches = hg.make_batches(ds.train_ids, cfg)
        idx = rank_batch_indices(len(batches), rank, WORLD)[:6]
        losses = []
        for k, i in enumerate(idx):
            nb = (idx[k + 1], batches[idx[k + 1]]) if k + 1 < len(idx) else None
            losses.append(tr.train_step(i, 0, batches[i], next_batch=nb).loss)
        torch.cuda.synchronize()
        caps = sum(e.captures for e in tr._engines.values())
        out[mode] = (np.array(losses), caps, np.frombuffer(tr.network.checksum_bytes(), np.uint8).copy())
        if ex is not None:
            assert not ex.timed_out
            ex.close()
    np.save(os.path.join(out_dir, f"p{rank}_losses.npy"), np.stack([out["gloo"][0], out["p2p"][0]]))
    np.save(os.path.join(out_dir, f"p{rank}_caps.npy"), np.array([out["gloo"][1], out["p2p"][1]]))
    np.save(os.path.join(out_dir, f"p{rank}_w.npy"), np.stack([out["gloo"][2], out["p2p"][2]]))
    dist.destroy_process_group()


def test_p2p_fused_allreduce_sgd_matches_gloo(tmp_path):
    """Two processes on one GPU exchange gradients through CUDA-IPC slots with
    hg_p2p_allreduce_sgd (captured in the step graph, no host collective per
    step): both ranks end bitwise equal, and equal to the gloo all-reduce +
    hg_sgd path ((g0 + g1) / 2 is the same float either way for P = 2)."""
    mp.start_processes(_p2p_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True,
                       start_method="spawn")
    w = [np.load(tmp_path / f"p{r}_w.npy") for r in range(WORLD)]
    np.testing.assert_array_equal(w[0][1], w[1][1])
    np.testing.assert_array_equal(w[0][0], w[0][1])
    for r in range(WORLD):
        caps = np.load(tmp_path / f"p{r}_caps.npy")
        assert caps[1] >= 1, "the P2P step was never captured in a CUDA graph"
        losses = np.load(tmp_path / f"p{r}_losses.npy")
        np.testing.assert_array_equal(losses[0], losses[1])
