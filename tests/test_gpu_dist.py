"""Data-parallel GPU path with two ranks sharing one B200 (gloo carries the
CUDA-tensor all-reduce because NCCL refuses duplicate GPUs): both ranks end
with bitwise-identical weights, and every step matches the serial DP oracle
(oracle/dp.py) in lockstep (its cache admission fed each rank's GPU norms):
integer metrics exact, loss within 1e-3, final weights within 1e-3."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD, STEPS = 2, 5


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
    ms, norms = [], {}
    for s, idx in enumerate(rank_batch_indices(len(batches), rank, WORLD)[:STEPS]):
        m = tr.train_iteration(idx, 0, tr.sample(idx, batches[idx]))
        ms.append([getattr(m, f) for f in FIELDS] + [m.loss])
        for l in (1, 2):
            norms[f"s{s}_l{l}"] = tr.last[3][l].cpu().numpy()
    np.save(os.path.join(out_dir, f"r{rank}_metrics.npy"), np.array(ms, dtype=np.float64))
    np.savez(os.path.join(out_dir, f"r{rank}_norms.npz"), **norms)
    np.save(os.path.join(out_dir, f"r{rank}_W.npy"), np.concatenate([tr.network.layers[l].weight.cpu().numpy().ravel()
                                                                    for l in range(3)]))
    np.save(os.path.join(out_dir, f"r{rank}_w.npy"), np.frombuffer(tr.network.checksum_bytes(), np.uint8))
    dist.destroy_process_group()


FIELDS = ["fetched_bytes", "baseline_bytes", "prune_writes", "hits", "misses", "admissions", "gradient_evictions",
          "staleness_evictions", "forced_evictions", "feature_hits", "feature_misses", "valid_entries"]


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
    nz = [dict(np.load(tmp_path / f"r{r}_norms.npz")) for r in range(WORLD)]
    metrics, onet = dp_serial_run(g, ds.features, ds.labels, ds.train_ids, ocfg, ds.num_classes, WORLD, STEPS,
                                  norms_for=lambda r, s: {l: nz[r][f"s{s}_l{l}"] for l in (1, 2)})
    for r in range(WORLD):
        got = np.load(tmp_path / f"r{r}_metrics.npy")
        for s in range(STEPS):
            m = metrics[r][s]
            np.testing.assert_array_equal(got[s, :len(FIELDS)], [getattr(m, f) for f in FIELDS],
                                          err_msg=f"rank {r} step {s}")
            assert abs(got[s, -1] - m.loss) <= 1e-3 * abs(m.loss), (r, s)
    W = np.load(tmp_path / "r0_W.npy")
    oW = np.concatenate([onet.layers[l].weight.ravel() for l in range(3)])
    assert np.linalg.norm(W - oW) <= 1e-3 * np.linalg.norm(oW)


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


def _timeout_worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    torch.cuda.set_device(0)
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.distributed import P2PAllReduce
    ds, g = _data()
    cfg = hg.TrainConfig(fanouts=(6, 4, 3), hidden=16, batch_size=96, epochs=1, eta=0.05,
                         kind=hg.LayerKind.SAGE_MEAN, p_grad=0.9, t_stale=3, seed=5)
    net = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes).network
    ex = P2PAllReduce(net.flat.numel(), rank, WORLD, "cuda:0", timeout_s=0.5)
    if rank == 0:           # rank 1 never joins this exchange
        before = net.flat.clone()
        grads = net.new_grads(zero=True)
        ex.sgd(net, grads, 0.05)
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, "timeout.npy"),
                np.array([ex.timed_out, bool(torch.equal(before, net.flat))]))
        try:
            ex.check()
            raised = False
        except RuntimeError:
            raised = True
        np.save(os.path.join(out_dir, "raised.npy"), np.array([raised]))
        torch.zeros(1, device="cuda").add_(1)      # the context is still usable
        torch.cuda.synchronize()
    ex.close()
    dist.destroy_process_group()


def test_p2p_exchange_timeout_is_reported_not_trapped(tmp_path):
    mp.start_processes(_timeout_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True,
                       start_method="spawn")
    flags = np.load(tmp_path / "timeout.npy")
    assert flags[0], "the missing peer was not detected"
    assert flags[1], "parameters changed although the exchange failed"
    assert np.load(tmp_path / "raised.npy")[0]
