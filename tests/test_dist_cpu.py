"""Multi-process (world_size 2, gloo, CPU) coverage of the data-parallel path:
batch assignment per rank, owner ranges (comms.partition_features), and the
gradient all-reduce hook driving two oracle workers — checked bitwise against
the serial DP oracle (oracle/dp.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.datagen import csr2_from_edges, power_law_dataset
from oracle.dp import dp_serial_run
from oracle.step import SAGE, OTrainConfig, OTrainer, make_batches
from paper_2301_07482_b200.distributed import owner_of, owner_ranges, rank_batch_indices

WORLD, STEPS = 2, 4


def _cfg():
    return OTrainConfig(fanouts=(6, 4, 3), hidden=16, batch_size=96, epochs=1, eta=0.05, kind=SAGE,
                        p_grad=0.9, t_stale=3, seed=5)


def _data():
    ds = power_law_dataset(1500, np.random.default_rng(2), m=3, feature_dim=8)
    return ds, csr2_from_edges(ds.src, ds.dst, ds.num_nodes)


def test_rank_batch_indices_partition_steps():
    got = [rank_batch_indices(10, r, 3) for r in range(3)]
    assert got == [[0, 3, 6], [1, 4, 7], [2, 5, 8]]
    with pytest.raises(ValueError):
        rank_batch_indices(10, 3, 3)


def test_owner_ranges_match_reference_partition():
    # comms.partition_features: first n % P devices take one extra row
    b = owner_ranges(10, 4)
    np.testing.assert_array_equal(b, [0, 3, 6, 8, 10])
    np.testing.assert_array_equal(owner_of(np.arange(10), b), [0, 0, 0, 1, 1, 1, 2, 2, 3, 3])


def _worker(rank, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    ds, g = _data()
    cfg = _cfg()
    tr = OTrainer(g, ds.features, ds.labels, ds.train_ids, cfg, ds.num_classes)
    batches = make_batches(ds.train_ids, cfg)

    def hook(grads):      # the same flat-bucket average the GPU hook performs
        arrays = [a for l in grads for a in l.arrays()]
        flat = torch.from_numpy(np.concatenate([a.ravel() for a in arrays]).astype(np.float32))
        dist.all_reduce(flat)
        flat.div_(WORLD)
        off = 0
        for a in arrays:
            a[...] = flat[off:off + a.size].numpy().reshape(a.shape)
            off += a.size

    ms = []
    for idx in rank_batch_indices(len(batches), rank, WORLD)[:STEPS]:
        m = tr.train_iteration(idx, 0, tr.sample(idx, batches[idx]), grad_hook=hook)
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


def test_two_rank_gloo_dp_matches_serial_oracle(tmp_path):
    mp.start_processes(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True, start_method="spawn")
    ds, g = _data()
    metrics, net = dp_serial_run(g, ds.features, ds.labels, ds.train_ids, _cfg(), ds.num_classes, WORLD, STEPS)
    want_w = np.frombuffer(net.checksum_bytes(), np.uint8)
    for r in range(WORLD):
        got = np.load(tmp_path / f"r{r}_metrics.npy")
        want = np.array([[m.hits, m.misses, m.admissions, m.fetched_bytes, m.prune_writes, m.loss]
                         for m in metrics[r]])
        np.testing.assert_array_equal(got, want)
        np.testing.assert_array_equal(np.load(tmp_path / f"r{r}_w.npy"), want_w)
