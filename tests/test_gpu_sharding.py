"""Sharded feature table: owner-range shards read one-sided.

* virtual shards (all P shards on one GPU, the same kernel path as peer
  shards): training runs are bitwise identical to the unsharded table, for
  fp32 and fp16 tables, and rows owned by other shards are counted;
* CUDA IPC shards (two processes sharing one B200; each holds only its own
  range and maps the other's): every row read through the shards equals the
  full table, and a 2-rank data-parallel run over IPC shards ends with the
  same weights and metrics as the same run over full replicated tables."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _data(dim=16):
    from oracle.datagen import csr2_from_edges, power_law_dataset
    ds = power_law_dataset(2500, np.random.default_rng(4), m=4, feature_dim=dim)
    return ds, csr2_from_edges(ds.src, ds.dst, ds.num_nodes)


def _cfg(hg, **kw):
    base = dict(fanouts=(8, 5, 3), hidden=32, batch_size=128, eta=0.05, kind=hg.LayerKind.SAGE_MEAN,
                p_grad=0.9, t_stale=4, seed=2)
    base.update(kw)
    return hg.TrainConfig(**base)


def _run(hg, g, feats, ds, steps=6, **kw):
    tr = hg.Trainer(g, feats, ds.labels, ds.train_ids, _cfg(hg, **kw), ds.num_classes)
    batches = hg.make_batches(ds.train_ids, tr.cfg)
    ms = [tr.train_iteration(i, 0, tr.sample(i, batches[i])) for i in range(steps)]
    return tr, ms


@pytest.mark.parametrize("dtype", [np.float32, np.float16])
@pytest.mark.parametrize("P", [1, 3, 8])
def test_virtual_shards_are_bit_transparent(P, dtype):
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200._state import GCTR_REMOTE_ROWS
    ds, g = _data()
    f = ds.features.astype(dtype)
    tr0, m0 = _run(hg, g, f, ds)
    sf = hg.ShardedFeatures.virtual(f, P)
    tr1, m1 = _run(hg, g, sf, ds)
    for a, b in zip(m0, m1):
        assert a == b
    assert tr0.network.checksum_bytes() == tr1.network.checksum_bytes()
    remote = int(tr1.cache.gctr[GCTR_REMOTE_ROWS].item())
    assert (remote == 0) if P == 1 else (remote > 0)


def test_virtual_shards_index_select_and_region():
    import paper_2301_07482_b200 as hg
    ds, g = _data(dim=24)
    for dtype in (torch.float32, torch.float16):
        full = torch.from_numpy(ds.features).to(dtype).cuda()
        sf = hg.ShardedFeatures.virtual(full, 5)
        ids = torch.randperm(ds.num_nodes, device="cuda")[:777]
        assert torch.equal(sf.index_select(0, ids), full[ids])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.distributed import make_allreduce_hook, owner_ranges, rank_batch_indices
    ds, g = _data()
    b = owner_ranges(ds.num_nodes, world)
    ok = []
    for dtype in (np.float32, np.float16):
        f = ds.features.astype(dtype)
        sf = hg.ShardedFeatures.from_process_group(f[b[rank]:b[rank + 1]], ds.num_nodes, rank, world, "cuda:0")
        ids = torch.arange(ds.num_nodes, device="cuda")
        ok.append(bool(torch.equal(sf.index_select(0, ids).cpu(), torch.from_numpy(f))))
        dist.barrier()
        sf.close()
    # 2-rank DP run over IPC shards vs the same run over replicated tables
    res = []
    for mode in ("ipc", "replicated"):
        feats = (hg.ShardedFeatures.from_process_group(ds.features[b[rank]:b[rank + 1]], ds.num_nodes, rank, world,
                                                       "cuda:0") if mode == "ipc" else ds.features)
        tr = hg.Trainer(g, feats, ds.labels, ds.train_ids, _cfg(hg), ds.num_classes)
        tr.grad_hook = make_allreduce_hook(world)
        batches = hg.make_batches(ds.train_ids, tr.cfg)
        ms = []
        for idx in rank_batch_indices(len(batches), rank, world)[:4]:
            m = tr.train_iteration(idx, 0, tr.sample(idx, batches[idx]))
            ms.append([m.hits, m.misses, m.admissions, m.fetched_bytes, m.prune_writes, m.feature_hits,
                       m.feature_misses, m.loss])
        res.append((np.array(ms), np.frombuffer(tr.network.checksum_bytes(), np.uint8)))
        torch.cuda.synchronize()
        dist.barrier()
        if mode == "ipc":
            del tr
            feats.close()
    np.save(os.path.join(out_dir, f"r{rank}_ok.npy"), np.array(ok))
    np.save(os.path.join(out_dir, f"r{rank}_m.npy"), np.stack([res[0][0], res[1][0]]))
    np.save(os.path.join(out_dir, f"r{rank}_w.npy"), np.stack([res[0][1], res[1][1]]))
    dist.destroy_process_group()


def test_ipc_shards_two_processes(tmp_path):
    world = 2
    mp.start_processes(_ipc_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        assert np.load(tmp_path / f"r{r}_ok.npy").all(), "rows read through IPC shards differ from the table"
        m = np.load(tmp_path / f"r{r}_m.npy")
        np.testing.assert_array_equal(m[0], m[1])
        w = np.load(tmp_path / f"r{r}_w.npy")
        np.testing.assert_array_equal(w[0], w[1])
    np.testing.assert_array_equal(np.load(tmp_path / "r0_w.npy"), np.load(tmp_path / "r1_w.npy"))


@pytest.mark.parametrize("kind", ["gcn", "gat"])
def test_virtual_shards_engine_other_layer_kinds(kind):
    """Sharded features under the CUDA-graph engine (pipelined sampling) for
    GCN and GAT: bitwise the same run as with the plain table."""
    import paper_2301_07482_b200 as hg
    ds, g = _data()
    k = hg.LayerKind.GCN if kind == "gcn" else hg.LayerKind.GAT
    runs = []
    for feats in (ds.features, hg.ShardedFeatures.virtual(ds.features, 4)):
        tr = hg.Trainer(g, feats, ds.labels, ds.train_ids, _cfg(hg, kind=k, heads=2), ds.num_classes)
        b = hg.make_batches(ds.train_ids, tr.cfg)[:10]
        ms = [tr.train_step(i, 0, s, next_batch=(i + 1, b[i + 1]) if i + 1 < len(b) else None) for i, s in enumerate(b)]
        runs.append(([(m.loss, m.hits, m.admissions, m.feature_hits) for m in ms], tr.network.checksum_bytes()))
    assert runs[0] == runs[1]


@pytest.mark.parametrize("P", [3, 8])
def test_owner_row_counters_give_the_reference_transfer_accounting(P):
    """Per-owner rows read by the sharded gather == requests_for_batch of the
    iteration's fetched ids (comms.py:326-349, restated in oracle/comms.py),
    and the one-/two-sided byte accounting (comms.py:283-323) follows."""
    import paper_2301_07482_b200 as hg
    from oracle.comms import fetch_bytes, merge_transfers, partition_features, requests_for_batch
    from paper_2301_07482_b200.distributed import transfer_accounting
    ds, g = _data()
    sf = hg.ShardedFeatures.virtual(ds.features, P)
    tr = hg.Trainer(g, sf, ds.labels, ds.train_ids, _cfg(hg), ds.num_classes)
    batches = hg.make_batches(ds.train_ids, tr.cfg)
    owner = partition_features(ds.num_nodes, P)
    region = tr.cache.feature_row_of >= 0
    for i in range(5):
        before = sf.owner_rows.clone()
        sub = tr.sample(i, batches[i])
        m = tr.train_iteration(i, 0, sub)
        pruned = tr.last[0]
        ids = sub.layers[0].src_nodes[pruned.layer_live[0]].cpu().numpy().astype(np.int64)
        fetched = ids[~region[ids]]
        assert len(fetched) == m.feature_misses
        counts = (sf.owner_rows - before).cpu().numpy()
        np.testing.assert_array_equal(counts, np.bincount(owner[fetched], minlength=P))
        acc = transfer_accounting(counts, sf.local_shard, tr.row_bytes)
        want = merge_transfers(requests_for_batch(owner, fetched, sf.local_shard))
        assert [(t["src"], t["dst"], t["num_ids"]) for t in acc["transfers"]] == want
        assert acc["two_sided"] == fetch_bytes(want, True, tr.row_bytes)
        assert acc["one_sided"]["payload_bytes"] + acc["local_rows"] * tr.row_bytes == m.fetched_bytes


def test_ingest_device_matches_in_memory_training(tmp_path):
    """A dataset written in the reference's directory format and ingested
    into the device layout (native parsers, CSR2 on the GPU, features
    streamed to HBM / pinned host / fp16) trains exactly like the same
    dataset built in memory."""
    import torch
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200.compat.data import Dataset, save_dataset
    from paper_2301_07482_b200.compat.graphs import CooGraph
    from paper_2301_07482_b200.ingest import ingest_device
    ds, g = _data()
    save_dataset(tmp_path, Dataset(CooGraph(ds.src, ds.dst, ds.num_nodes), ds.features, ds.labels, ds.train_ids,
                                   ds.val_ids, ds.test_ids))
    tr0, m0 = _run(hg, g, ds.features, ds)
    for placement, dtype in (("hbm", torch.float32), ("host", torch.float32), ("hbm", torch.float16)):
        dd = ingest_device(tmp_path, placement=placement, dtype=dtype)
        assert torch.equal(dd.graph.col_indices.cpu(), torch.as_tensor(g[2]).to(torch.int32))
        np.testing.assert_array_equal(dd.graph.end.cpu().numpy(), g[1])
        want = torch.from_numpy(ds.features).to(dtype)
        assert torch.equal(dd.features.cpu(), want)
        if dtype == torch.float32:
            tr = hg.Trainer(dd.graph, dd.features, dd.labels, dd.train_ids, _cfg(hg, feature_placement=placement),
                            dd.num_classes)
            batches = hg.make_batches(dd.train_ids, tr.cfg)
            m1 = [tr.train_iteration(i, 0, tr.sample(i, batches[i])) for i in range(6)]
            assert [a == b for a, b in zip(m0, m1)] == [True] * 6
            assert tr.network.checksum_bytes() == tr0.network.checksum_bytes()
