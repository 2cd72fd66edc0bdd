#!/usr/bin/env python
"""Benchmark: ReFresh per-iteration training throughput (seeds/s) on B200.

Workload (N=1 default, BASELINE.json configs[1]): ogbn-products-shaped
synthetic power-law graph (2.4M nodes, 62.4M edges, 100-d fp32 features,
47 classes), 3-layer GraphSAGE hidden 256, fanouts (15,10,5), batch 1024,
historical cache (p_grad 0.9, t_stale 20). A step = sample one batch + one
train_iteration (prune, feature gather, forward, loss, backward, SGD, cache
update). Inputs (graph 0.5 GB + features 0.96 GB) are far larger than L2,
batches touch random rows, so no L2 flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c2|c1]

--impl reference times the CPU oracle port (oracle/, the reference algorithm
restated in numpy) on the host cores, on the same dataset.
Multi-GPU (torchrun): data parallel, each rank trains its own batches with its
own cache replica; gradients are all-reduced (NCCL) before SGD; weak scaling.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training seeds/sec per iteration"
CONFIGS = {
    "c2": dict(workload="ogbn-products-shape synthetic power-law (2.4M nodes, 62.4M edges, 100-d fp32), "
                        "3-layer GraphSAGE hidden 256, fanout 15,10,5, batch 1024, cache p_grad 0.9 t_stale 20",
               n=2_400_000, m=13, d=100, classes=47),
    "c3": dict(workload="ogbn-papers100M-shape synthetic power-law (111M nodes, 1.55B edges, 128-d fp16), "
                        "3-layer GraphSAGE hidden 256, fanout 15,10,5, batch 1024, cache p_grad 0.9 t_stale 20",
               n=111_000_000, m=7, d=128, classes=172, fp16=True, capacity=6_000_000, max_capacity=24_000_000),
    "c5": dict(workload="ogbn-papers100M-shape synthetic power-law (111M nodes, 1.55B edges, 128-d fp16), "
                        "3-layer GAT (4 heads, hidden 256), fanout 15,10,5, batch 1024, cache p_grad 0.9 t_stale 20",
               n=111_000_000, m=7, d=128, classes=172, fp16=True, capacity=6_000_000, max_capacity=24_000_000,
               kind="gat"),
    "c4s": dict(workload="MAG240M-shape slice for one GPU: synthetic power-law (40M nodes, 280M edges, 768-d fp16, "
                         "61 GB), 3-layer GraphSAGE hidden 256, fanout 15,10,5, batch 1024, cache p_grad 0.9 t_stale 20",
                n=40_000_000, m=4, d=768, classes=153, fp16=True, capacity=6_000_000, max_capacity=12_000_000,
                feature_rows_frac=0.01),
    "c1": dict(workload="synthetic power-law 100K nodes / 2M edges, 128-d fp32, 3-layer GraphSAGE hidden 256, "
                        "fanout 15,10,5, batch 1024, cache p_grad 0.9 t_stale 20",
               n=100_000, m=10, d=128, classes=8),
}
FANOUTS, HIDDEN, BATCH, P_GRAD, T_STALE, ETA = (15, 10, 5), 256, 1024, 0.9, 20, 0.01


def make_data(cfg, seed=0):
    """Native power-law graph (C++) + numpy N(0,1) features; identical for both arms.
    At the papers100M shape the features (28 GB fp16) are drawn on the device
    instead (feats = None here, see device_features)."""
    from paper_2301_07482_b200.data import synth_edges
    src, dst = synth_edges(cfg["n"], cfg["m"], seed)
    rng = np.random.default_rng(seed)
    feats = None if cfg.get("fp16") else rng.standard_normal((cfg["n"], cfg["d"]), dtype=np.float32)
    labels = rng.integers(0, cfg["classes"], size=cfg["n"])
    perm = rng.permutation(cfg["n"])
    train = np.sort(perm[: int(0.6 * cfg["n"])])
    return src, dst, feats, labels, train


def device_features(cfg, dev, seed=0, lo=0, hi=None, chunk=1 << 22):
    """Rows [lo, hi) of the N(0,1) feature table, drawn on the device in row
    chunks (chunk c from its own seeded generator, so every rank's shard is
    the same slice of one table whatever the rank count), stored fp16."""
    import torch
    hi = cfg["n"] if hi is None else hi
    out = torch.empty((hi - lo, cfg["d"]), dtype=torch.float16, device=dev)
    gen = torch.Generator(device=dev)
    for c in range(lo // chunk, -(-hi // chunk)):
        a, b = c * chunk, min(cfg["n"], (c + 1) * chunk)
        gen.manual_seed(seed * 1_000_003 + c)
        x = torch.randn((b - a, cfg["d"]), generator=gen, device=dev)
        out[max(a, lo) - lo:min(b, hi) - lo] = x[max(a, lo) - a:min(b, hi) - a]
    return out


def aggregate_bytes(out, tr):
    """Algorithmic bytes of one step's k_aggregate launches (SAGE / GCN):
    per block b, U = live input rows, R = compute rows, E = their surviving
    edges: U.d.4 (input rows) + R.K1.4 (TS operand, bf16 hi + lo) + 4E (col)
    + 8R (offsets)."""
    import torch
    if tr.network.kind.value == "gat":
        return None
    counts = out["counts"].cpu().tolist()
    total = 0
    for b, blk in enumerate(out["blocks"]):
        R, U = counts[2 * b], counts[2 * b + 1]
        rows = out["rows"][b][:R].long()
        E = int((blk.end.long()[rows] - blk.blk_off.long()[rows]).sum().item()) if R else 0
        d = tr.network.dims[b]
        K1 = (2 * d if tr.network.kind.value == "sage_mean" else d) + 1
        K1 = (K1 + 31) // 32 * 32
        total += U * d * 4 + R * K1 * 4 + 4 * E + 8 * R
    return total


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.idx = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def _rows(self):
        self.f.flush()
        with open(self.f.name) as fh:
            return [r.split(",") for r in fh.read().strip().splitlines() if r.strip()]

    def wait_running(self, timeout=10.0):
        """Block until nvidia-smi has produced a sample; rows up to here are
        pre-timing and are dropped from the summary."""
        self.skip = 0
        if self.p is None:
            return
        t0 = time.time()
        while time.time() - t0 < timeout:
            n = len(self._rows())
            if n:
                self.skip = n
                return
            time.sleep(0.02)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        rows = self._rows()[getattr(self, "skip", 0):]
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 8 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) > 8 for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def cpu_reference(cfg, data, steps, warmup, budget_s=150.0):
    """Oracle port (numpy restatement of the reference) on the host cores."""
    from oracle.datagen import csr2_from_edges
    from oracle.step import SAGE, OTrainConfig, OTrainer, make_batches
    src, dst, feats, labels, train = data
    g = csr2_from_edges(src.astype(np.int64), dst.astype(np.int64), cfg["n"])
    ocfg = OTrainConfig(fanouts=FANOUTS, hidden=HIDDEN, batch_size=BATCH, eta=ETA, kind=SAGE, p_grad=P_GRAD,
                        t_stale=T_STALE, seed=0)
    tr = OTrainer(g, feats, labels, train, ocfg, cfg["classes"])
    batches = make_batches(train, ocfg)
    it = 0
    t_start = time.perf_counter()
    for _ in range(warmup):
        tr.train_iteration(it, 0, tr.sample(it, batches[it]))
        it += 1
        if time.perf_counter() - t_start > budget_s / 3:
            break
    done, seeds, t0 = 0, 0, time.perf_counter()
    while done < steps:
        m = tr.train_iteration(it, 0, tr.sample(it, batches[it]))
        seeds += m.num_seeds
        it += 1
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0))
    return {"value": seeds / dt, "ms_per_step": 1e3 * dt / done, "steps": done, "cores": cores,
            "sample": f"{done} full iterations (batch {BATCH}) of OTrainer on the same graph after "
                      f"{it - done} warm-up iterations; numpy/OpenBLAS threads = {cores}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--allreduce", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 gradient exchange: fused peer-memory kernel (default) or NCCL all_reduce")
    ap.add_argument("--replicate-features", action="store_true",
                    help="N>1: full feature table on every GPU instead of owner-range shards over NVLink")
    args = ap.parse_args()
    cfgd = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    config = {"workload": cfgd["workload"], "nodes": cfgd["n"], "edges": 2 * cfgd["m"] * (cfgd["n"] - cfgd["m"]),
              "feature_dim": cfgd["d"], "global_batch": BATCH * world, "fanouts": list(FANOUTS),
              "hidden": HIDDEN, "parallelism": f"dp{world}", "l2": "inputs > L2 (1.5 GB resident, random rows)"}
    base = {"metric": METRIC, "unit": "seeds/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic (native power-law generator, N(0,1) features)", "config": config}

    if args.impl == "reference":
        if rank != 0:
            return
        data = make_data(cfgd)
        r = cpu_reference(cfgd, data, args.steps, args.warmup, budget_s=150.0)
        out = dict(base, impl="reference", value=r["value"], ms_per_step=r["ms_per_step"],
                   cpu_baseline={"value": r["value"], "unit": "seeds/s", "cores": r["cores"], "kind": "port",
                                 "sample": r["sample"]},
                   e2e={"value": r["value"], "unit": "seeds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        out["steps"] = r["steps"]
        print(json.dumps(out))
        return

    import torch
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200 import _lib

    # HG_BENCH_ONE_GPU=1: every rank on cuda:0 over gloo (exercises the
    # multi-rank path, IPC shards included, on a 1-GPU box; not a scaling run)
    one_gpu = os.environ.get("HG_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    data = make_data(cfgd)
    src, dst, feats, labels, train = data
    from paper_2301_07482_b200.data import csr2_from_edges_device
    graph = csr2_from_edges_device(src, dst, cfgd["n"], dev)
    sharded = world > 1 and not args.replicate_features
    shard_note = None
    if sharded:
        # this rank's owner range only (comms.py:329-337); peers mapped over NVLink
        from paper_2301_07482_b200.distributed import owner_ranges
        bnd = owner_ranges(cfgd["n"], world)
        lo, hi = int(bnd[rank]), int(bnd[rank + 1])
        local_rows = device_features(cfgd, dev, lo=lo, hi=hi) if feats is None else feats[lo:hi]
        feats_dev, err = None, ""
        try:
            feats_dev = hg.ShardedFeatures.from_process_group(local_rows, cfgd["n"], rank, world, dev)
        except Exception as e:   # e.g. no peer access between these GPUs
            err = f"{type(e).__name__}: {e}"
        ok = torch.tensor([0 if feats_dev is None else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            # every rank falls back together to full local tables (never mixes layouts)
            if feats_dev is not None:
                torch.cuda.synchronize()
                dist.barrier()
                feats_dev.close()
            sharded, shard_note = False, f"IPC sharding unavailable ({err or 'on a peer rank'}); replicated"
            feats_dev = device_features(cfgd, dev) if feats is None else torch.from_numpy(feats).to(dev)
        del local_rows
    else:
        feats_dev = device_features(cfgd, dev) if feats is None else torch.from_numpy(feats).to(dev)
    config["features"] = (f"sharded {world}-way by owner range, remote rows read over NVLink (CUDA IPC)"
                          if sharded else (shard_note or "replicated in HBM"))
    del src, dst
    n_tl = 10   # extra steps after the timed regions for the phase timeline
    need = (args.warmup + 2 * args.steps + n_tl + 1) * world
    per_epoch = -(-len(train) // BATCH)
    kind = hg.LayerKind.GAT if cfgd.get("kind") == "gat" else hg.LayerKind.SAGE_MEAN
    tcfg = hg.TrainConfig(fanouts=FANOUTS, hidden=HIDDEN, batch_size=BATCH, eta=ETA, kind=kind, heads=4,
                          p_grad=P_GRAD, t_stale=T_STALE, seed=0, epochs=max(1, -(-need // per_epoch)),
                          capacity=cfgd.get("capacity"), max_capacity=cfgd.get("max_capacity"),
                          feature_rows=(int(cfgd["n"] * cfgd["feature_rows_frac"]) if "feature_rows_frac" in cfgd
                                        else None))
    tr = hg.Trainer(graph, feats_dev, labels, train, tcfg, cfgd["classes"])
    if world > 1:
        from paper_2301_07482_b200.distributed import P2PAllReduce, make_allreduce_hook
        hook, err = None, ""
        if args.allreduce == "p2p":
            # gradient exchange fused with SGD over CUDA-IPC slots (NVLink loads)
            try:
                hook = P2PAllReduce(tr.network.flat.numel(), rank, world, dev)
            except Exception as e:
                err = f"{type(e).__name__}: {e}"
            ok = torch.tensor([0 if hook is None else 1], dtype=torch.int32, device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0:
                if hook is not None:
                    hook.close()
                hook = None
                config["allreduce_note"] = f"P2P exchange unavailable ({err or 'on a peer rank'}); NCCL"
        if hook is None:
            hook = make_allreduce_hook(world)   # NCCL: captured in the step's CUDA graph
        tr.grad_hook = hook
        config["allreduce"] = ("fused P2P all-reduce + SGD (hg_p2p_allreduce_sgd)"
                               if getattr(hook, "fused_sgd", False) else f"{dist.get_backend()} all_reduce + hg_sgd")
    batches = hg.make_batches(train, tcfg)
    mem_setup = torch.cuda.memory_allocated(dev)
    if need > len(batches):
        raise SystemExit(f"need {need} batches, epoch has {len(batches)}")
    # rank r takes batch indices world*s + r (iteration number = global batch index)
    mine = [world * s + rank for s in range(args.warmup + 2 * args.steps + n_tl + 1)]
    # inputs of the device-resident steps packed into HBM before timing
    # (+1: the last timed step also samples a next batch, like every other one)
    n_res = args.warmup + args.steps + 1
    staged = tr.prestage(mine[:n_res], [batches[i] for i in mine[:n_res]])

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    no_ahead = os.environ.get("HG_NO_LOOKAHEAD") == "1"   # diagnostic: sample each batch in its own step

    def nxt(i):   # the batch announced for pipelined sampling (staged in HBM)
        return staged[i + 1] if i + 1 < len(staged) and not no_ahead else None

    for s in range(args.warmup):
        tr.train_step_resident(staged[s], nxt(s))
    torch.cuda.synchronize()
    # setup objects (graph, tables, captured graphs) move to the permanent GC
    # generation, so a cyclic-GC pass inside the timed steps scans only the
    # per-step garbage (a full pass over the setup heap stalled the host for
    # tens of ms in some e2e runs)
    gc.collect()
    gc.freeze()

    # ---- timed region 1: device-resident steps (value) ----
    clocks = ClockSampler(local)
    # device-side kernel timers (%globaltimer spans; the step is a CUDA graph,
    # where host events cannot bracket a single kernel node)
    timers = torch.zeros(8 * 8, dtype=torch.int64, device=dev)
    timers.view(8, 8)[:, 0] = -1
    g_before = tr.cache.gctr.clone()
    clocks.start()
    clocks.wait_running()
    barrier()
    torch.cuda.synchronize()
    _lib.call("hg_set_kernel_timers", _lib.ptr(timers))
    launches0 = _lib.load().hg_kernel_launches()
    caps0 = sum(e.captures for e in tr._engines.values())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    losses = []
    for s in range(args.warmup, args.warmup + args.steps):
        losses.append(tr.train_step_resident(staged[s], nxt(s)))
    e1.record()
    torch.cuda.synchronize()
    _lib.call("hg_set_kernel_timers", None)
    launches = _lib.load().hg_kernel_launches() - launches0
    barrier()
    clk = clocks.stop()
    t_dev = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    # seeds actually trained (an epoch's last batch can be short); the same
    # on every rank pattern-wise, so scale rank 0's by the world size
    seeds_value = world * sum(len(batches[mine[s]]) for s in range(args.warmup, args.warmup + args.steps))
    value = seeds_value / t_dev
    graph_mode = any(e.graph is not None for e in tr._engines.values())
    caps_value = sum(e.captures for e in tr._engines.values()) - caps0

    # roofline of the feature gather (k_load_rows): algorithmic bytes =
    # live layer-0 rows x (row read + fp32 row write + 3 index reads); the live
    # rows of the timed steps = delta(feature_hits + feature_misses)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md: MEASURED_PEAKS.json absent)"
    if os.path.exists(peaks_path):
        peak, peak_src = json.load(open(peaks_path))["hbm_gbs"], "measured"
    tv = timers.view(8, 8).cpu().tolist()
    names = ["k_load_rows", "k_aggregate", "k_transpose_agg", "k_select", "k_tsgemm (forward)", "k_tsgemm (dgrad)",
             "k_tsgemm (wgrad, split-K)"]
    per_kernel = {n: {"launches": int(tv[i][3]), "ms_total": tv[i][2] / 1e6,
                      "share_of_step": (tv[i][2] / 1e9) / t_dev} for i, n in enumerate(names)}
    g_delta = (tr.cache.gctr - g_before).cpu().tolist()
    remote_rows = g_delta[3]
    rows = g_delta[0] + g_delta[1]
    isz = tr.features.element_size()
    g_bytes = rows * (cfgd["d"] * isz + cfgd["d"] * 4 + 12)
    g_time = tv[0][2] / 1e9
    n_launch = max(1, int(tv[0][3]))
    achieved = g_bytes / g_time / 1e9 if g_time > 0 else 0.0
    # DRAM traffic of one warm k_load_rows launch from the committed ncu
    # --set full capture of this config (profiles/r01/traffic.json)
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "r01", "traffic.json")
    tkey = "c3" if args.config in ("c3", "c5") else args.config
    if os.path.exists(tpath):
        tj = json.load(open(tpath)).get(tkey)
        if tj:
            traffic, traffic_src = tj["traffic_bytes"], tj["capture"]
    roofline = {"kernel": "k_load_rows (hg_load_features, feature gather)", "bound": "hbm",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": peak_src, "traffic": traffic, "traffic_source": traffic_src,
                "bytes_per_launch": g_bytes / n_launch, "avg_launch_us": 1e6 * g_time / n_launch,
                "timing": "device %globaltimer span per launch, accumulated over the timed region",
                "share_of_step": g_time / t_dev if t_dev else None}

    # ---- timed region 2: end-to-end through the public API (host in, host out) ----
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h2d = d2h = 0
    for s in range(args.warmup + args.steps, args.warmup + 2 * args.steps):
        it = mine[s]
        nb = (mine[s + 1], batches[mine[s + 1]])
        m = tr.train_step(it, 0, batches[it], next_batch=nb, sync=False)
        # this step uploads the announced next batch's words (PCG64 state,
        # iteration, seed ids, labels), or its own when none was announced
        h2d += (12 + 2 * BATCH) * 4
        d2h += (1 + tr.cache.counters_vector().numel() + tr.cache.num_layers) * 8
    torch.cuda.synchronize()
    t_e2e = max_over_ranks(time.perf_counter() - t0)
    m = m.result()
    caps_e2e = sum(e.captures for e in tr._engines.values()) - caps0 - caps_value
    seeds_e2e = world * sum(len(batches[mine[s]]) for s in range(args.warmup + args.steps, args.warmup + 2 * args.steps))
    e2e = {"value": seeds_e2e / t_e2e, "unit": "seeds/s",
           "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
           "api": "Trainer.train_step (host seeds in via pinned staging, IterMetrics counters copied to pinned "
                  "host memory every step, sync=False: the host enqueues step s+1 while step s runs)"}

    # ---- phase timeline of the replayed step (after timing; %globaltimer marks) ----
    eng = tr._engine(BATCH)
    eng.enable_timeline(True)
    tl_steps = tr.prestage(mine[-(n_tl + 1):], [batches[i] for i in mine[-(n_tl + 1):]])
    acc = {}
    agg_bytes = []
    for i in range(n_tl):   # every step samples the next one (the last staged batch is lookahead only)
        tr.train_step_resident(tl_steps[i], None if no_ahead else tl_steps[i + 1])
        agg_bytes.append(aggregate_bytes(eng.out, tr))
        for k, v in eng.timeline_ms().items():
            acc[k] = acc.get(k, 0.0) + v / n_tl
    eng.enable_timeline(False)
    timeline = {k: round(v, 4) for k, v in acc.items()}

    row_b = cfgd["d"] * tr.features.element_size()
    nvlink = {"remote_rows_per_step": remote_rows / args.steps, "bytes_per_step": remote_rows * row_b / args.steps,
              "share_of_gathered_rows": remote_rows / max(1, g_delta[0] + g_delta[1])}
    # SAGE neighbour aggregation (k_aggregate, all layers): algorithmic bytes
    # per step from the counts of the post-timing steps (SURVEY 8(d):
    # U.d.4 + R.(K+1).4 + 4E + 8R per layer) over its timed per-step duration
    agg_roof = None
    if per_kernel["k_aggregate"]["launches"] and agg_bytes and agg_bytes[0] is not None:
        t_step = per_kernel["k_aggregate"]["ms_total"] / 1e3 / args.steps
        b_step = float(np.mean(agg_bytes))
        agg_roof = {"kernel": "k_aggregate (hg_aggregate_fwd, all layers)", "bound": "hbm",
                    "achieved": b_step / t_step / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": b_step / t_step / 1e9 / peak, "bytes_per_step": b_step,
                    "bytes_source": f"counts of the {n_tl} post-timing steps"}
    out = dict(base, value=value, nvlink_gather=nvlink, aggregate_roofline=agg_roof, ms_per_step=1e3 * t_dev / args.steps, e2e=e2e, roofline=roofline,
               gpu_launches=int(launches), clocks=clk, per_kernel=per_kernel, cuda_graph=graph_mode,
               graph_captures_in_timed={"value": caps_value, "e2e": caps_e2e},
               timeline_ms=timeline,
               loss_last=float(losses[-1].item()), io_saving_last=None)
    out["io_saving_e2e_last"] = 1.0 - m.fetched_bytes / m.baseline_bytes if m.baseline_bytes else None
    out["hbm_gb"] = {"allocated_after_setup": round(mem_setup / 1e9, 2),
                     "peak": round(torch.cuda.max_memory_allocated(dev) / 1e9, 2)}
    if cfgd.get("capacity"):
        config["cache_capacity_rows_per_layer"] = [cfgd["capacity"], cfgd["max_capacity"]]
    feat_bytes = cfgd["n"] * cfgd["d"] * tr.features.element_size()
    if feat_bytes < 2 * 126e6:
        # small graphs (C1) stay L2-resident across steps; no flush is done,
        # so this is a parity-size configuration, not a bench line
        config["l2"] = (f"inputs fit in L2 ({feat_bytes / 1e6:.0f} MB features), not flushed: "
                        "parity-size config, not a bench line")
    elif not cfgd.get("fp16"):
        config["l2"] = f"inputs > L2 ({feat_bytes / 1e9:.1f} GB features resident, random rows)"
    if cfgd.get("fp16"):
        out["dtype"] = "fp32 (fp16 feature table, converted in the gather)"
        config["l2"] = f"inputs > L2 ({cfgd['n'] * cfgd['d'] * 2 / 1e9:.0f} GB features resident, random rows)"
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cfgd.get("fp16"):
        out["cpu_baseline"] = {"value": None, "unit": "seeds/s", "cores": len(os.sched_getaffinity(0)),
                               "kind": "port", "sample": "not run at this shape (the numpy port needs the full "
                               f"{cfgd['n'] * cfgd['d'] * 2 / 1e9:.0f} GB feature table and the graph in host "
                               "RAM, minutes per iteration); see the C2 line for the CPU comparison"}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference(cfgd, data, steps=3, warmup=1, budget_s=args.cpu_budget)
        out["cpu_baseline"] = {"value": r["value"], "unit": "seeds/s", "cores": r["cores"], "kind": "port",
                               "sample": r["sample"]}
    if rank == 0:
        print(json.dumps(out))
    if sharded:
        torch.cuda.synchronize()
        barrier()
        del tr
        feats_dev.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
