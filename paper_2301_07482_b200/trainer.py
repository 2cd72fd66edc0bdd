"""Mini-batch training driver on the GPU (drop-in for histgnn/trainer.py).

Keeps the reference API: `TrainConfig` (trainer.py:59-83), `IterMetrics`
(:86-104), `write_metrics_csv`/`io_saving` (:110-123), `PrunedBatch`
(:138-150), `prune_with_cache` (:166-207), `make_batches` (:277-282),
`Trainer` (:285-433: `train_iteration`, `train`, `_load_input`) and
`run_plain_loop` (:439-469). Every per-iteration byte moves through the
hg_* kernels; the host keeps the integer policy decisions the reference makes
once per run or per window (batch permutation, PCG64 seeding, cache capacity).

Per iteration the host synchronises three times: after sampling (block
sizes, RNG draw count), after the prune walk (compute/live counts, which size
the GEMMs) and at the end (loss + counters for IterMetrics).
"""

from __future__ import annotations

import csv
import math
import os
from dataclasses import dataclass, fields

import numpy as np
import torch

from . import _lib
from ._state import GCTR_FEATURE_HITS, GCTR_FEATURE_MISSES, GCTR_PRUNE_WRITES, LAYER_CTR_LEN, CTR_VALID
from .distributed import apply_sgd
from .engine import StepEngine
from .cache import COUNTER_NAMES, CachePolicy, HistCache
from .graphs import Csr2Graph, _np, csr2_from_arrays
from .nn import (FeatureRows, Injection, LayerKind, Network, resolve_features_dev, backward, cross_entropy_dev, forward_pass, init_network, pad_columns,
                 pad_width,
                 layer_backward_dev, layer_forward_dev, load_features_dev, sgd_step, _dev_count)
from .sharding import ShardedFeatures
from .sampler import LayeredSubgraph, SamplePlan, SubgraphProducer, batch_rng, sample_layered, split_batches

_NET_TAG = 16807
_PERM_TAG = 1000000007


def _network_rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence((seed, _NET_TAG)))


def _perm_rng(seed: int, epoch: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence((seed, _PERM_TAG, epoch)))


@dataclass(frozen=True)
class TrainConfig:
    fanouts: tuple
    hidden: int = 64
    batch_size: int = 1024
    epochs: int = 1
    eta: float = 0.01
    kind: LayerKind = LayerKind.GCN
    p_grad: float = 0.9
    t_stale: float = 20
    capacity: int | None = None
    feature_rows: int | None = None
    refresh_retained: bool = False
    seed: int = 0
    probe_every: int = 0
    probe_layer: int = 1
    dtype: type = np.float32
    # B200 additions (not in the reference): where the raw feature table lives
    feature_placement: str = "hbm"      # "hbm" | "host" (pinned, read through UVA)
    max_capacity: int | None = None     # cache growth limit (see CachePolicy)
    heads: int = 4                      # GAT hidden-layer heads (LayerKind.GAT, oracle/gat.py)
    # data parallel: "local" = one cache per rank; "owner" = one cache sharded
    # by node owner over the torch.distributed group (shardcache.py)
    cache_sharding: str = "local"

    def __post_init__(self):
        if len(self.fanouts) == 0 or any(f < 1 for f in self.fanouts):
            raise ValueError("fanouts must be a non-empty tuple of positives")
        if self.batch_size < 1 or self.epochs < 1 or self.hidden < 1:
            raise ValueError("batch_size, epochs and hidden must be >= 1")
        if not math.isfinite(self.eta):
            raise ValueError("eta must be finite")
        if self.probe_every < 0:
            raise ValueError("probe_every must be >= 0")
        if self.feature_placement not in ("hbm", "host"):
            raise ValueError("feature_placement must be 'hbm' or 'host'")
        if self.cache_sharding not in ("local", "owner"):
            raise ValueError("cache_sharding must be 'local' or 'owner'")


@dataclass
class IterMetrics:
    iteration: int
    epoch: int
    num_seeds: int
    loss: float
    fetched_bytes: int
    baseline_bytes: int
    prune_writes: int
    hits: int
    misses: int
    admissions: int
    gradient_evictions: int
    staleness_evictions: int
    forced_evictions: int
    feature_hits: int
    feature_misses: int
    valid_entries: int
    estimation_error: float


METRIC_FIELDS = [f.name for f in fields(IterMetrics)]


def write_metrics_csv(path, metrics) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(METRIC_FIELDS)
        for m in metrics:
            w.writerow([getattr(m, name) for name in METRIC_FIELDS])


def io_saving(metrics) -> float:
    base = sum(m.baseline_bytes for m in metrics)
    if base == 0:
        return 0.0
    return 1.0 - sum(m.fetched_bytes for m in metrics) / base


def epoch_mean_estimation_error(metrics, epoch: int) -> float:
    """trainer.py:126-132: mean probe error of an epoch (nan-free), or nan."""
    vals = [m.estimation_error for m in metrics if m.epoch == epoch and not math.isnan(m.estimation_error)]
    return float(np.mean(vals)) if vals else math.nan


# ------------------------------------------------------------ drift probes
# (trainer.py:231-272; host-side bookkeeping of device-computed embeddings)


def cosine_rows(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Per-row cosine of two equally shaped matrices (trainer.py:234-241);
    nan where either row is all zeros."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    denom = np.sqrt((a * a).sum(axis=1) * (b * b).sum(axis=1))
    with np.errstate(invalid="ignore", divide="ignore"):
        cos = (a * b).sum(axis=1) / denom
    cos[denom == 0] = np.nan
    return cos


class EmbeddingLog:
    """Exact-embedding snapshots of a tracked node set keyed by iteration
    (trainer.py:244-272): `similarity(t, s)` is the mean cosine between the
    snapshots of iterations t and t - s over the nodes both contain,
    all-zero rows left out (nan when nothing is left)."""

    def __init__(self):
        self.records: dict = {}

    def record(self, iteration: int, ids, rows) -> None:
        self.records[iteration] = (np.array(ids, dtype=np.int64), np.array(rows))

    def similarity(self, t: int, s: int) -> float:
        older = t - s
        if s < 0 or older < 0:
            raise ValueError(f"need 0 <= s <= t, got t={t} s={s}")
        missing = [i for i in (t, older) if i not in self.records]
        if missing:
            raise ValueError(f"no snapshot for iterations {t} and {older}")
        (ids_t, rows_t), (ids_o, rows_o) = self.records[t], self.records[older]
        order_o = np.argsort(ids_o, kind="stable")
        pos = np.searchsorted(ids_o, ids_t, sorter=order_o)
        pos = np.minimum(pos, max(len(ids_o) - 1, 0))
        both = (len(ids_o) > 0) & (ids_o[order_o[pos]] == ids_t) if len(ids_o) else np.zeros(len(ids_t), bool)
        if not both.any():
            return math.nan
        # first occurrence per common id (ids within a snapshot are unique)
        keep_t = np.flatnonzero(both)
        _, first = np.unique(ids_t[keep_t], return_index=True)
        keep_t = keep_t[first]
        cos = cosine_rows(rows_t[keep_t], rows_o[order_o[pos[keep_t]]])
        cos = cos[np.isfinite(cos)]
        return float(cos.mean()) if cos.size else math.nan


# ------------------------------------------------------ cache-aware pruning


@dataclass
class PrunedBatch:
    """Device outcome of the cache walk. layer_live[l] / compute_rows[b] are
    int32 device tensors; injected[b] is an Injection (flags + cache rows) or
    None; keep/pos_of are the computed-row flags and positions per block."""

    sub: LayeredSubgraph
    compute_rows: list
    injected: list
    layer_live: list
    keep: list
    pos_of: list
    counts: list          # [(R_b, n_live_b)]
    counts_dev: torch.Tensor = None   # int32 [2L]: R_b, n_live_b on the device
    sizes_dev: torch.Tensor = None    # int32 [2L]: n_dst_b, n_src_b on the device

    def R_dev(self, b):
        return self.counts_dev[2 * b:2 * b + 1]

    def n_live_dev(self, b):
        return self.counts_dev[2 * b + 1:2 * b + 2]

    def n_dst_dev(self, b):
        return self.sizes_dev[2 * b:2 * b + 1]

    def injected_np(self, b: int):
        """Reference form (local rows sorted ascending, values) of injected[b]."""
        inj = self.injected[b]
        if inj is None:
            return None
        f = inj.flag.bool()
        loc = torch.nonzero(f).flatten()
        if inj.tables is not None:       # owner-sharded: read the rows through the injection kernel
            from .nn import inject_rows_dev
            n = int(inj.flag.shape[0])
            buf = torch.empty((n, inj.dim), dtype=torch.float32, device=inj.flag.device)
            inject_rows_dev(inj, buf, n, torch.tensor([n], dtype=torch.int32, device=buf.device), _lib.stream_ptr())
            vals = buf[loc]
        else:
            vals = inj.table[inj.row[loc].long()]
        return _np(loc).astype(np.int64), _np(vals)


def prune_with_cache(sub: LayeredSubgraph, cache: HistCache, current_iter: int, stream=None) -> PrunedBatch:
    """Walk blocks outermost-in (trainer.py:166-207); prunes sub in place."""
    dev = sub.layers[0].src_nodes.device
    s = stream or torch.cuda.current_stream(dev)
    sp = _lib.stream_ptr(s)
    L = sub.num_layers
    B = len(sub.seeds)
    sizes = []
    for b in range(L):
        blk = sub.layers[b]
        sizes += [blk.num_dst, blk.num_src]
    size_dev = torch.tensor(sizes, dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
    it_dev = torch.tensor([int(current_iter)], dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
    counts = torch.zeros(2 * L, dtype=torch.int32, device=dev)
    live_dst = None          # NULL = every seed row is live
    inj_flag = None
    compute, injected, live, keep_l, pos_l = [None] * L, [None] * L, [None] * (L + 1), [None] * L, [None] * L
    rows_buf, live_buf = [None] * L, [None] * L
    max_n = max(sizes)
    sb = _lib.query("hg_prune_scratch_bytes", max_n)
    scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
    for b in range(L - 1, -1, -1):
        blk = sub.layers[b]
        n_dst, n_src = blk.num_dst, blk.num_src
        keep = torch.empty(n_dst, dtype=torch.uint8, device=dev)
        rows = torch.empty(n_dst, dtype=torch.int32, device=dev)
        pos = torch.empty(n_dst, dtype=torch.int32, device=dev)
        src_mask = torch.empty(n_src, dtype=torch.uint8, device=dev)
        lv = torch.empty(n_src, dtype=torch.int32, device=dev)
        _lib.call("hg_prune_block", _lib.ptr(size_dev[2 * b:2 * b + 1]), n_dst, _lib.ptr(size_dev[2 * b + 1:2 * b + 2]),
                  n_src, _lib.ptr(live_dst), _lib.ptr(inj_flag), _lib.ptr(blk.adj.start), _lib.ptr(blk.adj.end),
                  _lib.ptr(blk.adj.col_indices), _lib.ptr(keep), _lib.ptr(rows), _lib.ptr(pos), _lib.ptr(src_mask),
                  _lib.ptr(lv), _lib.ptr(counts[2 * b:2 * b + 2]), _lib.ptr(cache.gctr), _lib.ptr(scratch), sb, sp)
        keep_l[b], pos_l[b], rows_buf[b], live_buf[b] = keep, pos, rows, lv
        live_dst, inj_flag = src_mask, None
        if b >= 1:
            lc = cache._layer(b)
            hit_flag = torch.empty(n_src, dtype=torch.uint8, device=dev)
            hit_row = torch.empty(n_src, dtype=torch.int32, device=dev)
            lc.lookup_dev(counts[2 * b + 1:2 * b + 2], n_src, lv, blk.src_nodes, n_src, it_dev, hit_flag,
                          hit_row, sp)
            inj = lc.injection(hit_flag, hit_row)
            if inj is not None:
                inj_flag = hit_flag
                injected[b - 1] = inj
    host = counts.cpu().tolist()
    cnt = []
    for b in range(L):
        R, nl = host[2 * b], host[2 * b + 1]
        cnt.append((R, nl))
        compute[b] = rows_buf[b][:R]
        live[b] = live_buf[b][:nl]
        sub.layers[b].adj.prune_writes += sub.layers[b].num_dst - R
    live[L] = torch.arange(B, dtype=torch.int32, device=dev)
    return PrunedBatch(sub, compute, injected, live, keep_l, pos_l, cnt, counts, size_dev)


# ----------------------------------------------------------------- trainer


class _EngineLast:
    """Exact-size views of the engine's last step, shaped like the API path's
    (pruned, tapes, grads, norms) tuple: pruned.layer_live / compute_rows and
    norms are sliced with the counts read back by train_step."""

    def __init__(self, out, counts):
        L = len(out["blocks"])
        self.out = out
        self.layer_live = [out["live"][b][:counts[2 * b + 1]] for b in range(L)]
        self.compute_rows = [out["rows"][b][:counts[2 * b]] for b in range(L)]
        self.norms = [None if out["norms"][l] is None else out["norms"][l][:counts[2 * l + 1]] for l in range(L)]

    def __getitem__(self, i):
        return (self, self.out["tapes"], self.out["grads"], self.norms)[i]


class PendingMetrics:
    """IterMetrics of a `Trainer.train_step(..., sync=False)` step whose
    counters are still in flight (device -> pinned host copy)."""

    def __init__(self, trainer, host_buf, event, iteration, epoch, num_seeds, nv):
        self._tr, self._buf, self._ev = trainer, host_buf, event
        self._args = (iteration, epoch, num_seeds, nv)
        self._m = None

    def _release(self):
        """Read the counters out of the (reused) pinned slot."""
        if self._m is None:
            self._ev.synchronize()
            it, ep, ns, nv = self._args
            self._m = self._tr._finish_pending(self._buf.tolist(), it, ep, ns, nv)
            self._buf = None

    def result(self) -> IterMetrics:
        self._release()
        return self._m

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self.result(), name)


def make_batches(train_ids, cfg: TrainConfig) -> list:
    out = []
    for epoch in range(cfg.epochs):
        out.extend(split_batches(train_ids, cfg.batch_size, _perm_rng(cfg.seed, epoch)))
    return out


def _device_graph(graph) -> Csr2Graph:
    if isinstance(graph, Csr2Graph) and isinstance(graph.start, torch.Tensor):
        return graph
    # reference (numpy) Csr2Graph or an (start, end, col) triple
    if isinstance(graph, tuple):
        return csr2_from_arrays(*graph)
    return csr2_from_arrays(graph.start, graph.end, graph.col_indices)


def _dtype_code(t: torch.Tensor) -> int:
    if isinstance(t, ShardedFeatures):
        return t.dtype_code
    if t.dtype == torch.float16:
        return 1
    if t.dtype == torch.float32:
        return 0
    raise ValueError(f"unsupported feature dtype {t.dtype} (fp32 / fp16)")


class Trainer:
    def __init__(self, graph, features, labels, train_ids, cfg: TrainConfig, num_classes=None, probe_nodes=None):
        _lib.require_cuda()
        self.graph = _device_graph(graph)
        self.device = self.graph.start.device
        self.cfg = cfg
        self.labels = np.asarray(labels, dtype=np.int64)
        self.train_ids = np.asarray(train_ids, dtype=np.int64)
        self.num_classes = int(num_classes or self.labels.max() + 1)
        if isinstance(features, ShardedFeatures):
            feats = features        # owner-range shards, peers mapped over NVLink (sharding.py)
        elif isinstance(features, torch.Tensor):
            feats = features
        else:
            feats = torch.from_numpy(np.ascontiguousarray(features))
        # the gather / aggregation kernels move rows as 16-byte vectors (at
        # most 1024 floats): a feature width that is not a multiple of 16
        # bytes is stored zero-padded (layer 0's weights get matching zero
        # rows, invisible through the reference-shaped views, nn._slab_views)
        self.in_dim = int(feats.shape[1])
        d_pad = pad_width(self.in_dim, feats.element_size())
        if d_pad > 1024:
            raise ValueError(f"feature width {self.in_dim} exceeds the kernels' 1024-float row limit")
        if cfg.hidden % 4 or cfg.hidden > 1024:
            raise ValueError(f"hidden must be a multiple of 4 and at most 1024 (got {cfg.hidden})")
        if d_pad != self.in_dim:
            if isinstance(feats, ShardedFeatures):
                raise ValueError("sharded feature tables need rows of a multiple of 16 bytes")
            feats = pad_columns(feats, d_pad)
        if isinstance(feats, ShardedFeatures):
            pass
        elif cfg.feature_placement == "hbm":
            feats = feats.to(self.device)
        elif feats.device.type != "cpu" or not feats.is_pinned():
            feats = feats.cpu().pin_memory()
        self.features = feats
        self.feature_dim = d_pad                                  # storage width of every layer-0 row
        self.row_bytes = self.in_dim * feats.element_size()       # the reference's I/O accounting unit
        depth = len(cfg.fanouts)
        dims = [self.in_dim] + [cfg.hidden] * (depth - 1) + [self.num_classes]
        self.network = init_network(cfg.kind, dims, _network_rng(cfg.seed), cfg.dtype, self.device, heads=cfg.heads,
                                    in_pad=self.feature_dim)
        policy = CachePolicy(cfg.p_grad, cfg.t_stale, cfg.capacity, cfg.max_capacity)
        feature_rows = self.graph.num_nodes // 10 if cfg.feature_rows is None else cfg.feature_rows
        if cfg.cache_sharding == "owner":
            import torch.distributed as dist
            from .sampler import layer_bounds
            from .shardcache import ShardedHistCache
            if not dist.is_initialized():
                raise ValueError("cache_sharding='owner' needs an initialised torch.distributed process group")
            F, _ = layer_bounds(cfg.batch_size, cfg.fanouts, self.graph.num_nodes)
            n_req = [F[depth - l] for l in range(1, depth)]     # sources of block l bound its live set
            self.cache = ShardedHistCache(self.graph.num_nodes, [cfg.hidden] * (depth - 1), policy, n_req,
                                          dist.get_rank(), dist.get_world_size(), feature_rows=feature_rows,
                                          refresh_retained=cfg.refresh_retained, dtype=cfg.dtype,
                                          device=self.device)
        else:
            self.cache = HistCache(self.graph.num_nodes, [cfg.hidden] * (depth - 1), policy,
                                   feature_rows=feature_rows, refresh_retained=cfg.refresh_retained, dtype=cfg.dtype,
                                   device=self.device)
        if feature_rows > 0:
            self.cache.backfill_features(self.features, graph=self.graph)
        self.plan = SamplePlan(cfg.fanouts, cfg.batch_size, cfg.seed)
        self.metrics = []
        self.last = None
        self._dtype_code = _dtype_code(self.features)
        # host placement: pinned (cudaHostAlloc) memory is UVA-mapped, so the
        # kernels dereference the host pointer directly over PCIe
        self.probe_nodes = None if probe_nodes is None else np.asarray(probe_nodes, dtype=np.int64)
        self.embedding_log = EmbeddingLog() if cfg.probe_every > 0 else None
        self._probe_record = None
        self.grad_hook = None   # callable(Grads) run between backward and SGD (data parallel)
        self.use_graphs = os.environ.get("HG_GRAPHS", "1") != "0"
        # layer 0 reads the feature rows in place (no fp32 copy of the input
        # frontier: SAGE / GCN aggregate them directly, GAT gathers them
        # straight into its transform operand) unless they sit in host memory
        # (UVA: one gather over PCIe beats one read per edge);
        # HG_FUSED_INPUT=0 restores the gather (A/B)
        self.fused_input = (cfg.feature_placement == "hbm" and os.environ.get("HG_FUSED_INPUT", "1") != "0")
        self._engines = {}
        self._ahead = None     # (key, device words) of the batch announced by the last step
        self._ctr_gen = 0      # bumped by every counter-moving step (engine metric rows re-sync on change)
        self._ctr_owner = None

    # ------------------------------------------------------------ pieces

    def sample(self, iteration: int, seeds) -> LayeredSubgraph:
        return sample_layered(self.graph, seeds, self.plan, batch_rng(self.cfg.seed, iteration))

    def _load_input(self, pruned: PrunedBatch, current_iter: int, stream=None, by_reference: bool = False):
        """trainer.py:326-343: feature-region hits + source fetches into the
        block-0 input matrix; returns (h, baseline_bytes). by_reference: the
        rows are not copied, h is a FeatureRows (their addresses) that the
        layer-0 aggregation reads in place."""
        b0 = pruned.sub.layers[0]
        dev = self.device
        sp = _lib.stream_ptr(stream)
        n_live0 = pruned.counts[0][1]
        region = self.cache.feature_table if self.cache.feature_table is not None else self.features
        if by_reference:
            rowp = torch.empty(b0.num_src, dtype=torch.int64, device=dev)
            resolve_features_dev(pruned.n_live_dev(0), n_live0, pruned.layer_live[0], b0.src_nodes,
                                 self.cache.feature_row_of_dev, region, self.features, self.feature_dim,
                                 self._dtype_code, rowp, self.cache.gctr, sp)
            return FeatureRows(rowp, self._dtype_code, self.feature_dim, b0.num_src), b0.num_src * self.row_bytes
        h = torch.empty((b0.num_src, self.feature_dim), dtype=torch.float32, device=dev)
        load_features_dev(pruned.n_live_dev(0), n_live0, pruned.layer_live[0], b0.src_nodes,
                          self.cache.feature_row_of_dev, region, self.features, self.feature_dim, self._dtype_code, h,
                          self.cache.gctr, sp)
        return h, b0.num_src * self.row_bytes

    # --------------------------------------------------------- main loop

    def train_iteration(self, iteration: int, epoch: int, sub: LayeredSubgraph, probe: bool = False) -> IterMetrics:
        """trainer.py:362-421. Returns IterMetrics (one device->host read)."""
        dev = self.device
        cache = self.cache
        before = cache.counters_vector().clone()
        labels_dev = torch.from_numpy(self.labels[sub.seeds].astype(np.int32)).pin_memory().to(dev, non_blocking=True)
        exact_sub = sub.copy() if probe else None      # before pruning mutates the CSR2 ends
        self._ctr_gen += 1
        self._probe_err = None
        loss_dev, baseline = self._step(iteration, sub, labels_dev, exact_sub=exact_sub)
        after = cache.counters_vector()
        host = torch.cat([loss_dev.view(1), (after - before).double(), after[CTR_VALID::LAYER_CTR_LEN]
                          [:cache.num_layers].double()]).cpu().tolist()
        loss, delta = host[0], [int(x) for x in host[1:1 + after.numel()]]
        valid = int(sum(host[1 + after.numel():]))
        m = self._metrics(iteration, epoch, len(sub.seeds), loss, delta, baseline, valid, sub)
        if probe:
            m.estimation_error = float(self._probe_err.item())
            if self.embedding_log is not None and self._probe_record is not None:
                self.embedding_log.record(iteration, *self._probe_record)
        return m

    def _estimation_probe(self, exact_sub: LayeredSubgraph, mixed_logits: torch.Tensor, stream) -> torch.Tensor:
        """trainer.py:345-358: relative error of the mixed (cache-pruned)
        logits against an exact recompute of the unpruned subgraph at the
        current weights (device scalar, fp64). Records the exact layer
        `probe_layer` embeddings of the tracked probe nodes."""
        dev = self.device
        b0 = exact_sub.layers[0]
        n0 = b0.num_src
        h = torch.empty((n0, self.feature_dim), dtype=torch.float32, device=dev)
        every = torch.arange(n0, dtype=torch.int32, device=dev)
        scratch_ctr = torch.zeros(8, dtype=torch.int64, device=dev)   # not the trainer's I/O counters
        load_features_dev(_dev_count(n0, dev), n0, every, b0.src_nodes, None, self.features, self.features,
                          self.feature_dim, self._dtype_code, h, scratch_ctr, _lib.stream_ptr(stream))
        exact = forward_pass(self.network, exact_sub.layers, h)
        diff = torch.linalg.vector_norm((mixed_logits - exact.logits).double())
        base = torch.linalg.vector_norm(exact.logits.double())
        self._probe_record = None
        li = self.cfg.probe_layer
        if self.probe_nodes is not None and 1 <= li <= exact_sub.num_layers:
            frontier = exact_sub.layers[li - 1].dst_nodes.long()
            present = torch.isin(frontier, torch.as_tensor(self.probe_nodes, device=dev))
            self._probe_record = (frontier[present].cpu().numpy(), exact.h_layers[li - 1][present].cpu().numpy())
        return diff / torch.clamp(base, min=1e-30)

    # ------------------------------------------- engine path (CUDA graph)

    def _engine(self, B: int) -> StepEngine:
        eng = self._engines.get(B)
        if eng is None:
            eng = self._engines[B] = StepEngine(self, B)
        return eng

    def _words(self, eng: StepEngine, iteration: int, seeds: np.ndarray) -> np.ndarray:
        bg = batch_rng(self.cfg.seed, iteration).bit_generator.state["state"]
        return eng.pack_inputs(iteration, seeds.astype(np.int32), self.labels[seeds].astype(np.int32),
                               (int(bg["state"]), int(bg["inc"])))

    def _ctr_key(self, eng):
        return (self._ctr_gen, self.cache._ops, id(eng))

    def _ctr_sync(self, eng) -> None:
        """The engine's metric row reports counter deltas since its previous
        row; re-base it when anything else moved the counters in between."""
        if eng.m_key != self._ctr_key(eng):
            eng.m_prev.copy_(self.cache.counters_vector())

    def _ctr_done(self, eng) -> None:
        self._ctr_gen += 1
        eng.m_key = self._ctr_key(eng)

    def _engine_step(self, iteration: int, seeds, next_batch=None):
        """Run one engine step; `next_batch=(iteration, seeds)` announces the
        following batch so the step samples it ahead (pipelined)."""
        seeds = np.asarray(seeds, dtype=np.int64)
        eng = self._engine(len(seeds))
        key = (len(seeds), int(iteration), hash(seeds.tobytes()))
        if self._ahead is not None and self._ahead[0] == key:
            words = self._ahead[1]          # uploaded (and sampled) by the previous step
        else:
            words = eng.upload(self._words(eng, iteration, seeds))
        self._ahead = None
        nxt = None
        if next_batch is not None:
            nit, nseeds = next_batch
            nseeds = np.asarray(nseeds, dtype=np.int64)
            if len(nseeds) == len(seeds):   # same engine (batch size): pipeline it
                nxt = eng.upload(self._words(eng, nit, nseeds))
                self._ahead = ((len(nseeds), int(nit), hash(nseeds.tobytes())), nxt)
        self._ctr_sync(eng)
        out = eng.step_words(words, nxt)
        self._ctr_done(eng)
        return eng, out

    def train_step_device(self, iteration: int, seeds, next_batch=None) -> torch.Tensor:
        """Device-resident step for throughput runs: sample + train one batch
        (graph replay after warm-up); returns the loss as a device scalar and
        does not synchronise. Sweeps run on the host every t_stale steps."""
        eng, out = self._engine_step(iteration, seeds, next_batch)
        self.cache.end_iteration(iteration)
        self._last_engine = (eng, out)
        return out["loss"]

    def prestage(self, iterations, seeds_list) -> list:
        """Pack (seeds, labels, PCG64 state, iteration) of several batches
        into HBM, for runs whose inputs are resident before timing starts."""
        out = []
        for it, seeds in zip(iterations, seeds_list):
            seeds = np.asarray(seeds, dtype=np.int64)
            eng = self._engine(len(seeds))
            out.append((it, len(seeds), torch.from_numpy(self._words(eng, it, seeds)).to(self.device)))
        return out

    def train_step_resident(self, staged, next_staged=None) -> torch.Tensor:
        """One step from prestage()d HBM inputs (no host traffic, no sync);
        `next_staged` is sampled ahead when given."""
        it, B, words = staged
        eng = self._engine(B)
        nxt = next_staged[2] if next_staged is not None and next_staged[1] == B else None
        self._ctr_sync(eng)
        out = eng.step_words(words, nxt)
        self._ctr_done(eng)
        self.cache.end_iteration(it)
        self._last_engine = (eng, out)
        return out["loss"]

    def train_step(self, iteration: int, epoch: int, seeds, next_batch=None, sync: bool = True):
        """Sample + train one batch through the engine and read IterMetrics
        back (trainer.py:362-421 semantics, sampling included).
        `next_batch=(iteration, seeds)` lets the step sample that batch ahead.
        sync=False: the metrics are copied device -> pinned host memory
        asynchronously and a PendingMetrics is returned (IterMetrics on
        `.result()` or on first attribute access), so the host can enqueue
        the next step while this one runs."""
        cache = self.cache
        eng, out = self._engine_step(iteration, seeds, next_batch)
        dev_buf = eng.m_row            # written by the step itself (hg_metrics_row)
        nv = eng.m_nv
        if not sync:
            ring = self._metrics_ring(eng, dev_buf.numel())
            pm = PendingMetrics(self, None, None, iteration, epoch, len(seeds), nv)
            i, host_buf = ring.acquire(pm)
            host_buf.copy_(dev_buf, non_blocking=True)
            pm._buf, pm._ev = host_buf, ring.issued(i)
            cache.end_iteration(iteration)
            self._last_engine = (eng, out)
            return pm
        host = dev_buf.cpu().tolist()
        loss, delta = host[0], [int(x) for x in host[1:1 + nv]]
        valid = int(sum(host[1 + nv:1 + nv + cache.num_layers]))
        n_src0 = int(host[1 + nv + cache.num_layers])
        counts = [int(x) for x in host[2 + nv + cache.num_layers:]]
        cache.end_iteration(iteration)
        self._last_engine = (eng, out)
        self.last = _EngineLast(out, counts)
        return self._metrics(iteration, epoch, len(seeds), loss, delta, n_src0 * self.row_bytes, valid, None,
                             prune_writes=delta[cache.num_layers * LAYER_CTR_LEN + GCTR_PRUNE_WRITES])

    def _metrics_ring(self, eng, numel: int):
        ring = getattr(eng, "metrics_ring", None)
        if ring is None or ring.bufs[0].numel() != numel:
            from .engine import PinnedRing
            ring = eng.metrics_ring = PinnedRing(8, numel, torch.float64)
        return ring

    def _finish_pending(self, host, iteration, epoch, num_seeds, nv):
        cache = self.cache
        loss, delta = host[0], [int(x) for x in host[1:1 + nv]]
        valid = int(sum(host[1 + nv:1 + nv + cache.num_layers]))
        n_src0 = int(host[1 + nv + cache.num_layers])
        return self._metrics(iteration, epoch, num_seeds, loss, delta, n_src0 * self.row_bytes, valid, None,
                             prune_writes=delta[cache.num_layers * LAYER_CTR_LEN + GCTR_PRUNE_WRITES])

    def _step(self, iteration: int, sub: LayeredSubgraph, labels_dev: torch.Tensor, exact_sub=None):
        dev = self.device
        stream = torch.cuda.current_stream(dev)
        sp = _lib.stream_ptr(stream)
        net, cache, cfg = self.network, self.cache, self.cfg
        it_dev = torch.tensor([int(iteration)], dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
        cache.begin_step(it_dev, sp)
        pruned = prune_with_cache(sub, cache, iteration, stream)
        h0, baseline = self._load_input(pruned, iteration, stream, by_reference=self.fused_input)
        L = sub.num_layers
        tapes = []
        h = h0
        for b in range(L):
            R, _ = pruned.counts[b]
            t = layer_forward_dev(net, b, sub.layers[b], h, pruned.compute_rows[b], R, pruned.R_dev(b),
                                  b < L - 1, pruned.injected[b], sp, pruned.n_dst_dev(b), live=pruned.layer_live[b],
                                  n_live=pruned.counts[b][1], n_live_dev=pruned.n_live_dev(b))
            tapes.append(t)
            h = t.h_out
        B = int(sub.seeds.shape[0])
        d_h, loss_dev = cross_entropy_dev(tapes[-1].h_out, labels_dev, B, net.dims[-1], sp)
        if exact_sub is not None:       # probe between the forward and the SGD step (trainer.py:376-381)
            self._probe_err = self._estimation_probe(exact_sub, tapes[-1].h_out, stream)
        grads = net.new_grads(zero=False)
        norms = [None] * L
        for l in range(L - 1, -1, -1):
            n_live = pruned.counts[l][1]
            d_prev, nrm = layer_backward_dev(net, l, sub.layers[l], tapes[l], d_h, grads, l >= 1, pruned.keep[l],
                                             pruned.pos_of[l], pruned.layer_live[l], n_live, sp,
                                             pruned.n_dst_dev(l), pruned.n_live_dev(l),
                                             need_rows=pruned.keep[l - 1] if l >= 1 else None)
            norms[l] = nrm
            d_h = d_prev
        apply_sgd(self.grad_hook, net, grads, cfg.eta)   # e.g. NCCL all-reduce of the flat bucket, then SGD
        for layer in range(1, L):
            n_live = pruned.counts[layer][1]
            if n_live == 0:
                continue
            cache._layer(layer).update_dev(pruned.n_live_dev(layer), n_live, pruned.layer_live[layer],
                                           sub.layers[layer].src_nodes, norms[layer], pruned.keep[layer - 1],
                                           tapes[layer - 1].h_out, it_dev, cache.refresh_retained, sp)
        cache.commit(sp)                 # owner-sharded cache: apply every rank's requests (no-op otherwise)
        cache.end_iteration(iteration)
        self.last = (pruned, tapes, grads, norms)
        return loss_dev, baseline

    def _metrics(self, iteration, epoch, num_seeds, loss, delta, baseline, valid, sub, prune_writes=None):
        nl = self.cache.num_layers
        tot = dict.fromkeys(COUNTER_NAMES, 0)
        from .cache import _LAYER_IDX
        for l in range(nl):
            for k, i in _LAYER_IDX.items():
                tot[k] += delta[l * LAYER_CTR_LEN + i]
        g = delta[nl * LAYER_CTR_LEN:]
        fh, fm = g[GCTR_FEATURE_HITS], g[GCTR_FEATURE_MISSES]
        return IterMetrics(
            iteration=iteration, epoch=epoch, num_seeds=num_seeds, loss=float(loss),
            fetched_bytes=fm * self.row_bytes, baseline_bytes=baseline,
            prune_writes=(sum(b.adj.prune_writes for b in sub.layers) if prune_writes is None else prune_writes),
            hits=tot["hits"], misses=tot["misses"], admissions=tot["admissions"],
            gradient_evictions=tot["gradient_evictions"], staleness_evictions=tot["staleness_evictions"],
            forced_evictions=tot["forced_evictions"], feature_hits=fh, feature_misses=fm,
            valid_entries=valid, estimation_error=math.nan)

    def train(self) -> list:
        """trainer.py:423-433: every batch of every epoch, in order. The
        producer thread's run-ahead (sampler.py:193-263) becomes the engine's
        pipelined sampler: each step samples the next batch on a side stream
        while it trains the current one."""
        cfg = self.cfg
        batches = make_batches(self.train_ids, cfg)
        per_epoch = max(1, math.ceil(len(self.train_ids) / cfg.batch_size))
        pe = cfg.probe_every

        def probing(it):
            return pe > 0 and it % pe == 0

        for iteration, seeds in enumerate(batches):
            if probing(iteration):
                # probe iterations run the eager API path (the exact recompute
                # sits between the forward and the SGD step)
                m = self.train_iteration(iteration, iteration // per_epoch, self.sample(iteration, seeds), probe=True)
                self.metrics.append(m)
                continue
            nxt = None
            if iteration + 1 < len(batches) and not probing(iteration + 1):
                nxt = (iteration + 1, batches[iteration + 1])
            self.metrics.append(self.train_step(iteration, iteration // per_epoch, seeds, next_batch=nxt))
        return self.metrics


# ------------------------------------------------------ reference baseline


def run_plain_loop(graph, features, labels, train_ids, cfg: TrainConfig, num_classes=None, on_step=None):
    """Cache-free loop sharing the trainer's rng streams and update order
    (trainer.py:439-469). Returns (network, per-iteration losses)."""
    _lib.require_cuda()
    g = _device_graph(graph)
    dev = g.start.device
    labels = np.asarray(labels, dtype=np.int64)
    train_ids = np.asarray(train_ids, dtype=np.int64)
    ncls = int(num_classes or labels.max() + 1)
    feats = features if isinstance(features, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(features))
    d_in = int(feats.shape[1])
    d = pad_width(d_in, feats.element_size())
    feats = pad_columns(feats.to(dev), d)
    depth = len(cfg.fanouts)
    dims = [d_in] + [cfg.hidden] * (depth - 1) + [ncls]
    network = init_network(cfg.kind, dims, _network_rng(cfg.seed), cfg.dtype, dev, heads=cfg.heads, in_pad=d)
    plan = SamplePlan(cfg.fanouts, cfg.batch_size, cfg.seed)
    losses = []
    gctr = torch.zeros(8, dtype=torch.int64, device=dev)
    sp = _lib.stream_ptr()
    for idx, seeds in enumerate(make_batches(train_ids, cfg)):
        sub = sample_layered(g, seeds, plan, batch_rng(cfg.seed, idx))
        b0 = sub.layers[0]
        h = torch.empty((b0.num_src, d), dtype=torch.float32, device=dev)
        live = torch.arange(b0.num_src, dtype=torch.int32, device=dev)
        load_features_dev(_dev_count(b0.num_src, dev), b0.num_src, live, b0.src_nodes, None, feats, feats, d,
                          _dtype_code(feats), h, gctr, sp)
        tape = forward_pass(network, sub.layers, h)
        labels_dev = torch.as_tensor(labels[seeds].astype(np.int32), device=dev)
        d_logits, loss = cross_entropy_dev(tape.logits.contiguous(), labels_dev, len(seeds), ncls, sp)
        grads, _, _ = backward(network, sub.layers, tape, d_logits, need_input=False)
        sgd_step(network, grads, cfg.eta)
        losses.append(float(loss.item()))
        if on_step is not None:
            on_step(idx, network)
    return network, losses


# -------------------------------------------------------------- inference


def evaluate(network: Network, graph, features, labels, ids, chunk_rows: int | None = None) -> float:
    """Exact full-graph accuracy on `ids` (trainer.py:485-506): argmax of
    full_graph_logits over the given node ids."""
    g = _device_graph(graph)
    N = int(g.num_nodes)
    ids = np.asarray(ids, dtype=np.int64)
    labels = np.asarray(labels, dtype=np.int64)
    if len(ids) and (ids.min() < 0 or ids.max() >= N):
        raise ValueError("evaluation ids out of range")
    h = full_graph_logits(network, g, features, chunk_rows)
    if len(ids) == 0:
        return float("nan")
    pred = h[torch.as_tensor(ids, device=h.device)].argmax(dim=1).cpu().numpy()
    return float((pred == labels[ids]).mean())


def full_graph_logits(network: Network, graph, features, chunk_rows: int | None = None) -> torch.Tensor:
    """Layer-wise inference over whole-graph blocks (trainer.py:473-482: every
    node is a dst row, block 0's sources carry no in-edges, deeper blocks use
    the in-degree), ReLU on every layer but the last; returns the device
    logits [N x C]. Each layer runs the training kernels (hg_aggregate_fwd ->
    TS operand -> tcgen05 GEMM with the scatter epilogue) over dst-row chunks
    of `chunk_rows` rows, so the GEMM operand stays bounded (default ~2 GB)
    while h stays resident in HBM."""
    _lib.require_cuda()
    g = _device_graph(graph)
    dev = g.start.device
    N = int(g.num_nodes)
    if int(g.end.max().item() if N else 0) >= 2 ** 31:
        raise ValueError("evaluate needs fewer than 2^31 edges (int32 block offsets)")
    feats = features if isinstance(features, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(features))
    feats = pad_columns(feats.to(dev), network.dims[0])
    if feats.shape[0] != N:
        raise ValueError("features must have one row per node")
    sp = _lib.stream_ptr()
    d0 = int(feats.shape[1])
    every = torch.arange(N, dtype=torch.int32, device=dev)
    # layer-0 input as fp32 rows (the training feature gather, all nodes live)
    h = torch.empty((N, d0), dtype=torch.float32, device=dev)
    gctr = torch.zeros(8, dtype=torch.int64, device=dev)
    load_features_dev(_dev_count(N, dev), N, every, every, None, feats, feats, d0, _dtype_code(feats), h, gctr, sp)
    start = g.start.to(torch.int32)
    end = g.end.to(torch.int32)
    deg = (end - start).contiguous()
    zero = torch.zeros_like(deg)
    from .nn import _kind_code, gat_layer_forward_dev, ts_bytes
    kind = _kind_code(network.kind)
    L = network.num_layers
    if network.kind is LayerKind.GAT:
        # whole-graph blocks: every node a dst row, sources = all nodes
        class _Full:
            num_src = num_dst = N
            adj = type("A", (), {"start": start, "end": end, "col_indices": g.col_indices})()
        cnt = _dev_count(N, dev)
        for l in range(L):
            t = gat_layer_forward_dev(network, l, _Full, h, every, N, cnt, l < L - 1, None, sp, cnt, every, N, cnt)
            h = t.h_out
        return h
    for l in range(L):
        d_in, d_out = network.dims[l], network.dims[l + 1]
        K = 2 * d_in if network.kind == LayerKind.SAGE_MEAN else d_in
        PT = torch.empty(ts_bytes(d_out, K + 1), dtype=torch.uint8, device=dev)
        _lib.call("hg_ts_pack", _lib.ptr(network.slab(l)), d_out, 1, d_out, K + 1, d_out, _lib.ptr(PT), sp)
        per_row = max(1, ts_bytes(1024, K + 1) // 1024)
        chunk = int(chunk_rows) if chunk_rows else max(128, min(N, (2 << 30) // per_row))
        A = torch.empty(ts_bytes(min(chunk, max(N, 1)), K + 1), dtype=torch.uint8, device=dev)
        h_out = torch.empty((N, d_out), dtype=torch.float32, device=dev)
        for r0 in range(0, N, chunk):
            R = min(chunk, N - r0)
            R_dev = _dev_count(R, dev)
            rows = every[r0:r0 + R]
            _lib.call("hg_aggregate_fwd", kind, _lib.ptr(R_dev), R, _lib.ptr(rows), _lib.ptr(start), _lib.ptr(end),
                      _lib.ptr(g.col_indices), _lib.ptr(deg), _lib.ptr(zero if l == 0 else deg), _lib.ptr(h), d_in,
                      _lib.ptr(A), None, sp)
            _lib.call("hg_ts_linear_fwd", _lib.ptr(R_dev), R, _lib.ptr(A), K + 1, _lib.ptr(PT), d_out, _lib.ptr(rows),
                      int(l < L - 1), _lib.ptr(h_out), sp)
        h = h_out
    return h
