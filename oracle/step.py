"""One training iteration on CPU (oracle restatement of histgnn/trainer.py + nn.py).

- prune_with_cache   trainer.py:153-207 (+ Csr2Graph.prune_many graphs.py:123-127)
- load_input         trainer.py:213-228,326-343 (feature region + source fetch)
- forward_pass       nn.py:91-163,260-297  (SAGE_MEAN / GCN block convolutions,
                                            scatter to full rows, injected rows)
- backward           nn.py:166-177,300-320 (hand reverse pass; injected = leaves)
- cross_entropy      nn.py:326-343 (fp64 log-sum-exp), node_grad_norms nn.py:346-349
- sgd_step           nn.py:355-360; init_network nn.py:73-85 (+ rng tags trainer.py:47-56)
- OTrainer.train_iteration trainer.py:362-421; train trainer.py:423-433
- run_plain_loop     trainer.py:439-469

Float work is fp32 storage with fp32 sparse accumulation and fp64 coefficient
construction, as in the reference; comparisons against it are tolerance-based.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, fields

import numpy as np
import scipy.sparse as sp

from . import gat as ogat
from .histcache import OCachePolicy, OHistCache
from .sampling import OBlock, OSubgraph, _segment_positions, batch_rng, sample_layered, split_batches

GCN, SAGE, GAT = "gcn", "sage_mean", "gat"
NET_TAG, PERM_TAG = 16807, 1000000007


# ------------------------------------------------------------------ params


@dataclass
class OLayer:
    weight: np.ndarray
    bias: np.ndarray
    weight_neigh: np.ndarray | None = None

    def arrays(self):
        out = [self.weight, self.bias]
        if self.weight_neigh is not None:
            out.append(self.weight_neigh)
        return out


@dataclass
class ONetwork:
    kind: str
    layers: list

    @property
    def num_layers(self):
        return len(self.layers)

    @property
    def dtype(self):
        return self.layers[0].weight.dtype

    def checksum_bytes(self):
        return b"".join(np.ascontiguousarray(a).tobytes() for l in self.layers for a in l.arrays())


def init_network(kind, dims, rng, dtype=np.float32, heads=4):
    """nn.py:73-85 — Glorot-uniform, self weight drawn before neighbour weight.
    GAT (no reference, oracle/gat.py): `heads` on hidden layers, 1 on the last."""
    out = []
    if kind == GAT:
        L = len(dims) - 1
        for l, (fi, fo) in enumerate(zip(dims[:-1], dims[1:])):
            out.append(ogat.init_layer(rng, fi, fo, heads if l < L - 1 else 1, dtype))
        return ONetwork(kind, out)
    for fi, fo in zip(dims[:-1], dims[1:]):
        lim = np.sqrt(6.0 / (fi + fo))
        w = rng.uniform(-lim, lim, size=(fi, fo)).astype(dtype)
        wn = rng.uniform(-lim, lim, size=(fi, fo)).astype(dtype) if kind == SAGE else None
        out.append(OLayer(w, np.zeros(fo, dtype), wn))
    return ONetwork(kind, out)


def network_rng(seed):
    return np.random.default_rng(np.random.SeedSequence((seed, NET_TAG)))


def perm_rng(seed, epoch):
    return np.random.default_rng(np.random.SeedSequence((seed, PERM_TAG, epoch)))


# ----------------------------------------------------------------- pruning


@dataclass
class OPruned:
    sub: OSubgraph
    compute_rows: list
    injected: list
    layer_live: list


def _row_sources(blk, rows):
    lo = blk.start[rows]
    n = blk.end[rows] - lo
    return blk.col[np.repeat(lo, n) + _segment_positions(n)]


def prune_with_cache(sub: OSubgraph, cache: OHistCache, it: int) -> OPruned:
    L = sub.num_layers
    compute, inj, live = [None] * L, [None] * L, [None] * (L + 1)
    live[L] = np.arange(len(sub.seeds), dtype=np.int64)
    served_loc, served_val = np.empty(0, np.int64), None
    for b in range(L - 1, -1, -1):
        blk = sub.layers[b]
        keep = np.zeros(blk.num_dst, bool)
        keep[live[b + 1]] = True
        if len(served_loc):
            keep[served_loc] = False
            inj[b] = (served_loc, served_val)
        rows = np.flatnonzero(keep)
        compute[b] = rows
        cut = np.flatnonzero(~keep)
        blk.end[cut] = blk.start[cut]             # O(1) row cut per pruned row
        blk.prune_writes += len(cut)
        need = np.zeros(blk.num_src, bool)
        need[rows] = True                         # dst is a prefix of src
        need[_row_sources(blk, rows)] = True
        live[b] = np.flatnonzero(need)
        if b >= 1:
            g = blk.src_nodes[live[b]]
            hit_ids, hit_vals, _ = cache.lookup(b, g, it)
            if len(hit_ids):
                served_loc = live[b][np.isin(g, hit_ids)]
                served_val = hit_vals
            else:
                served_loc, served_val = np.empty(0, np.int64), None
    return OPruned(sub, compute, inj, live)


# ----------------------------------------------------------------- loading


class OFeatureSource:
    def __init__(self, features):
        self.features = features
        self.fetched_bytes = 0
        self.fetched_rows = 0

    @property
    def row_bytes(self):
        return self.features.shape[1] * self.features.dtype.itemsize

    def fetch(self, ids):
        self.fetched_rows += len(ids)
        self.fetched_bytes += len(ids) * self.row_bytes
        return self.features[ids]


def load_input(pruned: OPruned, cache: OHistCache, source: OFeatureSource, it, dtype=np.float32):
    b0 = pruned.sub.layers[0]
    h = np.zeros((b0.num_src, source.features.shape[1]), dtype)
    live0 = pruned.layer_live[0]
    g = b0.src_nodes[live0]
    hit_ids, hit_vals, _ = cache.lookup(0, g, it)
    if len(hit_ids):
        hm = np.isin(g, hit_ids)
        h[live0[hm]] = hit_vals.astype(dtype)
        rest = live0[~hm]
    else:
        rest = live0
    if len(rest):
        h[rest] = source.fetch(b0.src_nodes[rest]).astype(dtype)
    return h, b0.num_src * source.row_bytes


# ------------------------------------------------------------------ layers


@dataclass
class OTape:
    rows: np.ndarray
    relu: np.ndarray | None
    amat: object = None   # sparse aggregation operator (GCN Â or SAGE M)
    agg: np.ndarray | None = None
    h_self: np.ndarray | None = None


def _agg_operator(kind, blk, rows, dtype):
    """nn.py:101-128 — CSR over the selected rows' surviving edges."""
    lo = blk.start[rows]
    cnt = blk.end[rows] - lo
    cols = blk.col[np.repeat(lo, cnt) + _segment_positions(cnt)]
    if kind == SAGE:
        inv = np.zeros(len(rows))
        nz = cnt > 0
        inv[nz] = 1.0 / cnt[nz]
        ptr = np.concatenate([[0], np.cumsum(cnt)])
        return sp.csr_matrix((np.repeat(inv, cnt).astype(dtype), cols, ptr),
                             shape=(len(rows), blk.num_src))
    # GCN: per row, edge entries then the self entry
    dd = blk.dst_deg[rows].astype(np.float64)
    w_e = 1.0 / np.sqrt((np.repeat(dd, cnt) + 1.0) * (blk.src_deg[cols] + 1.0))
    w_s = 1.0 / np.sqrt((dd + 1.0) * (blk.src_deg[rows] + 1.0))
    cnt1 = cnt + 1
    ptr = np.concatenate([[0], np.cumsum(cnt1)])
    last = ptr[1:] - 1
    idx = np.empty(int(cnt1.sum()), np.int64)
    val = np.empty(int(cnt1.sum()), np.float64)
    body = np.ones(len(idx), bool)
    body[last] = False
    idx[body], val[body] = cols, w_e
    idx[last], val[last] = rows, w_s
    return sp.csr_matrix((val.astype(dtype), idx, ptr), shape=(len(rows), blk.num_src))


def layer_forward_ctx(kind, p: OLayer, blk, h_in, rows, act):
    if h_in.shape[0] != blk.num_src:
        raise ValueError(f"h_in has {h_in.shape[0]} rows, frontier needs {blk.num_src}")
    if kind == GAT:
        return ogat.layer_forward(p, blk, h_in, rows, act)
    A = _agg_operator(kind, blk, rows, h_in.dtype)
    agg = A @ h_in
    if kind == GCN:
        z = agg @ p.weight + p.bias
        t = OTape(rows, None, A, agg, None)
    else:
        hs = h_in[rows]
        z = hs @ p.weight + agg @ p.weight_neigh + p.bias
        t = OTape(rows, None, A, agg, hs)
    if act:
        t.relu = z > 0
        z = np.where(t.relu, z, z.dtype.type(0))
    return z, t


def layer_backward(kind, p: OLayer, t: OTape, d_out, need_input=True):
    if kind == GAT:
        return ogat.layer_backward(p, t, d_out, need_input)
    dz = d_out if t.relu is None else np.where(t.relu, d_out, 0)
    db = dz.sum(axis=0)
    if kind == GCN:
        g = OLayer(t.agg.T @ dz, db, None)
        d_in = (t.amat.T @ (dz @ p.weight.T)) if need_input else None
        return g, d_in
    g = OLayer(t.h_self.T @ dz, db, t.agg.T @ dz)
    d_in = None
    if need_input:
        d_in = t.amat.T @ (dz @ p.weight_neigh.T)
        d_in[t.rows] += dz @ p.weight.T
    return g, d_in


@dataclass
class OBatchTape:
    h_input: np.ndarray
    entries: list
    h_layers: list

    @property
    def logits(self):
        return self.h_layers[-1]


def forward_pass(net: ONetwork, blocks, h_input, compute_rows=None, injected=None):
    if len(blocks) != net.num_layers:
        raise ValueError("block count does not match network depth")
    ents, hs = [], []
    h = h_input
    for l, blk in enumerate(blocks):
        rows = (np.arange(blk.num_dst, dtype=np.int64) if compute_rows is None or compute_rows[l] is None
                else np.asarray(compute_rows[l], np.int64))
        z, t = layer_forward_ctx(net.kind, net.layers[l], blk, h, rows, l < net.num_layers - 1)
        full = np.zeros((blk.num_dst, net.layers[l].weight.shape[1]), z.dtype)
        full[rows] = z
        if injected is not None and injected[l] is not None and len(injected[l][0]):
            full[np.asarray(injected[l][0], np.int64)] = injected[l][1]
        ents.append(t)
        hs.append(full)
        h = full
    return OBatchTape(h_input, ents, hs)


def backward(net: ONetwork, blocks, tape: OBatchTape, d_logits, need_input=True):
    L = net.num_layers
    grads, node_grads = [None] * L, [None] * L
    d = d_logits
    for l in range(L - 1, -1, -1):
        node_grads[l] = d
        t = tape.entries[l]
        grads[l], d = layer_backward(net.kind, net.layers[l], t, d[t.rows],
                                     need_input or l > 0)
    return grads, node_grads, d


def cross_entropy(logits, labels):
    labels = np.asarray(labels)
    if logits.shape[0] != len(labels):
        raise ValueError("labels do not match logit rows")
    if len(labels) and (labels.min() < 0 or labels.max() >= logits.shape[1]):
        raise ValueError("label id out of range")
    z = logits.astype(np.float64)
    z = z - z.max(axis=1, keepdims=True)
    lp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    n = len(labels)
    loss = float(-lp[np.arange(n), labels].sum() / n)
    g = np.exp(lp)
    g[np.arange(n), labels] -= 1.0
    return loss, (g / n).astype(logits.dtype)


def node_grad_norms(g):
    g = g.astype(np.float64, copy=False)
    return np.sqrt(np.einsum("ij,ij->i", g, g))


def sgd_step(net: ONetwork, grads, eta):
    e = net.dtype.type(eta)
    for p, g in zip(net.layers, grads):
        p.weight -= e * g.weight
        p.bias -= e * g.bias
        if getattr(p, "weight_neigh", None) is not None:
            p.weight_neigh -= e * g.weight_neigh
        if net.kind == GAT:
            p.att_src -= e * g.att_src
            p.att_dst -= e * g.att_dst


# ----------------------------------------------------------------- trainer


@dataclass(frozen=True)
class OTrainConfig:
    fanouts: tuple
    hidden: int = 64
    batch_size: int = 1024
    epochs: int = 1
    eta: float = 0.01
    kind: str = GCN
    p_grad: float = 0.9
    t_stale: float = 20
    capacity: int | None = None
    feature_rows: int | None = None
    refresh_retained: bool = False
    seed: int = 0
    dtype: type = np.float32
    heads: int = 4          # GAT hidden-layer heads (oracle/gat.py)


@dataclass
class OIterMetrics:
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
    estimation_error: float = math.nan


INT_METRICS = [f.name for f in fields(OIterMetrics)
               if f.name not in ("loss", "estimation_error")]


def make_batches(train_ids, cfg):
    out = []
    for e in range(cfg.epochs):
        out.extend(split_batches(train_ids, cfg.batch_size, perm_rng(cfg.seed, e)))
    return out


class OTrainer:
    """trainer.py:285-433 over a CSR2 full graph given as (start, end, col)."""

    def __init__(self, graph, features, labels, train_ids, cfg: OTrainConfig, num_classes=None):
        self.start, self.end, self.col = graph
        self.num_nodes = len(self.start)
        self.features = features
        self.labels = np.asarray(labels, np.int64)
        self.train_ids = np.asarray(train_ids, np.int64)
        self.cfg = cfg
        self.num_classes = int(num_classes or self.labels.max() + 1)
        depth = len(cfg.fanouts)
        dims = [features.shape[1]] + [cfg.hidden] * (depth - 1) + [self.num_classes]
        self.network = init_network(cfg.kind, dims, network_rng(cfg.seed), cfg.dtype, cfg.heads)
        frows = self.num_nodes // 10 if cfg.feature_rows is None else cfg.feature_rows
        self.cache = OHistCache(self.num_nodes, [cfg.hidden] * (depth - 1),
                                OCachePolicy(cfg.p_grad, cfg.t_stale, cfg.capacity),
                                feature_rows=frows, refresh_retained=cfg.refresh_retained,
                                dtype=cfg.dtype)
        if frows > 0:
            self.cache.backfill_features(features, self.end - self.start)
        self.source = OFeatureSource(features)
        self.metrics = []
        self.last = None   # (pruned, tape, node_grads, norms) of the last iteration

    def sample(self, idx, seeds):
        return sample_layered(self.start, self.end, self.col, self.num_nodes, seeds,
                              self.cfg.fanouts, batch_rng(self.cfg.seed, idx))

    def train_iteration(self, it, epoch, sub: OSubgraph, norms_override=None, grad_hook=None):
        """norms_override: optional {layer: fp64 norms aligned with the live
        rows} — the teacher-forced (lockstep) mode of SURVEY §8(c) Mode B.
        grad_hook(grads): called before SGD (data-parallel gradient averaging)."""
        before = self.cache.counters()
        f0 = self.source.fetched_bytes
        pr = prune_with_cache(sub, self.cache, it)
        h0, base = load_input(pr, self.cache, self.source, it, self.cfg.dtype)
        tape = forward_pass(self.network, sub.layers, h0, pr.compute_rows, pr.injected)
        loss, dlog = cross_entropy(tape.logits, self.labels[sub.seeds])
        grads, ng, _ = backward(self.network, sub.layers, tape, dlog, need_input=False)
        if grad_hook is not None:
            grad_hook(grads)
        sgd_step(self.network, grads, self.cfg.eta)
        used_norms = {}
        for layer in range(1, sub.num_layers):
            live = pr.layer_live[layer]
            if len(live) == 0:
                continue
            below = sub.layers[layer - 1]
            if norms_override is not None and layer in norms_override:
                nrm = np.asarray(norms_override[layer], np.float64)
            else:
                nrm = node_grad_norms(ng[layer - 1][live])
            used_norms[layer] = nrm
            self.cache.update_cache(layer, below.dst_nodes[live],
                                    below.dst_nodes[pr.compute_rows[layer - 1]],
                                    tape.h_layers[layer - 1][live], nrm, it)
        self.cache.end_iteration(it)
        after = self.cache.counters()
        d = {k: after[k] - before[k] for k in after}
        self.last = (pr, tape, ng, used_norms, grads)
        return OIterMetrics(it, epoch, len(sub.seeds), loss, self.source.fetched_bytes - f0, base,
                            sum(b.prune_writes for b in sub.layers), d["hits"], d["misses"],
                            d["admissions"], d["gradient_evictions"], d["staleness_evictions"],
                            d["forced_evictions"], d["feature_hits"], d["feature_misses"],
                            self.cache.valid_entries())

    def train(self, max_iters=None):
        batches = make_batches(self.train_ids, self.cfg)
        per_epoch = max(1, math.ceil(len(self.train_ids) / self.cfg.batch_size))
        for it, seeds in enumerate(batches):
            if max_iters is not None and it >= max_iters:
                break
            self.metrics.append(self.train_iteration(it, it // per_epoch, self.sample(it, seeds)))
        return self.metrics


def run_plain_loop(graph, features, labels, train_ids, cfg: OTrainConfig, num_classes=None, on_step=None):
    start, end, col = graph
    labels = np.asarray(labels, np.int64)
    ncls = int(num_classes or labels.max() + 1)
    depth = len(cfg.fanouts)
    dims = [features.shape[1]] + [cfg.hidden] * (depth - 1) + [ncls]
    net = init_network(cfg.kind, dims, network_rng(cfg.seed), cfg.dtype, cfg.heads)
    losses = []
    for idx, seeds in enumerate(make_batches(np.asarray(train_ids, np.int64), cfg)):
        sub = sample_layered(start, end, col, len(start), seeds, cfg.fanouts, batch_rng(cfg.seed, idx))
        h = features[sub.input_nodes].astype(cfg.dtype)
        tape = forward_pass(net, sub.layers, h)
        loss, dl = cross_entropy(tape.logits, labels[seeds])
        grads, _, _ = backward(net, sub.layers, tape, dl, need_input=False)
        sgd_step(net, grads, cfg.eta)
        losses.append(loss)
        if on_step is not None:
            on_step(idx, net)
    return net, losses


def full_graph_blocks(start, end, col, num_nodes, num_layers):
    """trainer.py:473-482 — whole-graph blocks; block 0's sources carry no
    in-edges (src_deg = 0), deeper blocks use the in-degree."""
    ids = np.arange(num_nodes, dtype=np.int64)
    deg = (np.asarray(end, np.int64) - np.asarray(start, np.int64))
    zero = np.zeros_like(deg)
    return [OBlock(ids, ids, np.asarray(start, np.int64), np.asarray(end, np.int64), np.asarray(col, np.int64), deg,
                   zero if b == 0 else deg) for b in range(num_layers)]


def evaluate(net: ONetwork, start, end, col, num_nodes, features, labels, ids):
    """trainer.py:485-506 — exact full-graph accuracy on `ids`; also returns
    the logits so tests can separate argmax near-ties."""
    h = np.asarray(features).astype(net.layers[0].weight.dtype)
    blocks = full_graph_blocks(start, end, col, num_nodes, net.num_layers)
    for l, blk in enumerate(blocks):
        h, _ = layer_forward_ctx(net.kind, net.layers[l], blk, h, np.arange(num_nodes, dtype=np.int64),
                                 l < net.num_layers - 1)
    ids = np.asarray(ids, np.int64)
    pred = h[ids].argmax(axis=1)
    return float((pred == np.asarray(labels)[ids]).mean()), h
