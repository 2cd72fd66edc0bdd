"""Sync-free, shape-static training step (sample -> prune -> gather -> forward
-> loss -> backward -> SGD -> cache update), replayed as CUDA graphs, with the
sampler software-pipelined one batch ahead.

This is the B200 runtime behind `Trainer.train` / `Trainer.train_step`: the
same kernels as the API functions (sampler.py, trainer.prune_with_cache,
nn.py), but every buffer is sized from host upper bounds of the batch
(layer_bounds: F[l+1] <= F[l] * (1 + fanout)) and every element count is read
by the kernels from device memory, so a whole iteration issues no host
synchronisation. The step's inputs live in static device tensors (seeds,
labels, the batch's PCG64 state, the iteration number) that are refreshed
from pinned host staging before each launch; after the first eager
iterations (which size the cache rings, cache.py:79-91) the step is captured
once with torch.cuda.graph and replayed. The graph is re-captured only when a
cache table is reallocated (growth past the preallocated headroom,
cache.py:93-101). Sweeps themselves (every t_stale iterations) run on the host
between replays.

Pipelining: sampling depends only on the graph, the seeds and the batch's
PCG64 state, never on the weights or the cache, so when the caller names the
next batch the step also samples it, on a side stream, into the other of two
preallocated sample slots, concurrently with the training of the current
batch (two graph variants, one per slot parity). A batch's training reads the
slot filled by the previous step; a mismatch (no lookahead, or a different
batch than announced) falls back to sampling it first.
"""

from __future__ import annotations

import ctypes
import gc
import os
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .distributed import apply_sgd
from .nn import (FeatureRows, Injection, LayerKind, build_csc, resolve_features_dev, resolve_hit_rows_dev, cross_entropy_dev, inject_rows_dev, layer_backward_dev,
                 layer_forward_dev,
                 load_features_dev, pack_dgrad_weights, pack_forward_weights, ts_bytes)
from .sampler import SamplerWorkspace, SampleSlot, layer_bounds, pcg_words, sample_blocks_dev


@dataclass
class DevBlock:
    """A sampled block with upper-bound shapes (counts on the device)."""

    src_nodes: torch.Tensor
    blk_off: torch.Tensor
    end: torch.Tensor
    col: torch.Tensor
    dst_deg: torch.Tensor
    src_deg: torch.Tensor
    n_dst_dev: torch.Tensor
    n_src_dev: torch.Tensor
    num_dst: int            # upper bound
    num_src: int            # upper bound
    num_edges_built: int    # upper bound

    @property
    def adj(self):
        return self

    @property
    def start(self):
        return self.blk_off

    @property
    def col_indices(self):
        return self.col


# HG_NODE_PRIO=1: streams get priorities (cache updates > training > lookahead
# sampler) and the captured step is instantiated with per-node priorities
_NODE_PRIO = os.environ.get("HG_NODE_PRIO") == "1"
# Cache-hit rows of a hidden layer's output: read in place from the cache ring
# by the next layer (hg_resolve_hit_rows) or copied into the output first
# (hg_inject_rows). HG_INPLACE_HITS=auto (default): in place for local rings of
# at most HG_INPLACE_MAX_GB (8) -- measured C2 (2.4 GB rings) +2.4 %, C3 (24 GB
# rings, random hits over the whole ring) -1 % -- else copied; 1: always
# (owner-sharded rings too), 0: never.
_INPLACE_HITS = os.environ.get("HG_INPLACE_HITS", "auto")
_INPLACE_MAX_BYTES = float(os.environ.get("HG_INPLACE_MAX_GB", "8")) * (1 << 30)


def _hits_in_place(inj) -> bool:
    if _INPLACE_HITS == "0":
        return False
    if _INPLACE_HITS == "1":
        return True
    return inj.tables is None and inj.table.numel() * inj.table.element_size() <= _INPLACE_MAX_BYTES
# HG_SAMP_AT: where the lookahead sampler forks off the step (start | pruned |
# forward0 | forward1 | loss); later forks keep it off the early critical path
_SAMP_AT = os.environ.get("HG_SAMP_AT", "start")
# HG_SAMP_L0_AT: with the sampler forked at the start, where its innermost
# (widest, most expensive) layer forks (start | forward0 | forward1 | loss)
_SAMP_L0_AT = os.environ.get("HG_SAMP_L0_AT", "start")
# HG_FUSED_DZ=0: d_in rows + a separate dz gather per layer (A/B)
_FUSED_DZ = os.environ.get("HG_FUSED_DZ", "1") != "0"


class _Graph:
    __slots__ = ("graph", "pool", "out", "key", "launches", "exec", "__weakref__")


class PinnedRing:
    """Reusable pinned host buffers for the per-step host<->device copies (no
    pinned allocation per step). Slot i is handed out again only after the
    copy last issued from it has completed (its event) and after its current
    holder, if any, has been released (`owner._release()` reads it out)."""

    def __init__(self, depth: int, numel: int, dtype):
        self.bufs = [torch.empty(numel, dtype=dtype, pin_memory=True) for _ in range(depth)]
        self.events = [None] * depth
        self.owners = [None] * depth
        self.i = 0

    def acquire(self, owner=None):
        i = self.i
        self.i = (i + 1) % len(self.bufs)
        prev = self.owners[i]
        if prev is not None:
            o = prev()
            if o is not None:
                o._release()
        if self.events[i] is not None:
            self.events[i].synchronize()
        self.owners[i] = None if owner is None else weakref.ref(owner)
        return i, self.bufs[i]

    def issued(self, i: int, stream=None):
        ev = self.events[i] or torch.cuda.Event()
        ev.record(stream)
        self.events[i] = ev
        return ev


class StepEngine:
    def __init__(self, trainer, B: int):
        # weak back-reference: no Trainer <-> engine cycle, so a dropped trainer
        # (and its graph pools) is freed at once, never by a GC pass that could
        # run (and cudaFree) in the middle of another capture
        self.tr = weakref.proxy(trainer)
        self.B = int(B)
        cfg = trainer.cfg
        g = trainer.graph
        self.dev = trainer.device
        self.L = len(cfg.fanouts)
        self.F, self.E = layer_bounds(self.B, cfg.fanouts, g.num_nodes)
        self.ws = SamplerWorkspace(g.num_nodes, self.dev)
        self.seeds = torch.empty(self.B, dtype=torch.int32, device=self.dev)    # sampler input
        self.labels = torch.empty(self.B, dtype=torch.int32, device=self.dev)   # training input
        self.it = torch.zeros(1, dtype=torch.int32, device=self.dev)            # training iteration
        self.F0 = torch.full((1,), self.B, dtype=torch.int32, device=self.dev)
        self.slots = [SampleSlot(g, self.B, cfg.fanouts), SampleSlot(g, self.B, cfg.fanouts)]
        self.slot_words = [None, None]   # staged input words of the batch each slot holds
        self.cur = 0                     # slot of the next batch to train
        # block 0's sources carry no in-edges (src_deg = 0): one persistent zero vector
        self.zero_deg = torch.zeros(self.slots[0].layers[-1]["Fn_max"], dtype=torch.int32, device=self.dev)
        # role priorities under HG_NODE_PRIO=1 (lower = served first):
        # HG_PRIO_SAMP / HG_PRIO_MAIN / HG_PRIO_CACHE, default 0 / -1 / -2
        roles = {0: int(os.environ.get("HG_PRIO_SAMP", "0")), -1: int(os.environ.get("HG_PRIO_MAIN", "-1")),
                 -2: int(os.environ.get("HG_PRIO_CACHE", "-2"))}
        pr = (lambda p: dict(priority=roles[p])) if _NODE_PRIO else (lambda p: {})
        self._prio = pr
        self.samp_stream = torch.cuda.Stream(self.dev, **pr(0))
        # backward inputs that depend only on the pruned blocks / the weights
        # (transposed CSC, TS-packed dgrad weights) are built on prep_stream
        # during the forward; weight-gradient GEMMs run on wgrad_stream
        self.prep_stream = torch.cuda.Stream(self.dev, **pr(-1))
        self.wgrad_stream = torch.cuda.Stream(self.dev, **pr(-1))
        self.inj_stream = torch.cuda.Stream(self.dev, **pr(-1))      # cache-hit row injection (forward)
        # cache updates of layer l run on side stream l, overlapping the
        # backward of layers < l (they only read the forward tape and norms[l])
        self.upd_streams = {l: torch.cuda.Stream(self.dev, **pr(-2)) for l in range(1, self.L)}
        self.graphs = {}          # (slot, lookahead) -> _Graph
        self.out = None
        self.capturing = False
        self.timeline = None      # optional int64[32] %globaltimer marks per step (enable_timeline)
        self.timeline_names = []
        self.captures = 0         # graph (re-)captures so far
        self.up_ring = PinnedRing(4, 12 + 2 * self.B, torch.int32)   # input words, host -> HBM
        # the step's IterMetrics row, written on the device at its end (hg_metrics_row)
        cache = trainer.cache
        vecs = [lc.ctr for lc in cache.layers.values()] + [cache.gctr]
        self.m_vecs = torch.tensor([v.data_ptr() for v in vecs], dtype=torch.int64, device=self.dev)
        self.m_lens = torch.tensor([v.numel() for v in vecs], dtype=torch.int32, device=self.dev)
        self.m_nv = sum(v.numel() for v in vecs)
        self.m_prev = torch.zeros(self.m_nv, dtype=torch.int64, device=self.dev)
        self.m_row = torch.zeros(1 + self.m_nv + len(vecs) - 1 + 1 + 2 * self.L, dtype=torch.float64,
                                 device=self.dev)
        self.m_key = None          # (trainer generation) the prev snapshot is valid for

    @property
    def graph(self):
        """Any captured graph (None before the first capture)."""
        return next(iter(self.graphs.values())).graph if self.graphs else None

    # ------------------------------------------------------------ inputs

    def pack_inputs(self, iteration: int, seeds: np.ndarray, labels: np.ndarray, pcg: tuple) -> np.ndarray:
        """One batch's input words (host), as staged in HBM."""
        # layout (int32 words): [0:10) PCG64 words (5 x int64, 8-byte aligned),
        # [10] iteration, [11] pad, [12:12+B) seeds, [12+B:12+2B) labels
        words = np.empty(12 + 2 * self.B, dtype=np.int32)
        words[:10] = np.array(pcg_words(*pcg), dtype=np.int64).view(np.int32)
        words[10] = iteration
        words[11] = 0
        words[12: 12 + self.B] = seeds
        words[12 + self.B:] = labels
        return words

    def upload(self, words: np.ndarray) -> torch.Tensor:
        """Host words -> HBM through a reused pinned staging slot."""
        i, buf = self.up_ring.acquire()
        buf.numpy()[:] = words
        dev = torch.empty(buf.shape, dtype=buf.dtype, device=self.dev)
        dev.copy_(buf, non_blocking=True)
        self.up_ring.issued(i)
        return dev

    def _stage_sample(self, words_dev: torch.Tensor):
        self.ws.state[:5].copy_(words_dev[:10].view(torch.int64))
        self.seeds.copy_(words_dev[12: 12 + self.B])

    def _stage_train(self, words_dev: torch.Tensor):
        self.it.copy_(words_dev[10:11])
        self.labels.copy_(words_dev[12 + self.B: 12 + 2 * self.B])

    def holds(self, words_dev: torch.Tensor) -> bool:
        """True if the next slot already holds this batch (sampled ahead)."""
        w = self.slot_words[self.cur]
        return w is not None and w is words_dev

    def step_words(self, words_dev: torch.Tensor, next_words: torch.Tensor | None = None) -> dict:
        """Train the batch whose input words are `words_dev`; when
        `next_words` is given, also sample that batch ahead (pipelined)."""
        s = self.cur
        if not self.holds(words_dev):
            # prologue / unannounced batch: sample it first, on this stream
            self._stage_sample(words_dev)
            sample_blocks_dev(self.tr.graph, self.seeds, self.F0, self.B, self.tr.cfg.fanouts, self.ws,
                              torch.cuda.current_stream(self.dev), self.slots[s])
        self._stage_train(words_dev)
        ahead = next_words is not None
        if ahead:
            self._stage_sample(next_words)
        out = self._launch(s, ahead)
        self.slot_words[s] = None
        if ahead:
            self.slot_words[1 - s] = next_words
            self.cur = 1 - s
        return out

    def _launch(self, s: int, ahead: bool) -> dict:
        if self._graphable():
            gk = (s, ahead)
            g = self.graphs.get(gk)
            if g is None or g.key != self._key():
                g = self._capture(s, ahead)
            if g.exec is not None:
                _lib.call("hg_graph_launch", g.exec, _lib.stream_ptr())
            else:
                g.graph.replay()
            _lib.load().hg_count_graph_replay(g.launches)
            self.out = g.out
            return self.out
        self.out = self.run(s, ahead)
        return self.out

    def enable_timeline(self, on: bool = True):
        """Record %globaltimer at phase boundaries of every step (a one-thread
        kernel per mark, on the stream that reaches the boundary); read with
        timeline_ms(). Changes the captured graphs (re-captured on next launch)."""
        self.timeline = torch.zeros(32, dtype=torch.int64, device=self.dev) if on else None
        self.timeline_names = []
        self.graphs = {}

    def timeline_ms(self) -> dict:
        """Phase boundary times of the last step, ms after its first mark."""
        if self.timeline is None:
            return {}
        t = self.timeline.cpu().tolist()
        return {n: (t[i] - t[0]) / 1e6 for i, n in enumerate(self.timeline_names)}

    def _mark(self, name: str, stream):
        if self.timeline is None:
            return
        if name not in self.timeline_names:
            self.timeline_names.append(name)
        i = self.timeline_names.index(name)
        _lib.call("hg_mark_time", self.timeline.data_ptr() + 8 * i, _lib.stream_ptr(stream))

    # -------------------------------------------------------------- step

    def _blocks(self, s: int) -> list:
        """DevBlocks (innermost first) over the buffers of sample slot s."""
        layers = self.slots[s].layers
        blocks = []
        for li in range(self.L - 1, -1, -1):
            r = layers[li]
            F_dev = self.F0 if li == 0 else layers[li - 1]["counts"][1:2]
            blocks.append(DevBlock(r["src"], r["blk_off"], r["blk_end"], r["col"], r["dst_deg"], None, F_dev,
                                   r["counts"][1:2], r["F_max"], r["Fn_max"], r["E_max"]))
        for b, blk in enumerate(blocks):
            blk.src_deg = self.zero_deg if b == 0 else blocks[b - 1].dst_deg
        return blocks

    def run(self, s: int, ahead: bool) -> dict:
        """Enqueue one full iteration on the current stream (no host sync):
        train the batch in slot s; if `ahead`, sample the staged next batch
        into slot 1-s on the sampler stream meanwhile."""
        tr, cfg, net, cache = self.tr, self.tr.cfg, self.tr.network, self.tr.cache
        dev, L, B = self.dev, self.L, self.B
        stream = torch.cuda.current_stream(dev)
        sp = _lib.stream_ptr(stream)
        self._mark("start", stream)

        def launch_ahead(layers=None):
            # the next batch (or some of its layers), sampled on the side
            # stream from this point on
            samp = self.samp_stream
            samp.wait_stream(stream)
            with torch.cuda.stream(samp):
                sample_blocks_dev(tr.graph, self.seeds, self.F0, B, cfg.fanouts, self.ws, samp, self.slots[1 - s],
                                  layers=layers)
                if layers is None or layers[1] == L:
                    self._mark("next_sampled (side)", samp)

        if ahead and _SAMP_AT == "start":
            launch_ahead(None if _SAMP_L0_AT == "start" else (0, L - 1))
        # forward weight operands (depend only on the weights): packed on the
        # injection stream concurrently with the prune walk
        PTs = [None] * L
        packed = None
        if net.kind is not LayerKind.GAT:
            # buffers owned by the main stream (allocated here), filled on the side stream
            PTs = [torch.empty(ts_bytes(net.dims[b + 1], (2 * net.dims[b] if net.kind is LayerKind.SAGE_MEAN
                                                         else net.dims[b]) + 1), dtype=torch.uint8, device=dev)
                   for b in range(L)]
            self.inj_stream.wait_stream(stream)
            for b in range(L):
                pack_forward_weights(net, b, _lib.stream_ptr(self.inj_stream), out=PTs[b])
            packed = torch.cuda.Event()
            packed.record(self.inj_stream)
        blocks = self._blocks(s)
        cache.begin_step(self.it, sp)     # owner-sharded cache: peers' previous commits first

        # ---- prune walk + lookups (trainer.py:166-207) ----
        counts = torch.empty(2 * L, dtype=torch.int32, device=dev)
        keep, pos, rows, live = [None] * L, [None] * L, [None] * L, [None] * (L + 1)
        injected = [None] * L
        live_dst, inj_flag = None, None
        sb = _lib.query("hg_prune_scratch_bytes", max(max(b.num_src, b.num_dst) for b in blocks))
        scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        for b in range(L - 1, -1, -1):
            blk = blocks[b]
            keep[b] = torch.empty(blk.num_dst, dtype=torch.uint8, device=dev)
            rows[b] = torch.empty(blk.num_dst, dtype=torch.int32, device=dev)
            pos[b] = torch.empty(blk.num_dst, dtype=torch.int32, device=dev)
            src_mask = torch.empty(blk.num_src, dtype=torch.uint8, device=dev)
            live[b] = torch.empty(blk.num_src, dtype=torch.int32, device=dev)
            _lib.call("hg_prune_block", _lib.ptr(blk.n_dst_dev), blk.num_dst, _lib.ptr(blk.n_src_dev), blk.num_src,
                      _lib.ptr(live_dst), _lib.ptr(inj_flag), _lib.ptr(blk.blk_off), _lib.ptr(blk.end),
                      _lib.ptr(blk.col), _lib.ptr(keep[b]), _lib.ptr(rows[b]), _lib.ptr(pos[b]), _lib.ptr(src_mask),
                      _lib.ptr(live[b]), _lib.ptr(counts[2 * b:2 * b + 2]), _lib.ptr(cache.gctr), _lib.ptr(scratch),
                      sb, sp)
            live_dst, inj_flag = src_mask, None
            if b >= 1:
                lc = cache._layer(b)
                hit_flag = torch.empty(blk.num_src, dtype=torch.uint8, device=dev)
                hit_row = torch.empty(blk.num_src, dtype=torch.int32, device=dev)
                lc.lookup_dev(counts[2 * b + 1:2 * b + 2], blk.num_src, live[b], blk.src_nodes, blk.num_src, self.it,
                              hit_flag, hit_row, sp)
                inj = lc.injection(hit_flag, hit_row)
                if inj is not None:
                    inj_flag = hit_flag
                    injected[b - 1] = inj
            self._mark(f"pruned{b}", stream)

        def R_dev(b):
            return counts[2 * b:2 * b + 1]

        def n_live_dev(b):
            return counts[2 * b + 1:2 * b + 2]

        self._mark("pruned", stream)
        if ahead and _SAMP_AT == "pruned":
            launch_ahead()
        # ---- off-critical-path backward prep (overlaps the forward) ----
        prep = self.prep_stream
        prep.wait_stream(stream)
        cscs, w_ts = [None] * L, [None] * L
        with torch.cuda.stream(prep):
            psp = _lib.stream_ptr(prep)
            gat = net.kind is LayerKind.GAT   # GAT needs the transposed edges at every layer (dz for dW)
            # outermost layer first: the backward consumes them in that order,
            # each layer waits only for its own transposed edges / weights
            prep_done = [None] * L
            for l in range(L - 1, (-1 if gat else 0), -1):
                cscs[l] = build_csc(blocks[l], keep[l], pos[l], blocks[l].n_dst_dev, psp)
                if not gat:
                    w_ts[l] = pack_dgrad_weights(net, l, psp)
                prep_done[l] = torch.cuda.Event()
                prep_done[l].record(prep)
            self._mark("backward_prep (side)", prep)
        # ---- layer-0 input (trainer.py:326-343) ----
        b0 = blocks[0]
        region = cache.feature_table if cache.feature_table is not None else tr.features
        if tr.fused_input:
            # K5 fused into K6: only the row addresses; layer 0 reads the rows in place
            rowp = torch.empty(b0.num_src, dtype=torch.int64, device=dev)
            resolve_features_dev(n_live_dev(0), b0.num_src, live[0], b0.src_nodes, cache.feature_row_of_dev,
                                 region, tr.features, tr.feature_dim, tr._dtype_code, rowp, cache.gctr, sp)
            h = FeatureRows(rowp, tr._dtype_code, tr.feature_dim, b0.num_src)
        else:
            h = torch.empty((b0.num_src, tr.feature_dim), dtype=torch.float32, device=dev)
            load_features_dev(n_live_dev(0), b0.num_src, live[0], b0.src_nodes, cache.feature_row_of_dev, region,
                              tr.features, tr.feature_dim, tr._dtype_code, h, cache.gctr, sp)

        self._mark("loaded", stream)
        # injected (cache-hit) rows of every layer output depend only on the
        # prune walk: written on a side stream while the layers compute, issued
        # after the feature gather so that the gather runs without HBM contention
        # (SAGE / GCN; the main stream joins before the next layer reads them)
        h_outs = [None] * L
        h_refs = [None] * L              # in-place inputs of layer b + 1 (HG_INPLACE_HITS)
        inj_stream = None
        if net.kind is not LayerKind.GAT and any(x is not None for x in injected):
            # outputs allocated on the main stream (it owns and frees them; the
            # side stream is joined before any main-stream use after it)
            h_outs = [torch.empty((blocks[b].num_dst, net.dims[b + 1]), dtype=torch.float32, device=dev)
                      for b in range(L)]
            inj_stream = self.inj_stream
            inj_stream.wait_stream(stream)              # after the lookups and the feature gather
            isp = _lib.stream_ptr(inj_stream)
            for b in range(L):
                if injected[b] is None:
                    continue
                if b < L - 1 and _hits_in_place(injected[b]):
                    # layer b + 1 reads the hit rows in place from the cache
                    # ring (nothing else reads injected rows of h_out: the
                    # backward's ReLU mask and the cache writes touch computed
                    # rows only)
                    rowp = torch.empty(blocks[b].num_dst, dtype=torch.int64, device=dev)
                    h_refs[b] = resolve_hit_rows_dev(injected[b], h_outs[b], blocks[b].num_dst,
                                                     blocks[b].n_dst_dev, rowp, isp)
                else:
                    inject_rows_dev(injected[b], h_outs[b], blocks[b].num_dst, blocks[b].n_dst_dev, isp)
        # ---- forward (nn.py:260-297) ----
        tapes = []
        for b in range(L):
            blk = blocks[b]
            if b == 0 and packed is not None:
                stream.wait_event(packed)               # forward weight operands
            if b == 1 and inj_stream is not None:
                stream.wait_stream(inj_stream)          # layer 1 reads layer 0's injected rows
            t = layer_forward_dev(net, b, blk, h, rows[b], blk.num_dst, R_dev(b), b < L - 1, injected[b], sp,
                                  blk.n_dst_dev, live=live[b], n_live=blk.num_src, n_live_dev=n_live_dev(b),
                                  h_out=h_outs[b], injected_already=inj_stream is not None, PT=PTs[b])
            tapes.append(t)
            h = t.h_out if h_refs[b] is None else h_refs[b]
            self._mark(f"forward{b}", stream)
            if ahead and _SAMP_AT == f"forward{b}":
                launch_ahead()
            if ahead and _SAMP_AT == "start" and _SAMP_L0_AT == f"forward{b}":
                launch_ahead((L - 1, L))
        d_h, loss = cross_entropy_dev(tapes[-1].h_out, self.labels, B, net.dims[-1], sp)
        self._mark("forward+loss", stream)
        if ahead and _SAMP_AT == "loss":
            launch_ahead()
        if ahead and _SAMP_AT == "start" and _SAMP_L0_AT == "loss":
            launch_ahead((L - 1, L))

        # ---- backward (nn.py:300-320) + SGD, cache updates (cache.py:188-204) ----
        # layer l's admission/ring update (l >= 1) is forked onto its own
        # stream as soon as norms[l] exist; different layers' caches share no
        # state, and the joins below order them before anything that follows
        grads = net.new_grads(zero=False)
        norms = [None] * L
        keepalive = []
        for l in range(L - 1, -1, -1):
            blk = blocks[l]
            if prep_done[l] is not None:
                stream.wait_event(prep_done[l])
            d_prev, nrm = layer_backward_dev(net, l, blk, tapes[l], d_h, grads, l >= 1, keep[l], pos[l], live[l],
                                             blk.num_src, sp, blk.n_dst_dev, n_live_dev(l), csc=cscs[l],
                                             W_ts=w_ts[l], wgrad_stream=self.wgrad_stream, keepalive=keepalive,
                                             need_rows=keep[l - 1] if l >= 1 else None,
                                             dz_prev=(tapes[l - 1], pos[l - 1]) if l >= 1 and _FUSED_DZ else None)
            norms[l] = nrm
            d_h = d_prev
            self._mark(f"backward{l}", stream)
            if l >= 1:
                side = self.upd_streams[l]
                side.wait_stream(stream)
                with torch.cuda.stream(side):
                    cache._layer(l).update_dev(n_live_dev(l), blocks[l].num_src, live[l], blocks[l].src_nodes,
                                               norms[l], keep[l - 1], tapes[l - 1].h_out, self.it,
                                               cache.refresh_retained, _lib.stream_ptr(side),
                                               allow_alloc=not self.capturing,
                                               mark=lambda what, l=l, side=side: self._mark(f"cache{l}_{what} (side)",
                                                                                            side))
                    self._mark(f"cache_update{l} (side)", side)
        stream.wait_stream(prep)
        if packed is not None:
            stream.wait_stream(self.inj_stream)      # only when work was enqueued there (graph capture)
        stream.wait_stream(self.wgrad_stream)
        apply_sgd(tr.grad_hook, net, grads, cfg.eta)   # all-reduce (NCCL or fused P2P) + SGD
        self._mark("sgd", stream)
        for side in self.upd_streams.values():
            stream.wait_stream(side)
        cache.commit(sp)                  # owner-sharded cache: every rank's requests, in batch order
        self._mark("cache_committed", stream)
        if ahead:
            stream.wait_stream(self.samp_stream)
        self._mark("joined", stream)
        from ._state import CTR_VALID
        _lib.call("hg_metrics_row", _lib.ptr(self.m_vecs), _lib.ptr(self.m_lens), int(self.m_lens.numel()),
                  _lib.ptr(self.m_prev), _lib.ptr(loss), _lib.ptr(blocks[0].n_src_dev), _lib.ptr(counts), 2 * L,
                  CTR_VALID, _lib.ptr(self.m_row), sp)
        return dict(loss=loss, counts=counts, blocks=blocks, live=live, rows=rows, keep=keep, tapes=tapes,
                    norms=norms, grads=grads, injected=injected, keepalive=(keepalive, cscs, w_ts))

    # ------------------------------------------------------------ driver

    def _key(self):
        c = self.tr.cache
        return (tuple(None if lc.table is None else lc.table.data_ptr() for lc in c.layers.values()),
                None if self.timeline is None else self.timeline.data_ptr())

    def _graphable(self) -> bool:
        hook = self.tr.grad_hook
        return (self.tr.use_graphs and (hook is None or getattr(hook, "graph_safe", False))
                and all(lc.table is not None for lc in self.tr.cache.layers.values()))

    def _capture(self, s: int, ahead: bool) -> _Graph:
        gc.collect()
        torch.cuda.synchronize(self.dev)
        # a fresh private memory pool per capture: a replaced graph (and its
        # pool) is released when it is dropped here
        self.graphs.pop((s, ahead), None)
        g = _Graph()
        g.exec = None
        g.graph = torch.cuda.CUDAGraph(keep_graph=True) if _NODE_PRIO else torch.cuda.CUDAGraph()
        g.pool = torch.cuda.graph_pool_handle()
        self.capturing = True
        n0 = _lib.load().hg_kernel_launches()
        try:
            # capture on a side stream; the staged inputs were copied on the
            # current stream, which the capture stream waits for
            side = torch.cuda.Stream(self.dev, **self._prio(-1))
            side.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(side):
                with torch.cuda.graph(g.graph, pool=g.pool, stream=side):
                    g.out = self.run(s, ahead)
            torch.cuda.current_stream(self.dev).wait_stream(side)
        finally:
            self.capturing = False
        if _NODE_PRIO:
            ex = ctypes.c_void_p()
            _lib.call("hg_graph_instantiate", ctypes.c_void_p(g.graph.raw_cuda_graph()), ctypes.byref(ex))
            g.exec = ex.value
            weakref.finalize(g, _lib.call, "hg_graph_exec_destroy", ctypes.c_void_p(ex.value))
        # capture records the launches without executing them
        g.launches = _lib.load().hg_kernel_launches() - n0
        _lib.load().hg_count_graph_replay(-g.launches)
        self.captures += 1
        g.key = self._key()
        self.graphs[(s, ahead)] = g
        return g
