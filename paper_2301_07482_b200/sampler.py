"""Layered fan-out sampling on the GPU (drop-in for histgnn/sampler.py).

Same names, argument meaning and errors as the reference:
`SamplePlan` (sampler.py:26-41), `LayerBlock` (:44-71), `LayeredSubgraph`
(:74-92), `split_batches` (:95-101), `batch_rng` (:104-106),
`sample_layered` (:166-190) and `SubgraphProducer` (:193-263).

`sample_layered` runs one `hg_sample_layer` launch chain per fanout on the
device. The caller's numpy Generator supplies the PCG64 state (host-side
seeding, identical streams) and is advanced by exactly the number of draws the
reference would have consumed, so callers that reuse one generator across
calls see the same stream as with the reference. Blocks are bit-identical to
the reference's (tests/test_gpu_sampler.py).
"""

from __future__ import annotations

import queue
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graphs import Csr2Graph, _np

_DONE = object()
_M64 = (1 << 64) - 1


@dataclass(frozen=True)
class SamplePlan:
    """fanouts are listed outermost first: fanouts[0] expands the seeds."""

    fanouts: tuple
    batch_size: int
    rng_seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "fanouts", tuple(int(f) for f in self.fanouts))
        if len(self.fanouts) == 0:
            raise ValueError("need at least one fanout")
        if any(f < 1 for f in self.fanouts):
            raise ValueError(f"all fanouts must be >= 1, got {self.fanouts}")
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")


@dataclass
class LayerBlock:
    """One bipartite block; device tensors (int32 local ids / offsets).

    dst_nodes is a prefix view of src_nodes. `blk_off` keeps the build-time
    row extents (pruning only touches adj.end)."""

    dst_nodes: torch.Tensor
    src_nodes: torch.Tensor
    adj: Csr2Graph
    dst_deg: torch.Tensor
    src_deg: torch.Tensor = None
    blk_off: torch.Tensor = field(default=None, repr=False)

    @property
    def num_dst(self) -> int:
        return int(self.dst_nodes.shape[0])

    @property
    def num_src(self) -> int:
        return int(self.src_nodes.shape[0])

    @property
    def num_edges_built(self) -> int:
        return int(self.adj.col_indices.shape[0])

    def copy(self) -> "LayerBlock":
        return LayerBlock(self.dst_nodes, self.src_nodes, self.adj.copy(), self.dst_deg, self.src_deg,
                          self.blk_off)

    def record_stream(self, s):
        for t in (self.src_nodes, self.adj.start, self.adj.end, self.adj.col_indices, self.dst_deg,
                  self.src_deg, self.blk_off):
            if t is not None:
                t.record_stream(s)

    def as_numpy(self) -> dict:
        return {"dst": _np(self.dst_nodes).astype(np.int64), "src": _np(self.src_nodes).astype(np.int64),
                "start": self.adj.start_np, "end": self.adj.end_np, "col": self.adj.col_np,
                "dst_deg": _np(self.dst_deg).astype(np.int64),
                "src_deg": _np(self.src_deg).astype(np.int64)}


@dataclass
class LayeredSubgraph:
    """layers[0] is the innermost block; layers[-1].dst_nodes are the seeds."""

    seeds: np.ndarray
    layers: list

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    @property
    def input_nodes(self) -> torch.Tensor:
        return self.layers[0].src_nodes

    def copy(self) -> "LayeredSubgraph":
        return LayeredSubgraph(self.seeds, [b.copy() for b in self.layers])

    def record_stream(self, s):
        for b in self.layers:
            b.record_stream(s)


def split_batches(ids, batch_size: int, rng: np.random.Generator) -> list:
    """Host permutation, identical to the reference (sampler.py:95-101)."""
    ids = np.asarray(ids, dtype=np.int64)
    if batch_size < 1:
        raise ValueError("batch_size must be >= 1")
    perm = rng.permutation(ids)
    return [perm[i:i + batch_size] for i in range(0, len(perm), batch_size)]


def batch_rng(rng_seed: int, batch_index: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence((int(rng_seed), int(batch_index))))


class SamplerWorkspace:
    """Per-sampler O(N) scratch: epoch-stamped global->local map and the
    self-clearing node bitmap, plus the device-resident sampler state
    (u64[6]: PCG64 state hi/lo, inc hi/lo, draws consumed, g2l epoch).
    One workspace serves one stream at a time."""

    def __init__(self, num_nodes: int, device):
        self.num_nodes = int(num_nodes)
        self.device = device
        self.g2l = torch.full((self.num_nodes,), -1, dtype=torch.int64, device=device)
        self.bitmap = torch.zeros(((self.num_nodes + 31) // 32,), dtype=torch.int32, device=device)
        self.state = torch.zeros(6, dtype=torch.int64, device=device)
        self.state[5] = 1                       # epoch 0xFFFFFFFF is the g2l fill
        self.lock = threading.Lock()

    def set_pcg(self, state: int, inc: int, dst=None):
        """Stage the PCG64 state of a batch (and zero the draw counter)."""
        vals = [(state >> 64) & _M64, state & _M64, (inc >> 64) & _M64, inc & _M64, 0]
        host = torch.tensor([v - (1 << 64) if v >= (1 << 63) else v for v in vals], dtype=torch.int64)
        (dst if dst is not None else self.state)[:5].copy_(host.pin_memory(), non_blocking=True)

    @property
    def stream_pos(self):
        return self.state[4:5]


def pcg_words(state: int, inc: int) -> list:
    """The 5 int64 words hg_sample_layer reads from state_dev[0:5]."""
    vals = [(state >> 64) & _M64, state & _M64, (inc >> 64) & _M64, inc & _M64, 0]
    return [v - (1 << 64) if v >= (1 << 63) else v for v in vals]


def layer_bounds(B: int, fanouts, num_nodes: int):
    """Host upper bounds per sampling layer (outermost first): frontier sizes
    F[0..L] and sampled edges E[0..L-1]."""
    F, E = [B], []
    for f in fanouts:
        e = max(1, F[-1] * f)
        E.append(e)
        F.append(min(num_nodes, F[-1] + e))
    return F, E


class SampleSlot:
    """Preallocated outputs of one batch's layered sampling (upper-bound
    shapes, device counts): lets a sampled batch outlive the CUDA graph that
    produced it (the engine samples batch i+1 while it trains batch i)."""

    def __init__(self, g: Csr2Graph, B: int, fanouts):
        dev = g.start.device
        N = g.num_nodes
        self.layers = []
        F_max = B
        for fanout in fanouts:
            E_max = max(1, F_max * fanout)
            Fn_max = min(N, F_max + E_max)
            sb = _lib.query("hg_sample_layer_scratch_bytes", F_max, N)
            self.layers.append(dict(
                F_max=F_max, E_max=E_max, Fn_max=Fn_max, fanout=fanout,
                cand_off=torch.empty(F_max + 1, dtype=torch.int64, device=dev),
                blk_off=torch.empty(F_max + 1, dtype=torch.int32, device=dev),
                blk_end=torch.empty(F_max, dtype=torch.int32, device=dev),
                dst_deg=torch.empty(F_max, dtype=torch.int32, device=dev),
                src_flat=torch.empty(E_max, dtype=torch.int32, device=dev),
                col=torch.empty(E_max, dtype=torch.int32, device=dev),
                src=torch.empty(Fn_max, dtype=torch.int32, device=dev),
                counts=torch.empty(4, dtype=torch.int32, device=dev),
                scratch=torch.empty(sb, dtype=torch.uint8, device=dev), sb=sb))
            F_max = Fn_max
        self.key = None     # which batch the slot currently holds (set by the engine)


def sample_blocks_dev(g: Csr2Graph, frontier: torch.Tensor, F0_dev: torch.Tensor, B: int, fanouts,
                      ws: SamplerWorkspace, stream, slot: SampleSlot | None = None, layers=None) -> list:
    """Launch every sampling layer with host upper bounds and device counts
    (no host synchronisation). ws.state must hold the batch's PCG64 state.
    Returns per layer (outermost first): dict of device buffers (the slot's
    preallocated ones when `slot` is given). `layers` = (first, stop): only
    those layers (outermost = 0); a later call continues where an earlier
    one stopped (the engine forks the innermost, widest layer later)."""
    N = g.num_nodes
    sp = _lib.stream_ptr(stream)
    if slot is None:
        slot = SampleSlot(g, B, fanouts)
    first, stop = layers if layers is not None else (0, len(slot.layers))
    F_dev = F0_dev
    if first > 0:
        prev = slot.layers[first - 1]
        frontier, F_dev = prev["src"], prev["counts"][1:2]
    raw = []
    for L in slot.layers[first:stop]:
        _lib.call("hg_sample_layer", _lib.ptr(g.start), _lib.ptr(g.end), _lib.ptr(g.col_indices), N,
                  _lib.ptr(frontier), _lib.ptr(F_dev), L["F_max"], L["fanout"], _lib.ptr(ws.state),
                  _lib.ptr(ws.g2l), _lib.ptr(ws.bitmap), _lib.ptr(L["cand_off"]), _lib.ptr(L["blk_off"]),
                  _lib.ptr(L["blk_end"]), _lib.ptr(L["dst_deg"]), _lib.ptr(L["src_flat"]), _lib.ptr(L["col"]),
                  _lib.ptr(L["src"]), _lib.ptr(L["counts"]), _lib.ptr(L["scratch"]), L["sb"], sp)
        raw.append(dict(F_dev=F_dev, F_max=L["F_max"], E_max=L["E_max"], Fn_max=L["Fn_max"],
                        blk_off=L["blk_off"], blk_end=L["blk_end"], dst_deg=L["dst_deg"], col=L["col"],
                        src=L["src"], counts=L["counts"]))
        frontier, F_dev = L["src"], L["counts"][1:2]
    return raw


_default_ws: dict = {}
_default_ws_lock = threading.Lock()


def default_workspace(g: Csr2Graph) -> SamplerWorkspace:
    key = (id(g), g.col_indices.data_ptr())
    with _default_ws_lock:
        ws = _default_ws.get(key)
        if ws is None:
            ws = SamplerWorkspace(g.num_nodes, g.start.device)
            _default_ws.clear()
            _default_ws[key] = ws
    return ws


def _pcg_state(rng: np.random.Generator):
    bg = rng.bit_generator
    if not isinstance(bg, np.random.PCG64):
        raise ValueError("sample_layered needs a PCG64-backed Generator (batch_rng / default_rng)")
    st = bg.state
    return int(st["state"]["state"]), int(st["state"]["inc"])


def _advance(rng: np.random.Generator, draws: int) -> None:
    """Consume exactly `draws` uniform doubles, like rng.random(draws)."""
    if draws <= 0:
        return
    bg = rng.bit_generator
    before = bg.state
    bg.advance(draws)
    after = bg.state
    after["has_uint32"], after["uinteger"] = before["has_uint32"], before["uinteger"]
    bg.state = after


def sample_layered(g: Csr2Graph, seeds, plan: SamplePlan, rng: np.random.Generator, *,
                   workspace: SamplerWorkspace | None = None, stream=None,
                   seeds_dev: torch.Tensor | None = None) -> LayeredSubgraph:
    """Expand seeds through len(plan.fanouts) sampling blocks on the GPU.

    `seeds_dev` (int32 device tensor) lets a device-resident pipeline skip the
    host copy; the caller then guarantees unique, in-range seeds."""
    _lib.require_cuda()
    if seeds_dev is None:
        seeds = np.asarray(seeds, dtype=np.int64)
        if len(seeds) == 0:
            raise ValueError("empty seed set")
        if len(np.unique(seeds)) != len(seeds):
            raise ValueError("seed ids must be unique")
        if seeds.min() < 0 or seeds.max() >= g.num_nodes:
            raise ValueError("seed id out of range")
    else:
        seeds = seeds_dev
    ws = workspace or default_workspace(g)
    dev = g.start.device
    s = stream or torch.cuda.current_stream(dev)
    state, inc = _pcg_state(rng)
    with ws.lock, torch.cuda.stream(s):
        ws.set_pcg(state, inc)
        B = int(seeds.shape[0])
        if seeds_dev is None:
            frontier = torch.from_numpy(seeds.astype(np.int32)).pin_memory().to(dev, non_blocking=True)
        else:
            frontier = seeds_dev
        F_dev = torch.tensor([B], dtype=torch.int32).pin_memory().to(dev, non_blocking=True)
        raw = sample_blocks_dev(g, frontier, F_dev, B, plan.fanouts, ws, s)
        raw = [(r["F_dev"], r["blk_off"], r["blk_end"], r["dst_deg"], r["col"], r["src"], r["counts"])
               for r in raw]
        # one host round trip per batch: all block sizes + the draw count
        sizes = torch.cat([torch.stack([r[0][0] for r in raw]).to(torch.int64),
                           torch.stack([r[6][0] for r in raw]).to(torch.int64),
                           torch.stack([r[6][1] for r in raw]).to(torch.int64),
                           ws.stream_pos]).cpu().tolist()
    L = len(plan.fanouts)
    n_dst, n_e, n_src, draws = sizes[:L], sizes[L:2 * L], sizes[2 * L:3 * L], sizes[3 * L]
    _advance(rng, draws)
    blocks = []
    for li, (F_dev, blk_off, blk_end, dst_deg, col_local, src_out, counts) in enumerate(raw):
        F, E, S = n_dst[li], n_e[li], n_src[li]
        src_nodes = src_out[:S]
        adj = Csr2Graph(blk_off[:F], blk_end[:F], col_local[:E], F)
        blocks.append(LayerBlock(src_nodes[:F], src_nodes, adj, dst_deg[:F], None, blk_off[:F + 1]))
    blocks.reverse()
    for i, b in enumerate(blocks):
        b.src_deg = (torch.zeros(b.num_src, dtype=torch.int32, device=dev) if i == 0
                     else blocks[i - 1].dst_deg)
    return LayeredSubgraph(seeds=seeds, layers=blocks)


class SubgraphProducer:
    """Samples batches on a worker thread (own CUDA stream + workspace) into a
    bounded FIFO (sampler.py:193-263): at most `queue_capacity` finished
    subgraphs plus one in flight; yields (batch_index, subgraph) in order;
    close() stops the worker promptly."""

    def __init__(self, graph, batches, plan: SamplePlan, queue_capacity: int = 2):
        if queue_capacity < 1:
            raise ValueError("queue_capacity must be >= 1")
        self._graph = graph
        self._batches = list(batches)
        self._plan = plan
        self._queue: queue.Queue = queue.Queue(maxsize=queue_capacity)
        self._stop = threading.Event()
        self._thread = threading.Thread(target=self._work, daemon=True)
        self._started = False
        self._error = None
        self.batches_sampled = 0
        self._device = graph.start.device
        self._stream = torch.cuda.Stream(self._device)
        self._ws = SamplerWorkspace(graph.num_nodes, self._device)

    def _put(self, item) -> bool:
        while not self._stop.is_set():
            try:
                self._queue.put(item, timeout=0.05)
                return True
            except queue.Full:
                continue
        return False

    def _work(self):
        try:
            torch.cuda.set_device(self._device)
            for idx, seeds in enumerate(self._batches):
                if self._stop.is_set():
                    return
                sub = sample_layered(self._graph, seeds, self._plan, batch_rng(self._plan.rng_seed, idx),
                                     workspace=self._ws, stream=self._stream)
                ev = torch.cuda.Event()
                ev.record(self._stream)
                self.batches_sampled += 1
                if not self._put((idx, sub, ev)):
                    return
        except BaseException as e:  # surface worker failures to the consumer
            self._error = e
        self._put(_DONE)

    def start(self):
        if not self._started:
            self._started = True
            self._thread.start()

    def __iter__(self):
        self.start()
        while True:
            item = self._queue.get()
            if item is _DONE:
                if self._error is not None:
                    raise self._error
                return
            idx, sub, ev = item
            cur = torch.cuda.current_stream(self._device)
            cur.wait_event(ev)
            sub.record_stream(cur)
            yield idx, sub

    def close(self):
        self._stop.set()
        if self._started:
            while True:
                try:
                    self._queue.get_nowait()
                except queue.Empty:
                    break
            self._thread.join(timeout=5.0)

    def __enter__(self):
        self.start()
        return self

    def __exit__(self, *exc):
        self.close()
