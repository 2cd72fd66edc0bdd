"""Block GNN compute on the GPU (drop-in for histgnn/nn.py).

Names and semantics follow the reference: `LayerKind` (nn.py:28-30),
`LayerParams`/`Network` (:33-70), `init_network` (:73-85, host RNG so weights
are bit-identical), `forward_pass` (:260-297), `backward` (:300-320),
`cross_entropy` (:326-343), `node_grad_norms` (:346-349), `sgd_step`
(:355-360). The work is done by hg_aggregate_fwd / hg_ts_linear_{fwd,dgrad,
wgrad} (tcgen05) / hg_inject_rows / hg_gather_dz / hg_build_csc /
hg_transpose_agg / hg_gat_* / hg_cross_entropy / hg_sgd.

Parameters of all layers live in ONE flat fp32 device buffer (one gradient
bucket for the data-parallel all-reduce); layer l occupies a
[(K_l + 1) x d_out] row-major slab = [W_self ; W_neigh ; bias] (SAGE, K = 2 d_in)
or [W ; bias] (GCN, K = d_in). `LayerParams` exposes reference-shaped views.

Dead rows: rows of an output that are neither computed nor injected are not
written on the device (no kernel reads them); numpy views of `h_layers` and
node gradients fill them with zeros like the reference.
"""

from __future__ import annotations

import enum
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .graphs import _np

KIND_GCN, KIND_SAGE = 0, 1

def _wgrad_splits(R: int, K1: int, n: int) -> int:
    """Split-K factor for dP = A^T dz: ~1 CTA per SM, >= 8 chunks of 32 rows each."""
    tiles = ((K1 + 127) // 128) * ((n + 255) // 256)
    chunks = max(1, (R + 31) // 32)
    return max(1, min(148 // tiles, chunks // 8))


class LayerKind(enum.Enum):
    GCN = "gcn"
    SAGE_MEAN = "sage_mean"
    GAT = "gat"        # not in the reference (nn.py:28-30); defined by oracle/gat.py


def _kind_code(kind: LayerKind) -> int:
    return KIND_SAGE if kind is LayerKind.SAGE_MEAN else KIND_GCN


def _slab_k(kind: LayerKind, fi: int) -> int:
    """Rows above the bias row of a layer slab: SAGE [W_self; W_neigh],
    GCN [W], GAT [W; a_src; a_dst]."""
    if kind is LayerKind.SAGE_MEAN:
        return 2 * fi
    if kind is LayerKind.GAT:
        return fi + 2
    return fi


@dataclass
class LayerParams:
    """Views into the flat parameter (or gradient) buffer."""

    weight: torch.Tensor
    bias: torch.Tensor
    weight_neigh: torch.Tensor | None = None
    att_src: torch.Tensor | None = None      # GAT only
    att_dst: torch.Tensor | None = None

    def named_arrays(self):
        pairs = [("weight", self.weight), ("bias", self.bias)]
        if self.weight_neigh is not None:
            pairs.append(("weight_neigh", self.weight_neigh))
        if self.att_src is not None:
            pairs += [("att_src", self.att_src), ("att_dst", self.att_dst)]
        return pairs

    def numpy(self):
        return {k: _np(v) for k, v in self.named_arrays()}


def _slab_views(flat: torch.Tensor, kind: LayerKind, dims, offsets, in_dim=None):
    """Reference-shaped views of every layer slab. `dims` are the storage
    widths; layer 0's input may be stored zero-padded (in_dim = the logical
    feature width): its weight views then take the first in_dim rows of each
    [fi_pad]-row block, so the padded rows are invisible (and stay zero: their
    gradients are products with zero feature columns)."""
    out = []
    for l, (fi, fo) in enumerate(zip(dims[:-1], dims[1:])):
        K = _slab_k(kind, fi)
        fl = in_dim if (l == 0 and in_dim is not None) else fi
        slab = flat[offsets[l]:offsets[l] + (K + 1) * fo].view(K + 1, fo)
        if kind is LayerKind.SAGE_MEAN:
            out.append(LayerParams(slab[:fl], slab[K], slab[fi:fi + fl]))
        elif kind is LayerKind.GAT:
            out.append(LayerParams(slab[:fl], slab[K], None, slab[fi], slab[fi + 1]))
        else:
            out.append(LayerParams(slab[:fl], slab[K], None))
    return out


def pad_width(d: int, itemsize: int = 4) -> int:
    """Row width the kernels need: rows move as 16-byte vectors."""
    m = max(1, 16 // itemsize)
    return -(-int(d) // m) * m


def pad_columns(x, width: int):
    """Zero-pad the columns of a 2-d host array / device tensor to `width`
    (returned unchanged when already that wide)."""
    if x.shape[1] == width:
        return x
    if isinstance(x, torch.Tensor):
        out = torch.zeros((x.shape[0], width), dtype=x.dtype, device=x.device)
        out[:, :x.shape[1]] = x
        return out
    x = np.asarray(x)
    out = np.zeros((x.shape[0], width), dtype=x.dtype)
    out[:, :x.shape[1]] = x
    return out


def _offsets(kind, dims):
    offs, o = [], 0
    for fi, fo in zip(dims[:-1], dims[1:]):
        K = _slab_k(kind, fi)
        offs.append(o)
        o += (K + 1) * fo
    return offs, o


@dataclass
class Network:
    kind: LayerKind
    dims: list
    flat: torch.Tensor                       # all parameters, fp32, device
    offsets: list
    layers: list = field(default_factory=list)
    heads: list | None = None                # GAT heads per layer (hidden H, output 1)
    in_dim: int | None = None                # logical layer-0 input width when dims[0] is padded

    def __post_init__(self):
        if not self.layers:
            self.layers = _slab_views(self.flat, self.kind, self.dims, self.offsets, self.in_dim)
        if self.heads is None:
            self.heads = [1] * (len(self.dims) - 1)

    @property
    def num_layers(self) -> int:
        return len(self.dims) - 1

    @property
    def logical_dims(self) -> list:
        """Reference layer widths (dims[0] unpadded)."""
        return [self.in_dim if self.in_dim is not None else self.dims[0]] + list(self.dims[1:])

    @property
    def dtype(self):
        return np.float32

    def slab(self, l: int) -> torch.Tensor:
        fi, fo = self.dims[l], self.dims[l + 1]
        K = _slab_k(self.kind, fi)
        return self.flat[self.offsets[l]:self.offsets[l] + (K + 1) * fo].view(K + 1, fo)

    def checksum_bytes(self) -> bytes:
        """Same byte order as histgnn Network.checksum_bytes (nn.py:65-70)."""
        return b"".join(np.ascontiguousarray(_np(a)).tobytes() for p in self.layers for _, a in p.named_arrays())

    def new_grads(self, zero: bool = True) -> "Grads":
        """zero=False: every slab is fully overwritten by the dP GEMMs (beta=0)."""
        return Grads(self, torch.zeros_like(self.flat) if zero else torch.empty_like(self.flat))


@dataclass
class Grads:
    net: Network
    flat: torch.Tensor

    @property
    def layers(self):
        return _slab_views(self.flat, self.net.kind, self.net.dims, self.net.offsets, self.net.in_dim)

    def __getitem__(self, l):
        return self.layers[l]

    def __len__(self):
        return self.net.num_layers

    def slab(self, l):
        fi, fo = self.net.dims[l], self.net.dims[l + 1]
        K = _slab_k(self.net.kind, fi)
        return self.flat[self.net.offsets[l]:self.net.offsets[l] + (K + 1) * fo].view(K + 1, fo)


def init_network(kind: LayerKind, dims, rng: np.random.Generator, dtype=np.float32, device=None,
                 heads: int = 4, in_pad: int | None = None) -> Network:
    """Glorot-uniform weights, zero biases (nn.py:73-85); host RNG, then upload.
    GAT (oracle/gat.py init_layer): per layer W, then a_src, a_dst ~
    U(+-sqrt(6/(F+1))); `heads` on hidden layers, 1 on the output layer."""
    _lib.require_cuda()
    if np.dtype(dtype) != np.float32:
        raise ValueError("the device network computes in fp32")
    dims = [int(d) for d in dims]
    L = len(dims) - 1
    hl = [heads if l < L - 1 else 1 for l in range(L)] if kind is LayerKind.GAT else [1] * L
    sdims = [int(in_pad) if in_pad else dims[0]] + dims[1:]   # storage widths
    if sdims[0] < dims[0]:
        raise ValueError("in_pad must be >= the input width")
    offs, total = _offsets(kind, sdims)
    host = np.zeros(total, dtype=np.float32)
    for l, (fi, fo) in enumerate(zip(dims[:-1], dims[1:])):
        fs = sdims[l]
        s = np.sqrt(6.0 / (fi + fo))
        w = rng.uniform(-s, s, size=(fi, fo)).astype(np.float32)
        K = _slab_k(kind, fs)
        slab = host[offs[l]:offs[l] + (K + 1) * fo].reshape(K + 1, fo)
        slab[:fi] = w
        if kind is LayerKind.SAGE_MEAN:
            slab[fs:fs + fi] = rng.uniform(-s, s, size=(fi, fo)).astype(np.float32)
        elif kind is LayerKind.GAT:
            if fo % hl[l]:
                raise ValueError(f"layer {l}: d_out {fo} not divisible by {hl[l]} heads")
            la = np.sqrt(6.0 / (fo // hl[l] + 1))
            slab[fs] = rng.uniform(-la, la, size=fo).astype(np.float32)
            slab[fs + 1] = rng.uniform(-la, la, size=fo).astype(np.float32)
    flat = torch.from_numpy(host).to(torch.device(device or "cuda"))
    return Network(kind, sdims, flat, offs, heads=hl, in_dim=dims[0] if sdims[0] != dims[0] else None)


def network_from_numpy(kind: LayerKind, layers, device=None, heads=None, in_pad: int | None = None) -> Network:
    """Pack reference-style per-layer arrays (weight, bias, weight_neigh /
    att_src, att_dst); in_pad stores layer 0's input zero-padded (pad_width)."""
    dims = [layers[0]["weight"].shape[0]] + [p["weight"].shape[1] for p in layers]
    if in_pad is None:
        in_pad = pad_width(dims[0])
    sdims = [int(in_pad)] + dims[1:]
    offs, total = _offsets(kind, sdims)
    host = np.zeros(total, dtype=np.float32)
    for l, p in enumerate(layers):
        fi, fo = p["weight"].shape
        fs = sdims[l]
        K = _slab_k(kind, fs)
        slab = host[offs[l]:offs[l] + (K + 1) * fo].reshape(K + 1, fo)
        slab[:fi] = p["weight"]
        slab[K] = p["bias"]
        if kind is LayerKind.SAGE_MEAN:
            slab[fs:fs + fi] = p["weight_neigh"]
        elif kind is LayerKind.GAT:
            slab[fs] = p["att_src"]
            slab[fs + 1] = p["att_dst"]
    return Network(kind, sdims, torch.from_numpy(host).to(torch.device(device or "cuda")), offs,
                   heads=None if heads is None else list(heads), in_dim=dims[0] if sdims[0] != dims[0] else None)


# ---------------------------------------------------------------- tapes


@dataclass
class LayerTape:
    rows: torch.Tensor          # int32 [R] compute rows (sorted)
    R: int
    R_dev: torch.Tensor         # int32 [1]
    A: torch.Tensor             # [R, K+4] GEMM operand (self|agg|1|pad)
    K: int
    relu: bool
    h_out: torch.Tensor         # [n_dst, d_out] (dead rows unwritten)
    inj: object = None          # Injection or None
    row_w: torch.Tensor | None = None   # fp32 [R] SAGE mean weights 1/cnt (the backward's edge weights)

    @property
    def valid_rows(self) -> torch.Tensor:
        """bool [n_dst]: rows that hold data (computed or injected)."""
        valid = torch.zeros(self.h_out.shape[0], dtype=torch.bool, device=self.h_out.device)
        if self.R:
            valid[self.rows.long()] = True
        if self.inj is not None:
            valid |= self.inj.flag.bool()
        return valid


@dataclass
class BatchTape:
    h_input: torch.Tensor
    entries: list
    h_layers: list              # device tensors (dead rows unwritten)

    @property
    def logits(self) -> torch.Tensor:
        return self.h_layers[-1]

    def h_layer_np(self, l: int) -> np.ndarray:
        """Reference view of h_layers[l]: dead rows are zeros."""
        h = self.h_layers[l]
        valid = self.entries[l].valid_rows
        return _np(torch.where(valid[:, None], h, torch.zeros((), dtype=h.dtype, device=h.device)))


@dataclass
class Injection:
    """Rows of a block output served from a table instead of computed."""

    flag: torch.Tensor          # uint8 [n_dst]
    row: torch.Tensor           # int32 [n_dst] row in `table` (owner << 26 | row with `tables`)
    table: torch.Tensor         # [*, d_out] fp32 (None when the rows live in the owners' rings)
    locals_dev: torch.Tensor | None = None
    tables: torch.Tensor | None = None   # int64 [P] ring base pointers (owner-sharded cache)
    dim: int = 0                          # row width of the rings (with `tables`)


def load_features_dev(n_live_dev, n_max: int, live, src_nodes, feature_row_of, region, feats, dim: int,
                      dtype_code: int, out: torch.Tensor, gctr, stream) -> None:
    """Layer-0 input rows (trainer.py:326-343) through hg_load_features with
    a workspace (the TMA copy path for fp32 features)."""
    if hasattr(feats, "load_rows"):   # sharding.ShardedFeatures (peer shards over NVLink)
        feats.load_rows(n_live_dev, n_max, live, src_nodes, feature_row_of,
                        region if feature_row_of is not None else None, out, gctr, stream)
        return
    sb = int(_lib.query("hg_load_features_scratch_bytes", max(int(n_max), 1)))
    scratch = torch.empty(sb, dtype=torch.uint8, device=out.device)
    _lib.call("hg_load_features", _lib.ptr(n_live_dev), n_max, _lib.ptr(live), _lib.ptr(src_nodes),
              _lib.ptr(feature_row_of), _lib.ptr(region), _lib.ptr(feats), dim, dtype_code, _lib.ptr(out),
              _lib.ptr(gctr), _lib.ptr(scratch), sb, stream)


@dataclass
class FeatureRows:
    """Layer-0 input by reference (K5 fused into K6): rowp[loc] is the address
    of local source loc's feature row (region row, table row or owner-shard
    row); the layer-0 aggregation reads the rows in place."""

    rowp: torch.Tensor          # int64 [n_src]
    dtype_code: int             # 0 fp32, 1 fp16 feature rows; 2 fp32 hidden-layer rows
    dim: int                    # (padded) row width
    num_rows: int

    @property
    def shape(self):
        return (self.num_rows, self.dim)

    @property
    def device(self):
        return self.rowp.device


def resolve_features_dev(n_live_dev, n_max: int, live, src_nodes, feature_row_of, region, feats, dim: int,
                         dtype_code: int, rowp: torch.Tensor, gctr, stream) -> None:
    """hg_resolve_feature_rows: rowp[live[i]] = address of the row (the
    accounting of load_features_dev, no row copied)."""
    if hasattr(feats, "load_rows"):   # sharding.ShardedFeatures
        _lib.call("hg_resolve_feature_rows", _lib.ptr(n_live_dev), n_max, _lib.ptr(live), _lib.ptr(src_nodes),
                  _lib.ptr(feature_row_of), _lib.ptr(region if feature_row_of is not None else None), None,
                  _lib.ptr(feats.ptrs_dev), _lib.ptr(feats.bounds_dev), feats.num_shards, feats.local_shard, dim,
                  dtype_code, _lib.ptr(rowp), _lib.ptr(gctr), _lib.ptr(feats.owner_rows), stream)
        return
    _lib.call("hg_resolve_feature_rows", _lib.ptr(n_live_dev), n_max, _lib.ptr(live), _lib.ptr(src_nodes),
              _lib.ptr(feature_row_of), _lib.ptr(region), _lib.ptr(feats), None, None, 0, 0, dim, dtype_code,
              _lib.ptr(rowp), _lib.ptr(gctr), None, stream)


def _dev_count(n: int, dev) -> torch.Tensor:
    return torch.tensor([n], dtype=torch.int32, device=dev)


@dataclass
class GatTape(LayerTape):
    """GAT forward state kept for the backward (oracle/gat.py GATTape)."""
    z: torch.Tensor = None         # [n_src, HF] (rows of `live` valid)
    el: torch.Tensor = None        # [n_src, H]
    er: torch.Tensor = None
    mx: torch.Tensor = None        # [R, H] per-row logit max
    ssum: torch.Tensor = None      # [R, H] per-row exp sums
    live: torch.Tensor = None
    n_live: int = 0
    n_live_dev: torch.Tensor = None
    heads: int = 1


def _att_rows(slab: torch.Tensor, d_in: int):
    """(a_src, a_dst, bias) rows of a GAT slab [W; a_src; a_dst; bias]."""
    return slab[d_in], slab[d_in + 1], slab[d_in + 2]


def gat_layer_forward_dev(net: Network, l: int, blk, h_in, rows, R, R_dev, act, inj, stream, n_dst_dev,
                          live, n_live, n_live_dev) -> GatTape:
    """GAT block layer (oracle/gat.py layer_forward) on the device:
    z[live] = h_in[live] W on tcgen05, per-head scores, then the attention
    softmax + aggregation over the surviving edges and the self loop."""
    dev = h_in.device
    d_in, HF, H = net.dims[l], net.dims[l + 1], net.heads[l]
    if live is None:
        live = torch.arange(blk.num_src, dtype=torch.int32, device=dev)
        n_live, n_live_dev = blk.num_src, _dev_count(blk.num_src, dev)
    A = torch.empty(ts_bytes(n_live, d_in), dtype=torch.uint8, device=dev)
    if isinstance(h_in, FeatureRows):     # layer 0: the transform operand straight from the feature rows
        if h_in.dim != d_in:
            raise ValueError(f"feature rows of width {h_in.dim} for a layer of input width {d_in}")
        _lib.call("hg_gather_rows_ts", _lib.ptr(n_live_dev), n_live, _lib.ptr(live), _lib.ptr(h_in.rowp),
                  h_in.dtype_code, d_in, _lib.ptr(A), stream)
    else:
        _lib.call("hg_gather_dz", _lib.ptr(n_live_dev), n_live, _lib.ptr(live), _lib.ptr(h_in), None, d_in, 0,
                  _lib.ptr(A), stream)
    slab = net.slab(l)
    PT = torch.empty(ts_bytes(HF, d_in), dtype=torch.uint8, device=dev)      # TS(W^T)
    _lib.call("hg_ts_pack", _lib.ptr(slab), HF, 1, HF, d_in, HF, _lib.ptr(PT), stream)
    z = torch.empty((blk.num_src, HF), dtype=torch.float32, device=dev)
    _lib.call("hg_ts_linear_fwd", _lib.ptr(n_live_dev), n_live, _lib.ptr(A), d_in, _lib.ptr(PT), HF, _lib.ptr(live),
              0, _lib.ptr(z), stream)
    a_src, a_dst, bias = _att_rows(slab, d_in)
    el = torch.empty((blk.num_src, H), dtype=torch.float32, device=dev)
    er = torch.empty((blk.num_src, H), dtype=torch.float32, device=dev)
    _lib.call("hg_gat_scores", _lib.ptr(n_live_dev), n_live, _lib.ptr(live), _lib.ptr(z), HF, H, _lib.ptr(a_src),
              _lib.ptr(a_dst), _lib.ptr(el), _lib.ptr(er), stream)
    n_dst = blk.num_dst
    h_out = torch.empty((n_dst, HF), dtype=torch.float32, device=dev)
    mx = torch.empty((max(R, 1), H), dtype=torch.float32, device=dev)
    ssum = torch.empty((max(R, 1), H), dtype=torch.float32, device=dev)
    _lib.call("hg_gat_aggregate", _lib.ptr(R_dev), R, _lib.ptr(rows), _lib.ptr(blk.adj.start), _lib.ptr(blk.adj.end),
              _lib.ptr(blk.adj.col_indices), _lib.ptr(z), _lib.ptr(el), _lib.ptr(er), HF, H, _lib.ptr(bias), int(act),
              _lib.ptr(h_out), _lib.ptr(mx), _lib.ptr(ssum), stream)
    if inj is not None:
        nd = n_dst_dev if n_dst_dev is not None else _dev_count(n_dst, dev)
        inject_rows_dev(inj, h_out, n_dst, nd, stream)
    return GatTape(rows, R, R_dev, A, d_in, act, h_out, inj, z=z, el=el, er=er, mx=mx, ssum=ssum, live=live,
                   n_live=n_live, n_live_dev=n_live_dev, heads=H)


def gat_layer_backward_dev(net: Network, l: int, blk, t: GatTape, d_h, grads, need_input, keep, pos_of, stream,
                           n_dst_dev=None, csc=None, wgrad_stream=None, keepalive=None):
    """oracle/gat.py layer_backward on the device. Writes the layer's slab of
    `grads`; returns (d_in [n_src, d_in] valid on the live rows, fp64 norms
    aligned with the live list) or (None, None)."""
    dev = d_h.device
    d_in, HF, H = net.dims[l], net.dims[l + 1], t.heads
    R, n_live = t.R, t.n_live
    if n_dst_dev is None:
        n_dst_dev = _dev_count(blk.num_dst, dev)
    gz = torch.empty((max(R, 1), HF), dtype=torch.float32, device=dev)
    cc = torch.empty((max(R, 1), H), dtype=torch.float32, device=dev)
    der = torch.empty((max(R, 1), H), dtype=torch.float32, device=dev)
    part = torch.empty(int(_lib.query("hg_gat_param_scratch_bytes", HF)) // 4, dtype=torch.float32, device=dev)
    part_dst, part_src = part[: 2 * (part.numel() // 3)], part[2 * (part.numel() // 3):]
    _lib.call("hg_gat_bwd_dst", _lib.ptr(t.R_dev), R, _lib.ptr(t.rows), _lib.ptr(blk.adj.start), _lib.ptr(blk.adj.end),
              _lib.ptr(blk.adj.col_indices), _lib.ptr(t.z), _lib.ptr(t.el), _lib.ptr(t.er), _lib.ptr(t.mx),
              _lib.ptr(t.ssum), _lib.ptr(d_h), _lib.ptr(t.h_out), int(t.relu), HF, H, _lib.ptr(gz), _lib.ptr(cc),
              _lib.ptr(der), _lib.ptr(part_dst), stream)
    if csc is None:
        csc = build_csc(blk, keep, pos_of, n_dst_dev, stream)
    slab = net.slab(l)
    a_src, a_dst, _ = _att_rows(slab, d_in)
    dz = torch.empty(ts_bytes(n_live, HF), dtype=torch.uint8, device=dev)
    dl = torch.empty((max(n_live, 1), H), dtype=torch.float32, device=dev)
    _lib.call("hg_gat_bwd_src", _lib.ptr(t.n_live_dev), n_live, _lib.ptr(t.live), _lib.ptr(csc.seg_lo),
              _lib.ptr(csc.seg_hi), _lib.ptr(csc.vals), _lib.ptr(t.rows), _lib.ptr(n_dst_dev), _lib.ptr(pos_of),
              _lib.ptr(t.z), _lib.ptr(t.el), _lib.ptr(t.er), _lib.ptr(t.mx), _lib.ptr(t.ssum), _lib.ptr(gz),
              _lib.ptr(cc), _lib.ptr(der), _lib.ptr(a_src), _lib.ptr(a_dst), HF, H, _lib.ptr(dz), _lib.ptr(dl),
              _lib.ptr(part_src), stream)
    t.bwd = (gz, cc, der, dl)     # kept for inspection (tools/gat_diag.py)
    gslab = grads.slab(l)
    g_src, g_dst, g_bias = _att_rows(gslab, d_in)
    _lib.call("hg_gat_param_grads", R, n_live, HF, _lib.ptr(part_dst), _lib.ptr(part_src), _lib.ptr(g_src),
              _lib.ptr(g_dst), _lib.ptr(g_bias), stream)
    splits = _wgrad_splits(n_live, d_in, HF)

    def wgrad(sp):
        wp = torch.empty(splits * d_in * HF, dtype=torch.float32, device=dev)
        _lib.call("hg_ts_linear_wgrad", _lib.ptr(t.n_live_dev), n_live, _lib.ptr(t.A), d_in, _lib.ptr(dz), HF,
                  _lib.ptr(gslab), _lib.ptr(wp), splits, sp)
        return wp

    if wgrad_stream is not None:
        cur = torch.cuda.current_stream(dev)
        wgrad_stream.wait_stream(cur)
        with torch.cuda.stream(wgrad_stream):
            wp = wgrad(_lib.stream_ptr(wgrad_stream))
        if keepalive is not None:
            keepalive.extend([dz, wp, part, gz, cc, der, dl])
    else:
        wgrad(stream)
    if not need_input:
        return None, None
    W_ts = pack_dgrad_weights(net, l, stream)
    SG = torch.empty((max(n_live, 1), d_in), dtype=torch.float32, device=dev)
    _lib.call("hg_ts_linear_dgrad", _lib.ptr(t.n_live_dev), n_live, _lib.ptr(dz), HF, _lib.ptr(W_ts), d_in,
              _lib.ptr(SG), stream)
    d_full = torch.empty((blk.num_src, d_in), dtype=torch.float32, device=dev)
    norms = torch.empty(max(n_live, 1), dtype=torch.float64, device=dev)
    _lib.call("hg_gat_scatter_norms", _lib.ptr(t.n_live_dev), n_live, _lib.ptr(t.live), _lib.ptr(SG), d_in,
              _lib.ptr(d_full), _lib.ptr(norms), stream)
    if keepalive is not None:
        keepalive.extend([W_ts, SG])
    return d_full, norms[:n_live]


def inject_rows_dev(inj: Injection, h_out: torch.Tensor, n_dst: int, n_dst_dev, stream) -> None:
    if inj.tables is not None:       # owner-sharded cache: straight from the owners' rings
        _lib.call("hg_inject_rows_sharded", _lib.ptr(n_dst_dev), n_dst, _lib.ptr(inj.flag), _lib.ptr(inj.row),
                  _lib.ptr(inj.tables), int(h_out.shape[1]), _lib.ptr(h_out), stream)
        return
    """h_out[r] = table[row[r]] for the injected rows (nn.py:290-293)."""
    _lib.call("hg_inject_rows", _lib.ptr(n_dst_dev), n_dst, _lib.ptr(inj.flag), _lib.ptr(inj.row),
              _lib.ptr(inj.table), int(h_out.shape[1]), _lib.ptr(h_out), stream)


def resolve_hit_rows_dev(inj: Injection, h_out: torch.Tensor, n_dst: int, n_dst_dev, rowp: torch.Tensor,
                         stream) -> FeatureRows:
    """The next layer's input by reference: rowp[r] = the cache row of every
    injected r (local table or owner ring), else h_out row r; the layer reads
    its sources in place (hg_aggregate_fwd_rows), no hit row is copied."""
    _lib.call("hg_resolve_hit_rows", _lib.ptr(n_dst_dev), n_dst, _lib.ptr(inj.flag), _lib.ptr(inj.row),
              _lib.ptr(inj.table if inj.tables is None else None), _lib.ptr(inj.tables), int(h_out.shape[1]),
              _lib.ptr(h_out), _lib.ptr(rowp), stream)
    return FeatureRows(rowp, 2, int(h_out.shape[1]), n_dst)   # dtype 2: hidden-layer fp32 rows


def layer_forward_dev(net: Network, l: int, blk, h_in: torch.Tensor, rows: torch.Tensor, R: int,
                      R_dev: torch.Tensor, act: bool, inj: Injection | None, stream,
                      n_dst_dev: torch.Tensor | None = None, live=None, n_live=None, n_live_dev=None,
                      h_out: torch.Tensor | None = None, injected_already: bool = False,
                      PT: torch.Tensor | None = None) -> LayerTape:
    """h_out / injected_already: the engine preallocates the output and writes
    the injected rows on a side stream (they do not depend on the layer);
    PT: the forward weight operand packed ahead (pack_forward_weights)."""
    if net.kind is LayerKind.GAT:
        if h_in.shape[0] != blk.num_src:
            raise ValueError(f"h_in has {h_in.shape[0]} rows, frontier needs {blk.num_src}")
        return gat_layer_forward_dev(net, l, blk, h_in, rows, R, R_dev, act, inj, stream, n_dst_dev, live, n_live,
                                     n_live_dev)
    dev = h_in.device
    d_in = net.dims[l]
    d_out = net.dims[l + 1]
    if h_in.shape[0] != blk.num_src:
        raise ValueError(f"h_in has {h_in.shape[0]} rows, frontier needs {blk.num_src}")
    kind = _kind_code(net.kind)
    K = 2 * d_in if kind == KIND_SAGE else d_in
    # GEMM operand [self | agg | 1] written by the aggregation directly as TS
    # (bf16 hi/lo core-matrix tiles, csrc/hg_ts.cuh)
    A = torch.empty(ts_bytes(R, K + 1), dtype=torch.uint8, device=dev)
    # SAGE: the forward hands the backward its per-row weights 1/cnt
    row_w = torch.empty(max(R, 1), dtype=torch.float32, device=dev) if kind == KIND_SAGE and l > 0 else None
    if isinstance(h_in, FeatureRows):     # layer 0 reading the feature rows in place
        _lib.call("hg_aggregate_fwd_rows", kind, _lib.ptr(R_dev), R, _lib.ptr(rows), _lib.ptr(blk.adj.start),
                  _lib.ptr(blk.adj.end), _lib.ptr(blk.adj.col_indices), _lib.ptr(blk.dst_deg),
                  _lib.ptr(blk.src_deg), _lib.ptr(h_in.rowp), h_in.dtype_code, d_in, _lib.ptr(A),
                  _lib.ptr(row_w), stream)
    else:
        _lib.call("hg_aggregate_fwd", kind, _lib.ptr(R_dev), R, _lib.ptr(rows), _lib.ptr(blk.adj.start),
                  _lib.ptr(blk.adj.end), _lib.ptr(blk.adj.col_indices), _lib.ptr(blk.dst_deg),
                  _lib.ptr(blk.src_deg), _lib.ptr(h_in), d_in, _lib.ptr(A), _lib.ptr(row_w), stream)
    if PT is None:
        PT = pack_forward_weights(net, l, stream)
    n_dst = blk.num_dst
    if h_out is None:
        h_out = torch.empty((n_dst, d_out), dtype=torch.float32, device=dev)
    # z = [A | 1] . P on tcgen05, ReLU + scatter to h_out[rows] in the epilogue
    _lib.call("hg_ts_linear_fwd", _lib.ptr(R_dev), R, _lib.ptr(A), K + 1, _lib.ptr(PT), d_out, _lib.ptr(rows),
              int(act), _lib.ptr(h_out), stream)
    if inj is not None and not injected_already:
        nd = n_dst_dev if n_dst_dev is not None else _dev_count(n_dst, dev)
        inject_rows_dev(inj, h_out, n_dst, nd, stream)
    return LayerTape(rows, R, R_dev, A, K, act, h_out, inj, row_w)


def ts_bytes(rows: int, cols: int) -> int:
    return int(_lib.query("hg_ts_bytes", int(rows), int(cols)))


def _rows_tensor(rows, n_dst, dev):
    if rows is None:
        return torch.arange(n_dst, dtype=torch.int32, device=dev), n_dst
    r = torch.as_tensor(np.asarray(rows if not isinstance(rows, torch.Tensor) else _np(rows), dtype=np.int64)
                        .astype(np.int32), device=dev)
    return r, int(r.shape[0])


def _injection_from_values(inj, n_dst, d_out, dev) -> Injection | None:
    if inj is None:
        return None
    loc = np.asarray(_np(inj[0]), dtype=np.int64)
    if len(loc) == 0:
        return None
    vals = inj[1]
    table = (vals if isinstance(vals, torch.Tensor) else torch.as_tensor(np.asarray(vals, np.float32)))
    table = table.to(dev, torch.float32).contiguous()
    flag = torch.zeros(n_dst, dtype=torch.uint8, device=dev)
    row = torch.full((n_dst,), -1, dtype=torch.int32, device=dev)
    li = torch.as_tensor(loc, device=dev)
    flag[li] = 1
    row[li] = torch.arange(len(loc), dtype=torch.int32, device=dev)
    return Injection(flag, row, table)


def forward_pass(network: Network, blocks, h_input, compute_rows=None, injected=None) -> BatchTape:
    """Run all blocks; rows absent from compute_rows[l] are dead unless
    injected[l] overwrites them. ReLU on every layer except the last.
    injected[l] may be (locals, values) like the reference, or an Injection."""
    if len(blocks) != network.num_layers:
        raise ValueError("block count does not match network depth")
    dev = network.flat.device
    stream = _lib.stream_ptr()
    h = h_input if isinstance(h_input, torch.Tensor) else torch.as_tensor(np.asarray(h_input, np.float32))
    h = pad_columns(h.to(dev, torch.float32), network.dims[0]).contiguous()
    ents, hs = [], []
    h_prev = h
    for l, blk in enumerate(blocks):
        rows, R = _rows_tensor(None if compute_rows is None else compute_rows[l], blk.num_dst, dev)
        inj = None if injected is None else injected[l]
        if inj is not None and not isinstance(inj, Injection):
            inj = _injection_from_values(inj, blk.num_dst, network.dims[l + 1], dev)
        t = layer_forward_dev(network, l, blk, h_prev, rows, R, _dev_count(R, dev), l < network.num_layers - 1,
                              inj, stream)
        ents.append(t)
        hs.append(t.h_out)
        h_prev = t.h_out
    return BatchTape(h, ents, hs)


# --------------------------------------------------------------- backward


@dataclass
class BlockCsc:
    vals: torch.Tensor
    seg_lo: torch.Tensor
    seg_hi: torch.Tensor


def build_csc(blk, keep: torch.Tensor, pos_of: torch.Tensor, n_dst_dev, stream, scratch=None) -> BlockCsc:
    dev = keep.device
    E = blk.num_edges_built
    n_src = blk.num_src
    keys = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    vals = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    seg_lo = torch.empty(max(n_src, 1), dtype=torch.int32, device=dev)
    seg_hi = torch.empty(max(n_src, 1), dtype=torch.int32, device=dev)
    sb = _lib.query("hg_csc_scratch_bytes", E, n_src)
    if scratch is None or scratch.numel() < sb:
        scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
    _lib.call("hg_build_csc", _lib.ptr(n_dst_dev), _lib.ptr(blk.blk_off), _lib.ptr(keep), _lib.ptr(pos_of),
              _lib.ptr(blk.adj.col_indices), E, n_src, _lib.ptr(keys), _lib.ptr(vals), _lib.ptr(seg_lo),
              _lib.ptr(seg_hi), _lib.ptr(scratch), sb, stream)
    return BlockCsc(vals, seg_lo, seg_hi)


def pack_forward_weights(net: Network, l: int, stream, out: torch.Tensor | None = None) -> torch.Tensor:
    """TS(P^T) of layer l (SAGE / GCN): the B operand of the forward GEMM."""
    d_in, d_out = net.dims[l], net.dims[l + 1]
    K = 2 * d_in if _kind_code(net.kind) == KIND_SAGE else d_in
    PT = out if out is not None else torch.empty(ts_bytes(d_out, K + 1), dtype=torch.uint8, device=net.flat.device)
    _lib.call("hg_ts_pack", _lib.ptr(net.slab(l)), d_out, 1, d_out, K + 1, d_out, _lib.ptr(PT), stream)
    return PT


def pack_dgrad_weights(net: Network, l: int, stream) -> torch.Tensor:
    """TS(P[:K]) of layer l: the B operand of the input-gradient GEMM
    (GAT: the W rows only)."""
    d_in, d_out = net.dims[l], net.dims[l + 1]
    K = 2 * d_in if _kind_code(net.kind) == KIND_SAGE and net.kind is not LayerKind.GAT else d_in
    W = torch.empty(ts_bytes(K, d_out), dtype=torch.uint8, device=net.flat.device)
    _lib.call("hg_ts_pack", _lib.ptr(net.slab(l)), d_out, 0, K, d_out, K, _lib.ptr(W), stream)
    return W


def layer_backward_dev(net: Network, l: int, blk, t: LayerTape, d_h: torch.Tensor, grads: Grads,
                       need_input: bool, keep, pos_of, live, n_live, stream, n_dst_dev=None, n_live_dev=None,
                       csc: BlockCsc | None = None, W_ts: torch.Tensor | None = None, wgrad_stream=None,
                       keepalive: list | None = None, need_rows=None, dz_prev=None, dz=None):
    """Writes dP into grads; returns (d_in [n_src, d_in] with rows valid on
    `live`, fp64 norms aligned with `live`) or (None, None).

    `dz_prev` = (tape, pos_of) of layer l-1: instead of d_in, the transposed
    aggregation writes that layer's ReLU-masked dz operand directly (its
    hg_gather_dz fused away) and returns it as `DzOperand` in place of d_in;
    `dz`: this layer's dz operand, already built that way by layer l+1.

    Engine options: `csc` / `W_ts` prebuilt off the critical path (they
    depend only on the pruned block / the weights), and `wgrad_stream`: the
    weight-gradient GEMM forks onto it (only SGD waits for it) while the
    input-gradient chain continues; buffers it reads are appended to
    `keepalive`, which the caller holds until the streams are joined;
    `need_rows` (uint8 per input row): only rows the previous layer computes
    get a gradient row, the others only their norm."""
    if net.kind is LayerKind.GAT:
        return gat_layer_backward_dev(net, l, blk, t, d_h, grads, need_input, keep, pos_of, stream, n_dst_dev,
                                      csc, wgrad_stream, keepalive)
    dev = t.h_out.device
    d_in_dim, d_out = net.dims[l], net.dims[l + 1]
    R, K = t.R, t.K
    if isinstance(d_h, DzOperand):
        dz = d_h
    if isinstance(dz, DzOperand):
        dz = dz.ts
    else:
        # dz (ReLU-masked output gradient of the compute rows) as a TS operand
        dz = torch.empty(ts_bytes(R, d_out), dtype=torch.uint8, device=dev)
        _lib.call("hg_gather_dz", _lib.ptr(t.R_dev), R, _lib.ptr(t.rows), _lib.ptr(d_h), _lib.ptr(t.h_out), d_out,
                  int(t.relu), _lib.ptr(dz), stream)
    dP = grads.slab(l)
    splits = _wgrad_splits(R, K + 1, d_out)

    def wgrad(sp):
        part = torch.empty(splits * (K + 1) * d_out, dtype=torch.float32, device=dev)
        _lib.call("hg_ts_linear_wgrad", _lib.ptr(t.R_dev), R, _lib.ptr(t.A), K + 1, _lib.ptr(dz), d_out,
                  _lib.ptr(dP), _lib.ptr(part), splits, sp)
        return part

    if wgrad_stream is not None:
        cur = torch.cuda.current_stream(dev)
        wgrad_stream.wait_stream(cur)
        with torch.cuda.stream(wgrad_stream):
            part = wgrad(_lib.stream_ptr(wgrad_stream))
        if keepalive is not None:
            keepalive.extend([dz, part])
    else:
        wgrad(stream)
    if not need_input:
        return None, None
    SG = torch.empty((R, K), dtype=torch.float32, device=dev)
    if W_ts is None:
        W_ts = pack_dgrad_weights(net, l, stream)
    _lib.call("hg_ts_linear_dgrad", _lib.ptr(t.R_dev), R, _lib.ptr(dz), d_out, _lib.ptr(W_ts), K, _lib.ptr(SG), stream)
    if n_dst_dev is None:
        n_dst_dev = _dev_count(blk.num_dst, dev)
    if n_live_dev is None:
        n_live_dev = _dev_count(n_live, dev)
    if csc is None:
        csc = build_csc(blk, keep, pos_of, n_dst_dev, stream)
    norms = torch.empty(max(n_live, 1), dtype=torch.float64, device=dev)
    if dz_prev is not None:
        tp, pos_prev = dz_prev
        d_in = None
        dzp = DzOperand(torch.empty(ts_bytes(tp.R, d_in_dim), dtype=torch.uint8, device=dev))
        dz_args = (_lib.ptr(dzp.ts), _lib.ptr(tp.R_dev), tp.R, _lib.ptr(pos_prev), _lib.ptr(tp.h_out), int(tp.relu))
    else:
        d_in = torch.empty((blk.num_src, d_in_dim), dtype=torch.float32, device=dev)
        dzp = None
        dz_args = (None, None, 0, None, None, 0)
    _lib.call("hg_transpose_agg", _kind_code(net.kind), _lib.ptr(n_live_dev), n_live, _lib.ptr(live),
              _lib.ptr(csc.seg_lo), _lib.ptr(csc.seg_hi), _lib.ptr(csc.vals), _lib.ptr(t.rows),
              _lib.ptr(blk.adj.start), _lib.ptr(blk.adj.end), _lib.ptr(blk.dst_deg), _lib.ptr(blk.src_deg),
              _lib.ptr(n_dst_dev), _lib.ptr(pos_of), _lib.ptr(SG), K, d_in_dim, _lib.ptr(d_in), _lib.ptr(norms),
              _lib.ptr(need_rows), _lib.ptr(t.row_w), *dz_args, stream)
    return (dzp if dzp is not None else d_in), norms[:n_live]


@dataclass
class DzOperand:
    """A layer's dz operand (TS bytes) built by the next layer's transposed
    aggregation (hg_transpose_agg with dz output)."""
    ts: torch.Tensor


def _keep_pos(rows: torch.Tensor, R: int, n_dst: int, dev):
    keep = torch.zeros(n_dst, dtype=torch.uint8, device=dev)
    pos = torch.full((n_dst,), -1, dtype=torch.int32, device=dev)
    if R:
        keep[rows.long()] = 1
        pos[rows.long()] = torch.arange(R, dtype=torch.int32, device=dev)
    return keep, pos


def backward(network: Network, blocks, tape: BatchTape, d_logits, need_input: bool = True):
    """Reverse pass (nn.py:300-320). Returns (grads, node_grads, input_grad);
    node_grads[l] = dL/dh_layers[l] for every dst row (device tensors, fully
    materialised here, zeros where the reference has zeros)."""
    dev = network.flat.device
    stream = _lib.stream_ptr()
    grads = network.new_grads()
    L = network.num_layers
    node_grads = [None] * L
    d_h = d_logits if isinstance(d_logits, torch.Tensor) else torch.as_tensor(np.asarray(d_logits, np.float32))
    d_h = d_h.to(dev, torch.float32).contiguous()
    for l in range(L - 1, -1, -1):
        node_grads[l] = d_h
        t = tape.entries[l]
        blk = blocks[l]
        want = need_input or l > 0
        keep, pos = _keep_pos(t.rows, t.R, blk.num_dst, dev)
        live = torch.arange(blk.num_src, dtype=torch.int32, device=dev)
        d_prev, _ = layer_backward_dev(network, l, blk, t, d_h, grads, want, keep, pos, live, blk.num_src, stream)
        d_h = d_prev
    if d_h is not None and network.in_dim is not None:
        d_h = d_h[:, :network.in_dim]
    return grads, node_grads, d_h


def cross_entropy(logits, labels):
    """Mean softmax cross entropy, fp64 (nn.py:326-343). Returns (loss, d_logits)."""
    lab = np.asarray(labels)
    if logits.shape[0] != len(lab):
        raise ValueError("labels do not match logit rows")
    if len(lab) and (lab.min() < 0 or lab.max() >= logits.shape[1]):
        raise ValueError("label id out of range")
    dev = logits.device if isinstance(logits, torch.Tensor) else torch.device("cuda")
    z = logits if isinstance(logits, torch.Tensor) else torch.as_tensor(np.asarray(logits, np.float32), device=dev)
    z = z.contiguous()
    B, C = z.shape
    labels_dev = torch.as_tensor(lab.astype(np.int32), device=dev)
    d, loss = cross_entropy_dev(z, labels_dev, B, C, _lib.stream_ptr())
    return float(loss.item()), d


def cross_entropy_dev(z, labels_dev, B, C, stream):
    dev = z.device
    d = torch.empty((B, C), dtype=torch.float32, device=dev)
    row = torch.empty(B, dtype=torch.float64, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.call("hg_cross_entropy", _lib.ptr(z), _lib.ptr(labels_dev), B, C, _lib.ptr(d), _lib.ptr(row),
              _lib.ptr(loss), stream)
    return d, loss


def node_grad_norms(node_grads) -> torch.Tensor:
    """Per-row Euclidean norms in fp64 (nn.py:346-349)."""
    g = node_grads if isinstance(node_grads, torch.Tensor) else torch.as_tensor(np.asarray(node_grads, np.float32))
    g = g.to(torch.device("cuda"), torch.float32).contiguous()
    n, d = g.shape
    out = torch.empty(n, dtype=torch.float64, device=g.device)
    if n:
        _lib.call("hg_row_norms", _lib.ptr(g), n, d, _lib.ptr(out), _lib.stream_ptr())
    return out


def sgd_step(network: Network, grads: Grads, eta: float) -> None:
    """p -= float32(eta) * g over the whole flat buffer (nn.py:355-360)."""
    _lib.call("hg_sgd", _lib.ptr(network.flat), _lib.ptr(grads.flat), network.flat.numel(),
              float(np.float32(eta)), _lib.stream_ptr())
