"""GAT block layer — CPU restatement (TEST INFRASTRUCTURE ONLY).

The reference has no GAT (`LayerKind` is GCN / SAGE_MEAN only,
histgnn/nn.py:28-30; GAT is out of its scope), so parity for
this layer is UNPINNED by the reference: this file defines it, in the
reference's block/tape style (nn.py:131-177: a forward that returns a tape,
a hand-written reverse pass), and is itself checked against a dense
formulation and finite differences (tests/test_oracle_gat.py).

Layer (graph attention, Velickovic et al., multi-head, concatenated):
  z      = h_in @ W                                  [n_src, H*F]
  el[j]  = <z[j, h], a_src[h]>,  er[i] = <z[i, h], a_dst[h]>       per head h
  over the in-edges of a compute row i that survived pruning PLUS a self
  loop (i, i) (dst rows are a prefix of the block's sources, sampler.py:150):
  e_ij   = LeakyReLU_0.2(el[j] + er[i])
  a_ij   = softmax_j(e_ij)                           per head
  out[i] = sum_j a_ij z[j] + bias ; ReLU except on the last layer.
Heads: `heads` on hidden layers, 1 on the output layer.
Parameters per layer: weight [d_in, d_out], bias [d_out], att_src [d_out],
att_dst [d_out] (head h owns columns h*F:(h+1)*F). Init: Glorot-uniform
weight, then att_src, att_dst ~ U(+-sqrt(6/(F+1))) from the same generator,
zero bias (nn.py:73-85 order: weight first).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SLOPE = 0.2


@dataclass
class GATParams:
    weight: np.ndarray
    bias: np.ndarray
    att_src: np.ndarray
    att_dst: np.ndarray
    heads: int

    def arrays(self):
        return [self.weight, self.bias, self.att_src, self.att_dst]


@dataclass
class GATTape:
    rows: np.ndarray
    h_in: np.ndarray
    z: np.ndarray          # [n_src, H, F]
    src: np.ndarray        # edge sources (local src ids), per row edges then self
    seg: np.ndarray        # row index (0..R-1) of every edge
    alpha: np.ndarray      # [E', H]
    pre: np.ndarray        # [E', H] el + er before LeakyReLU
    relu: np.ndarray | None


def init_layer(rng, fi, fo, heads, dtype=np.float32) -> GATParams:
    lim = np.sqrt(6.0 / (fi + fo))
    w = rng.uniform(-lim, lim, size=(fi, fo)).astype(dtype)
    F = fo // heads
    la = np.sqrt(6.0 / (F + 1))
    a_s = rng.uniform(-la, la, size=fo).astype(dtype)
    a_d = rng.uniform(-la, la, size=fo).astype(dtype)
    return GATParams(w, np.zeros(fo, dtype), a_s, a_d, heads)


def _edges(blk, rows):
    """Per compute row: its surviving in-edges (CSR2 order) then the self loop."""
    lo = np.asarray(blk.start, np.int64)[rows]
    cnt = np.asarray(blk.end, np.int64)[rows] - lo
    col = np.asarray(blk.col, np.int64)
    R = len(rows)
    cnt1 = cnt + 1
    ptr = np.concatenate([[0], np.cumsum(cnt1)])
    E = int(ptr[-1])
    src = np.empty(E, np.int64)
    seg = np.repeat(np.arange(R), cnt1)
    pos = np.arange(E) - ptr[seg]
    body = pos < cnt[seg]
    src[body] = col[lo[seg[body]] + pos[body]]
    src[~body] = rows[seg[~body]]
    return src, seg, ptr


def layer_forward(p: GATParams, blk, h_in, rows, act):
    """Returns (out [R, d_out] for the compute rows, tape)."""
    dt = h_in.dtype
    rows = np.asarray(rows, np.int64)
    H = p.heads
    fo = p.weight.shape[1]
    F = fo // H
    z = (h_in @ p.weight).reshape(-1, H, F)
    el = np.einsum("nhf,hf->nh", z, p.att_src.reshape(H, F))
    er = np.einsum("nhf,hf->nh", z, p.att_dst.reshape(H, F))
    src, seg, ptr = _edges(blk, rows)
    pre = el[src] + er[rows][seg]
    e = np.where(pre > 0, pre, dt.type(SLOPE) * pre)
    R = len(rows)
    m = np.full((R, H), -np.inf, dt)
    np.maximum.at(m, seg, e)
    w = np.exp(e - m[seg])
    s = np.zeros((R, H), dt)
    np.add.at(s, seg, w)
    alpha = (w / s[seg]).astype(dt)
    out = np.zeros((R, H, F), dt)
    np.add.at(out, seg, alpha[:, :, None] * z[src])
    out = out.reshape(R, fo) + p.bias
    relu = None
    if act:
        relu = out > 0
        out = np.where(relu, out, dt.type(0))
    return out.astype(dt), GATTape(rows, h_in, z, src, seg, alpha, pre, relu)


def layer_backward(p: GATParams, t: GATTape, d_out, need_input=True):
    """d_out: [R, d_out] gradient of the compute rows' outputs. Returns
    (GATParams of gradients, d_in [n_src, d_in] or None)."""
    dt = d_out.dtype
    H = p.heads
    fo = p.weight.shape[1]
    F = fo // H
    g = d_out if t.relu is None else np.where(t.relu, d_out, dt.type(0))
    db = g.sum(axis=0)
    gh = g.reshape(-1, H, F)
    R = len(t.rows)
    zs = t.z[t.src]                                     # [E', H, F]
    d_alpha = np.einsum("ehf,ehf->eh", gh[t.seg], zs)    # [E', H]
    c = np.zeros((R, H), dt)
    np.add.at(c, t.seg, t.alpha * d_alpha)
    de = t.alpha * (d_alpha - c[t.seg])
    ds = np.where(t.pre > 0, de, dt.type(SLOPE) * de)
    dz = np.zeros_like(t.z)
    np.add.at(dz, t.src, t.alpha[:, :, None] * gh[t.seg])
    d_el = np.zeros((t.z.shape[0], H), dt)
    np.add.at(d_el, t.src, ds)
    d_er = np.zeros((R, H), dt)
    np.add.at(d_er, t.seg, ds)
    a_s = p.att_src.reshape(H, F)
    a_d = p.att_dst.reshape(H, F)
    dz += d_el[:, :, None] * a_s
    dz[t.rows] += d_er[:, :, None] * a_d
    d_as = np.einsum("nh,nhf->hf", d_el, t.z).reshape(fo)
    d_ad = np.einsum("rh,rhf->hf", d_er, t.z[t.rows]).reshape(fo)
    dz2 = dz.reshape(-1, fo)
    gw = t.h_in.T @ dz2
    d_in = dz2 @ p.weight.T if need_input else None
    return GATParams(gw.astype(dt), db.astype(dt), d_as.astype(dt), d_ad.astype(dt), H), (
        None if d_in is None else d_in.astype(dt))


def dense_forward(p: GATParams, adj_rows, h_in, rows, act):
    """Dense restatement for checking layer_forward: adj_rows[r] = list of
    source ids of compute row r (self loop excluded; it is added here)."""
    H = p.heads
    fo = p.weight.shape[1]
    F = fo // H
    z = (h_in.astype(np.float64) @ p.weight.astype(np.float64)).reshape(-1, H, F)
    out = np.zeros((len(rows), fo))
    for r, i in enumerate(rows):
        nb = list(adj_rows[r]) + [i]
        for h in range(H):
            sc = np.array([z[j, h] @ p.att_src[h * F:(h + 1) * F] + z[i, h] @ p.att_dst[h * F:(h + 1) * F]
                           for j in nb])
            sc = np.where(sc > 0, sc, SLOPE * sc)
            a = np.exp(sc - sc.max())
            a /= a.sum()
            out[r, h * F:(h + 1) * F] = sum(a[k] * z[j, h] for k, j in enumerate(nb))
    out += p.bias
    return np.maximum(out, 0) if act else out
