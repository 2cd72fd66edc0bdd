"""Synthetic benchmark datasets built natively.

`synth_edges` runs the reference's preferential-attachment process
(histgnn/data.py:243-270) in C++ (hg_synth_power_law), bit-identical to the
reference for the same numpy Generator (the PCG64 stream and numpy's bounded
integer draw are reproduced exactly), in seconds instead of the reference's
minutes-to-hours. `synth_power_law_host` completes the reference Dataset
(features, labels, 60/20/20 split from the continued stream);
`synth_power_law_native` draws the features on the GPU instead (papers100M
shape, where host N(0,1) draws would take minutes).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .graphs import Csr2Graph


@dataclass
class DeviceDataset:
    graph: Csr2Graph
    features: torch.Tensor        # [N, d] device (fp32 / fp16)
    labels: np.ndarray            # int64[N] host
    train_ids: np.ndarray
    val_ids: np.ndarray
    test_ids: np.ndarray
    num_classes: int
    src: np.ndarray | None = None  # host edge list (int32), kept for CPU baselines
    dst: np.ndarray | None = None

    @property
    def num_nodes(self) -> int:
        return self.graph.num_nodes


def _pcg_words(bg) -> np.ndarray:
    st = bg.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"])],
                    dtype=np.uint64)


def synth_edges(n: int, m: int, rng: np.random.Generator | int = 0):
    """Edges of histgnn.data.synth_power_law(n, rng, m) (data.py:243-266),
    bit-identical, as int32 (src, dst). `rng` (a numpy Generator over PCG64,
    or an int seed for default_rng) is advanced exactly as the reference's
    pool draws advance it, so the caller's next draws (features, labels,
    split) continue the reference's stream."""
    if not isinstance(rng, np.random.Generator):
        rng = np.random.default_rng(rng)
    if not isinstance(rng.bit_generator, np.random.PCG64):
        raise ValueError("synth_edges reproduces numpy's PCG64 stream only")
    if m < 1 or n < m + 1:
        raise ValueError(f"need n >= m + 1 >= 2, got n={n} m={m}")
    fwd = m * (n - m)
    if n >= 2 ** 31:
        raise ValueError("node ids must fit in int32")
    src = np.empty(2 * fwd, dtype=np.int32)
    dst = np.empty(2 * fwd, dtype=np.int32)
    words = _pcg_words(rng.bit_generator)
    got = _lib.load().hg_synth_power_law(n, m, words.ctypes.data_as(_lib.P), src.ctypes.data_as(_lib.P),
                                         dst.ctypes.data_as(_lib.P))
    if got != 2 * fwd:
        raise ValueError(f"need n >= m + 1 >= 2, got n={n} m={m}")
    st = rng.bit_generator.state
    w = [int(x) for x in words]
    st["state"]["state"] = (w[0] << 64) | w[1]
    st["state"]["inc"] = (w[2] << 64) | w[3]
    st["has_uint32"], st["uinteger"] = w[4], w[5]
    rng.bit_generator.state = st
    return src, dst


def synth_power_law_host(n: int, rng: np.random.Generator, m: int = 3, feature_dim: int = 32, classes: int = 8):
    """histgnn.data.synth_power_law (data.py:243-270) with the edge process in
    C++: returns (src, dst, features fp32, labels int64, train, val, test),
    identical to the reference's Dataset fields for the same Generator."""
    src, dst = synth_edges(n, m, rng)
    feats = rng.standard_normal((n, feature_dim)).astype(np.float32)
    labels = rng.integers(0, classes, size=n)
    p = rng.permutation(n)                       # data.py:173-182 (_split_ids)
    a, b = int(0.6 * n), int(0.2 * n)
    return src, dst, feats, np.asarray(labels, np.int64), np.sort(p[:a]), np.sort(p[a:a + b]), np.sort(p[a + b:])


def csr2_from_edges_device(src: np.ndarray, dst: np.ndarray, n: int, device="cuda") -> Csr2Graph:
    """In-neighbour CSR2 with stable in-row order (graphs.py:161-172), built on
    the GPU by hg_build_csr2 (counts, scan, placement, per-row sort of the
    edge indices; no library sort)."""
    _lib.require_cuda()
    dev = torch.device(device)
    s = torch.as_tensor(np.ascontiguousarray(src, dtype=np.int32) if isinstance(src, np.ndarray) else src,
                        device=dev).to(torch.int32).contiguous()
    d = torch.as_tensor(np.ascontiguousarray(dst, dtype=np.int32) if isinstance(dst, np.ndarray) else dst,
                        device=dev).to(torch.int32).contiguous()
    E = int(s.numel())
    start = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    end = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    col = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    sb = _lib.query("hg_build_csr2_scratch_bytes", E, max(n, 1))
    scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
    _lib.call("hg_build_csr2", _lib.ptr(s), _lib.ptr(d), E, max(n, 1), _lib.ptr(start), _lib.ptr(end),
              _lib.ptr(col), _lib.ptr(scratch), sb, _lib.stream_ptr())
    del scratch, s, d
    return Csr2Graph(start[:n], end[:n], col[:E], n)


def synth_power_law_native(n: int, m: int, feature_dim: int, classes: int, seed: int = 0,
                           feature_dtype=torch.float32, device="cuda", keep_edges=False) -> DeviceDataset:
    _lib.require_cuda()
    rng = np.random.default_rng(seed)
    src, dst = synth_edges(n, m, rng)
    g = csr2_from_edges_device(src, dst, n, device)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    feats = torch.randn((n, feature_dim), generator=gen, device=device, dtype=torch.float32).to(feature_dtype)
    labels = rng.integers(0, classes, size=n)
    perm = rng.permutation(n)
    a, b = int(0.6 * n), int(0.2 * n)
    return DeviceDataset(g, feats, labels, np.sort(perm[:a]), np.sort(perm[a:a + b]), np.sort(perm[a + b:]),
                         classes, src if keep_edges else None, dst if keep_edges else None)
