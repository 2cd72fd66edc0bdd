"""Synthetic benchmark datasets built natively.

`synth_power_law_native` runs the reference's preferential-attachment process
(histgnn/data.py:243-270) in C++ (hg_synth_power_law) and builds the CSR2 and
N(0,1) features on the GPU, so the products / papers shapes are generated in
seconds instead of minutes-to-hours. Labels are uniform classes and the split
is 60/20/20 like data.py:173-182. Not bit-identical to numpy's stream — parity
fixtures use the reference generator (oracle/datagen.py).
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


def synth_edges(n: int, m: int, seed: int = 0):
    fwd = m * (n - m)
    src = np.empty(2 * fwd, dtype=np.int32)
    dst = np.empty(2 * fwd, dtype=np.int32)
    got = _lib.load().hg_synth_power_law(n, m, seed, src.ctypes.data_as(_lib.P), dst.ctypes.data_as(_lib.P))
    if got != 2 * fwd:
        raise ValueError(f"need n >= m + 1 >= 2, got n={n} m={m}")
    return src, dst


def csr2_from_edges_device(src: np.ndarray, dst: np.ndarray, n: int, device="cuda") -> Csr2Graph:
    """In-neighbour CSR2 with stable in-row order (graphs.py:161-172), on the GPU."""
    d = torch.as_tensor(dst, device=device).long()
    s = torch.as_tensor(src, device=device)
    counts = torch.bincount(d, minlength=n)
    ptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=ptr[1:])
    order = torch.sort(d, stable=True).indices
    col = s[order].to(torch.int32).contiguous()
    del d, s, order
    return Csr2Graph(ptr[:-1].clone(), ptr[1:].clone(), col, n)


def synth_power_law_native(n: int, m: int, feature_dim: int, classes: int, seed: int = 0,
                           feature_dtype=torch.float32, device="cuda", keep_edges=False) -> DeviceDataset:
    _lib.require_cuda()
    src, dst = synth_edges(n, m, seed)
    g = csr2_from_edges_device(src, dst, n, device)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    feats = torch.randn((n, feature_dim), generator=gen, device=device, dtype=torch.float32).to(feature_dtype)
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, classes, size=n)
    perm = rng.permutation(n)
    a, b = int(0.6 * n), int(0.2 * n)
    return DeviceDataset(g, feats, labels, np.sort(perm[:a]), np.sort(perm[a:a + b]), np.sort(perm[a + b:]),
                         classes, src if keep_edges else None, dst if keep_edges else None)
