"""Helpers shared by the -m gpu parity tests."""

from __future__ import annotations

import numpy as np
import torch


def dev_sub_from_golden(seeds, blocks, device="cuda"):
    """Build a device LayeredSubgraph from golden numpy blocks (innermost first)."""
    from paper_2301_07482_b200.graphs import Csr2Graph
    from paper_2301_07482_b200.sampler import LayerBlock, LayeredSubgraph

    out = []
    for b in blocks:
        t = lambda a: torch.as_tensor(np.asarray(a, np.int64).astype(np.int32), device=device)  # noqa: E731
        src = t(b["src"])
        n_dst = len(b["dst"])
        col = t(b["col"])
        blk_off = t(np.concatenate([b["start"], [len(b["col"])]]))
        adj = Csr2Graph(t(b["start"]), t(b["end"]), col, n_dst)
        out.append(LayerBlock(src[:n_dst], src, adj, t(b["dst_deg"]), t(b["src_deg"]), blk_off))
    return LayeredSubgraph(np.asarray(seeds, np.int64), out)


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.linalg.norm(b), 1e-30)
    return float(np.linalg.norm(a - b) / den)


def assert_close(a, b, tol=1e-3, what=""):
    e = rel_err(a, b)
    assert e <= tol, f"{what}: relative error {e:.3e} > {tol}"
