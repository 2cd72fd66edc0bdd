"""Dataset text formats (TEST INFRASTRUCTURE ONLY): line-by-line Python
restatements of histgnn/data.py:109-129 (_read_int_lines) and
graphs.py:186-218 (read_edge_list), the checker for the native parsers
(csrc/hg_ingest.cu via paper_2301_07482_b200/ingest.py)."""

from __future__ import annotations

import numpy as np


def read_int_lines(path, what, upper=None):
    vals = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line:
                continue
            try:
                v = int(line)
            except ValueError:
                raise ValueError(f"{path}:{lineno}: expected a {what}, got {line!r}") from None
            if v < 0:
                raise ValueError(f"{path}:{lineno}: negative {what} {v}")
            if upper is not None and v >= upper:
                raise ValueError(f"{path}:{lineno}: {what} {v} out of range [0, {upper})")
            vals.append(v)
    return np.asarray(vals, dtype=np.int64)


def read_edge_list(path, num_nodes=None):
    src, dst = [], []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            parts = raw.split("#", 1)[0].split()
            if not parts:
                continue
            if len(parts) != 2:
                raise ValueError(f"{path}:{lineno}: expected 'src dst', got {raw.strip()!r}")
            try:
                s, d = int(parts[0]), int(parts[1])
            except ValueError:
                raise ValueError(f"{path}:{lineno}: non-integer node id in {raw.strip()!r}") from None
            if s < 0 or d < 0:
                raise ValueError(f"{path}:{lineno}: negative node id")
            src.append(s)
            dst.append(d)
    src, dst = np.asarray(src, np.int64), np.asarray(dst, np.int64)
    if num_nodes is None:
        num_nodes = int(max(src.max(initial=-1), dst.max(initial=-1))) + 1
    for what, a in (("src", src), ("dst", dst)):
        if len(a) and a.max() >= num_nodes:
            raise ValueError(f"{path}: {what} id out of range: saw {int(a.max())} for a graph with {num_nodes} nodes")
    return src, dst, num_nodes
