"""Helpers to read the committed golden fixtures (tests/golden/*.npz, *.json)."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SUB_FIELDS = ("dst", "src", "start", "end", "col", "dst_deg", "src_deg")


@functools.lru_cache(maxsize=None)
def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@functools.lru_cache(maxsize=None)
def load_json(name):
    with open(os.path.join(GOLDEN, name + ".json")) as fh:
        return json.load(fh)


def golden_sub(z, tag):
    """[{field: array}] innermost first, plus the seeds."""
    L = int(z[f"{tag}_L"])
    blocks = [{f: z[f"{tag}_b{i}_{f}"] for f in SUB_FIELDS} |
              {"prune_writes": int(z[f"{tag}_b{i}_prune_writes"])} for i in range(L)]
    return z[f"{tag}_seeds"], blocks


def assert_sub_equal(blocks_a, blocks_b, fields=SUB_FIELDS):
    assert len(blocks_a) == len(blocks_b)
    for i, (a, b) in enumerate(zip(blocks_a, blocks_b)):
        for f in fields:
            np.testing.assert_array_equal(np.asarray(a[f]), np.asarray(b[f]),
                                          err_msg=f"block {i} field {f}")


def oblock_dict(b):
    return {"dst": b.dst_nodes, "src": b.src_nodes, "start": b.start, "end": b.end,
            "col": b.col, "dst_deg": b.dst_deg, "src_deg": b.src_deg}


def sha(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
