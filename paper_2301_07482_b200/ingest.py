"""Dataset ingest into the device layout (reference:
histgnn/data.py:81-151 `save_features` / `load_features` / `ingest`,
graphs.py:186-226 `read_edge_list`).

The directory format is the reference's: `edges.txt` ("src dst" per line,
'#' comments), `features.bin` (u64 rows, u64 cols, little-endian, then fp32
row-major), `labels.txt`, `train.txt`, `val.txt`, `test.txt` (one integer per
line). The text files are parsed by the library's multi-threaded parsers
(hg_parse_edge_list / hg_parse_int_lines) straight into int32 / int64
arrays; errors carry the reference's wording (file:line). The graph goes to
the device CSR2 build; the feature table is streamed from the file in row
chunks through a pinned staging buffer into HBM (optionally fp16), into
pinned host memory for UVA reads, or -- for an owner-sharded table -- only
this rank's row range is read.
"""

from __future__ import annotations

import ctypes
import os
import struct
import numpy as np
import torch

from . import _lib

FEATURE_HEADER = struct.Struct("<QQ")
DATASET_FILES = ("edges.txt", "features.bin", "labels.txt", "train.txt", "val.txt", "test.txt")
_NOT_INT, _NEGATIVE, _RANGE, _FIELDS = 1, 2, 3, 4


def _line(path, lineno: int) -> str:
    with open(path, "rb") as fh:
        for i, raw in enumerate(fh, start=1):
            if i == lineno:
                return raw.decode("utf-8", errors="replace")
    return ""


def read_int_lines(path, what: str, upper: int | None = None, nthreads: int = 0) -> np.ndarray:
    """data.py:109-129: one integer per non-blank line; ValueError names the
    file and the 1-based line of the first bad entry."""
    path = os.fspath(path)
    cnt, err, eline, evalue = ctypes.c_longlong(), ctypes.c_int(), ctypes.c_longlong(), ctypes.c_longlong()
    up = -1 if upper is None else int(upper)
    args = (path.encode(), up)
    _lib.call("hg_parse_int_lines", *args, None, ctypes.byref(cnt), ctypes.byref(err), ctypes.byref(eline),
              ctypes.byref(evalue), nthreads)
    if err.value:
        line = _line(path, eline.value).strip()
        if err.value == _NOT_INT:
            raise ValueError(f"{path}:{eline.value}: expected a {what}, got {line!r}")
        if err.value == _NEGATIVE:
            raise ValueError(f"{path}:{eline.value}: negative {what} {evalue.value}")
        raise ValueError(f"{path}:{eline.value}: {what} {evalue.value} out of range [0, {upper})")
    out = np.empty(cnt.value, dtype=np.int64)
    if cnt.value:
        _lib.call("hg_parse_int_lines", *args, out.ctypes.data, ctypes.byref(cnt), ctypes.byref(err),
                  ctypes.byref(eline), ctypes.byref(evalue), nthreads)
    return out


def read_edge_list(path, num_nodes: int | None = None, nthreads: int = 0):
    """graphs.py:186-218 + CooGraph validation (graphs.py:48-57): returns
    (src, dst, num_nodes) with int32 ids."""
    path = os.fspath(path)
    cnt, ms, md = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_longlong()
    err, eline = ctypes.c_int(), ctypes.c_longlong()
    _lib.call("hg_parse_edge_list", path.encode(), None, None, ctypes.byref(cnt), ctypes.byref(ms), ctypes.byref(md),
              ctypes.byref(err), ctypes.byref(eline), nthreads)
    if err.value:
        raw = _line(path, eline.value).strip()
        if err.value == _FIELDS:
            raise ValueError(f"{path}:{eline.value}: expected 'src dst', got {raw!r}")
        if err.value == _NOT_INT:
            raise ValueError(f"{path}:{eline.value}: non-integer node id in {raw!r}")
        if err.value == _NEGATIVE:
            raise ValueError(f"{path}:{eline.value}: negative node id")
        raise ValueError(f"{path}:{eline.value}: node id exceeds the device's int32 id range")
    if num_nodes is None:
        num_nodes = int(max(ms.value, md.value)) + 1
    for what, hi in (("src", ms.value), ("dst", md.value)):
        if cnt.value and hi >= num_nodes:
            raise ValueError(f"{path}: {what} id out of range: saw {hi} for a graph with {num_nodes} nodes")
    src = np.empty(cnt.value, dtype=np.int32)
    dst = np.empty(cnt.value, dtype=np.int32)
    if cnt.value:
        _lib.call("hg_parse_edge_list", path.encode(), src.ctypes.data, dst.ctypes.data, ctypes.byref(cnt),
                  ctypes.byref(ms), ctypes.byref(md), ctypes.byref(err), ctypes.byref(eline), nthreads)
    return src, dst, int(num_nodes)


def feature_header(path):
    """(rows, cols) of a features.bin, with the reference's checks (data.py:91-106)."""
    path = os.fspath(path)
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        header = fh.read(FEATURE_HEADER.size)
    if len(header) < FEATURE_HEADER.size:
        raise ValueError(f"{path}: truncated header ({len(header)} bytes, need {FEATURE_HEADER.size})")
    rows, cols = FEATURE_HEADER.unpack(header)
    payload = size - FEATURE_HEADER.size
    if payload != rows * cols * 4:
        raise ValueError(f"{path}: header promises {rows}x{cols} floats ({rows * cols * 4} bytes), payload holds "
                         f"{payload} bytes")
    return int(rows), int(cols)


def load_feature_rows(path, lo: int = 0, hi: int | None = None, device=None, placement: str = "hbm",
                      dtype=torch.float32, chunk_bytes: int = 64 << 20) -> torch.Tensor:
    """Rows [lo, hi) of a features.bin as a [hi-lo, cols] tensor: in HBM
    (streamed through a reused pinned buffer, converted to `dtype` on the
    device) or in pinned host memory (placement "host", fp32, read by the
    kernels over UVA). Only the requested byte range is read."""
    rows, cols = feature_header(path)
    hi = rows if hi is None else int(hi)
    if not 0 <= lo <= hi <= rows:
        raise ValueError(f"row range [{lo}, {hi}) outside the {rows} rows of {path}")
    n = hi - lo
    base = FEATURE_HEADER.size + lo * cols * 4
    if placement == "host":
        if dtype != torch.float32:
            raise ValueError("host placement keeps the file's fp32 rows")
        out = torch.empty((n, cols), dtype=torch.float32, pin_memory=True)
        with open(path, "rb") as fh:
            fh.seek(base)
            fh.readinto(memoryview(out.numpy()).cast("B"))
        return out
    if placement != "hbm":
        raise ValueError("placement must be 'hbm' or 'host'")
    _lib.require_cuda()
    dev = torch.device(device or "cuda")
    out = torch.empty((n, cols), dtype=dtype, device=dev)
    step = max(1, chunk_bytes // max(1, cols * 4))
    bufs = [torch.empty((min(step, max(n, 1)), cols), dtype=torch.float32, pin_memory=True) for _ in range(2)]
    evs = [None, None]
    stream = torch.cuda.current_stream(dev)
    with open(path, "rb") as fh:
        for k, a in enumerate(range(0, n, step)):
            b = min(n, a + step)
            buf, i = bufs[k & 1], k & 1
            if evs[i] is not None:
                evs[i].synchronize()                 # the copy that last used this buffer is done
            fh.seek(base + a * cols * 4)
            fh.readinto(memoryview(buf[: b - a].numpy()).cast("B"))
            tmp = buf[: b - a].to(dev, non_blocking=True)
            out[a:b].copy_(tmp)                      # fp32 -> dtype on the device
            evs[i] = torch.cuda.Event()
            evs[i].record(stream)
    return out


def check_dataset_files(directory) -> dict:
    d = os.fspath(directory)
    paths = {name: os.path.join(d, name) for name in DATASET_FILES}
    for name, path in paths.items():
        if not os.path.exists(path):
            raise FileNotFoundError(f"{d}: missing {name}")
    return paths


def ingest_device(directory, device=None, placement: str = "hbm", dtype=torch.float32, rank: int | None = None,
                  world: int | None = None, group=None) -> DeviceDataset:
    """data.py:132-151 into the device layout. placement: "hbm" (whole table
    on this GPU), "host" (pinned, UVA), or "sharded" (this rank's owner range
    of comms.py:329-337 only, peers mapped over CUDA IPC; a collective over
    the torch.distributed group)."""
    from .data import DeviceDataset, csr2_from_edges_device
    paths = check_dataset_files(directory)
    labels = read_int_lines(paths["labels.txt"], "class id")
    n = len(labels)
    rows, _cols = feature_header(paths["features.bin"])
    if rows != n:
        raise ValueError(f"{paths['features.bin']}: {rows} feature rows for {n} labeled nodes")
    src, dst, _ = read_edge_list(paths["edges.txt"], num_nodes=n)
    splits = [read_int_lines(paths[name], "node id", upper=n) for name in ("train.txt", "val.txt", "test.txt")]
    dev = torch.device(device or "cuda")
    graph = csr2_from_edges_device(src, dst, n, dev)
    del src, dst
    if placement == "sharded":
        import torch.distributed as dist
        from .distributed import owner_ranges
        from .sharding import ShardedFeatures
        rank = dist.get_rank(group) if rank is None else rank
        world = dist.get_world_size(group) if world is None else world
        b = owner_ranges(n, world)
        local = load_feature_rows(paths["features.bin"], int(b[rank]), int(b[rank + 1]), dev, "hbm", dtype)
        feats = ShardedFeatures.from_process_group(local, n, rank, world, dev, group=group)
    else:
        feats = load_feature_rows(paths["features.bin"], 0, n, dev, placement, dtype)
    return DeviceDataset(graph, feats, labels, *splits, num_classes=int(labels.max()) + 1 if n else 0)
