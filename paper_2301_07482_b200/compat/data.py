"""histgnn.data's dataset format and container (data.py:30-151) for
reference-typed callers. The text files are parsed by the library's
multi-threaded parsers (ingest.read_int_lines / read_edge_list), so a
reference user's `ingest(directory)` is the same call with the same errors;
`paper_2301_07482_b200.ingest.ingest_device` is the device-layout variant
(CSR2 in HBM, features streamed to HBM / pinned host / owner shards).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .. import ingest as _ing
from ..ingest import DATASET_FILES, FEATURE_HEADER
from .graphs import CooGraph

__all__ = ["Dataset", "save_features", "load_features", "ingest", "save_dataset", "FEATURE_HEADER", "DATASET_FILES"]


@dataclass
class Dataset:
    """data.py:30-75: a graph, fp32 features, labels and disjoint splits."""

    graph: CooGraph
    features: np.ndarray
    labels: np.ndarray
    train_ids: np.ndarray
    val_ids: np.ndarray
    test_ids: np.ndarray

    def __post_init__(self):
        self.features = np.ascontiguousarray(self.features)
        if self.features.ndim != 2:
            raise ValueError("features must be a 2-d matrix")
        self.labels = np.asarray(self.labels, dtype=np.int64)
        n = self.graph.num_nodes
        if self.features.shape[0] != n:
            raise ValueError(f"{self.features.shape[0]} feature rows for {n} graph nodes")
        if self.labels.shape[0] != n:
            raise ValueError(f"{self.labels.shape[0]} labels for {n} graph nodes")
        if n and self.labels.min() < 0:
            raise ValueError("negative class id")
        splits = []
        for name in ("train_ids", "val_ids", "test_ids"):
            ids = np.asarray(getattr(self, name), dtype=np.int64)
            setattr(self, name, ids)
            if ids.size and (ids.min() < 0 or ids.max() >= n):
                raise ValueError(f"{name} contains node ids outside [0, {n})")
            splits.append(set(ids.tolist()))
        if splits[0] & splits[1] or splits[0] & splits[2] or splits[1] & splits[2]:
            raise ValueError("train/val/test splits overlap")

    @property
    def num_nodes(self) -> int:
        return self.graph.num_nodes

    @property
    def feature_dim(self) -> int:
        return self.features.shape[1]

    @property
    def num_classes(self) -> int:
        return int(self.labels.max()) + 1 if self.labels.size else 0


def save_features(path, features) -> None:
    mat = np.ascontiguousarray(features, dtype="<f4")
    if mat.ndim != 2:
        raise ValueError("features must be a 2-d matrix")
    with open(path, "wb") as fh:
        fh.write(FEATURE_HEADER.pack(*mat.shape))
        fh.write(mat.tobytes())


def load_features(path) -> np.ndarray:
    """data.py:91-106 (header checks shared with the device loader)."""
    rows, cols = _ing.feature_header(path)
    return np.fromfile(path, dtype="<f4", offset=FEATURE_HEADER.size).astype(np.float32).reshape(rows, cols)


def ingest(directory) -> Dataset:
    """data.py:132-151 with the native parsers."""
    paths = _ing.check_dataset_files(directory)
    labels = _ing.read_int_lines(paths["labels.txt"], "class id")
    n = labels.shape[0]
    features = load_features(paths["features.bin"])
    if features.shape[0] != n:
        raise ValueError(f"{paths['features.bin']}: {features.shape[0]} feature rows for {n} labeled nodes")
    src, dst, _ = _ing.read_edge_list(paths["edges.txt"], num_nodes=n)
    splits = [_ing.read_int_lines(paths[name], "node id", upper=n) for name in ("train.txt", "val.txt", "test.txt")]
    return Dataset(CooGraph(src.astype(np.int64), dst.astype(np.int64), n), features, labels, *splits)


def save_dataset(directory, ds) -> None:
    d = os.fspath(directory)
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "edges.txt"), "w", encoding="utf-8") as fh:
        fh.writelines(f"{s} {t}\n" for s, t in zip(ds.graph.src, ds.graph.dst))
    save_features(os.path.join(d, "features.bin"), ds.features)
    for name, ids in (("labels.txt", ds.labels), ("train.txt", ds.train_ids), ("val.txt", ds.val_ids),
                      ("test.txt", ds.test_ids)):
        with open(os.path.join(d, name), "w", encoding="utf-8") as fh:
            fh.writelines(f"{v}\n" for v in ids)
