"""C-ABI boundary checks that need no GPU: the library loads and exports every
symbol include/hgb200.h declares, and the ctypes table matches the header."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hgb200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    syms = header_symbols()
    for s in ("hg_sample_layer", "hg_prune_block", "hg_cache_lookup", "hg_load_features", "hg_aggregate_fwd",
              "hg_transpose_agg", "hg_cache_rank", "hg_cache_write"):
        assert s in syms


def test_library_exports_every_header_symbol():
    from paper_2301_07482_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libhgb200.so not built (run __graft_entry__.build())")
    lib = _lib.load()
    for s in header_symbols():
        assert hasattr(lib, s), f"{s} missing from libhgb200.so"
    assert lib.hg_version() >= 10000


def test_ctypes_table_covers_header():
    from paper_2301_07482_b200 import _lib
    assert set(header_symbols()) == set(_lib.SIGNATURES), set(header_symbols()) ^ set(_lib.SIGNATURES)


def test_ctypes_arity_matches_header():
    from paper_2301_07482_b200 import _lib
    text = open(HEADER).read()
    for name, (_, args) in _lib.SIGNATURES.items():
        m = re.search(r"\b" + name + r"\s*\(([^)]*)\)", text, re.S)
        assert m, name
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), (name, len(params), len(args))


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2301_07482_b200 as hg
    from paper_2301_07482_b200._lib import HgError
    with pytest.raises(HgError):
        hg.build_csr2(hg.CooGraph([0, 1], [1, 2], 3))


def test_integration_stub_binds_the_header_signature():
    """The binding stub INTEGRATION.md shows a maintainer is executable and
    its argtypes equal the package's table (and so the header's arity)."""
    import ctypes
    import types
    from paper_2301_07482_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    stub = [b for b in blocks if "hg_sample_layer.argtypes" in b]
    assert len(stub) == 1

    class FakeLib:
        def __init__(self, *_):
            self.fns = {}

        def __getattr__(self, name):
            return self.__dict__["fns"].setdefault(name, types.SimpleNamespace())

    ns = {}
    real = ctypes.CDLL
    ctypes.CDLL = FakeLib
    try:
        exec(compile(stub[0], "INTEGRATION.md", "exec"), ns)
    finally:
        ctypes.CDLL = real
    for name in ("hg_sample_layer", "hg_sample_layer_scratch_bytes"):
        got = getattr(ns["_lib"], name)
        res, args = _lib.SIGNATURES[name]
        assert got.argtypes == args, name
        assert got.restype == res, name
