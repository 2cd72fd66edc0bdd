"""ctypes binding of the C-ABI library `libhgb200.so` (include/hgb200.h).

The product path has no CPU fallback: if the library is missing, or no CUDA
device is visible, every entry point raises instead of computing something
else. `load()` returns the CDLL with argtypes declared from the header.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhgb200.so")
if os.environ.get("HG_LIB_PATH"):          # A/B variants (tools/build_variant.sh); diagnostics only
    LIB_PATH = os.path.abspath(os.environ["HG_LIB_PATH"])

P = ctypes.c_void_p
I32 = ctypes.c_int
U32 = ctypes.c_uint
I64 = ctypes.c_longlong
U64 = ctypes.c_ulonglong
F64 = ctypes.c_double
F32 = ctypes.c_float
S = ctypes.c_char_p

# name -> (restype, argtypes); mirrors include/hgb200.h
SIGNATURES = {
    "hg_version": (I32, []),
    "hg_last_error": (ctypes.c_char_p, []),
    "hg_device_sync": (I32, []),
    "hg_kernel_launches": (I64, []),
    "hg_count_graph_replay": (None, [I64]),
    "hg_graph_instantiate": (I32, [P, P]),
    "hg_graph_launch": (I32, [P, P]),
    "hg_graph_exec_destroy": (I32, [P]),
    "hg_mark_time": (I32, [P, P]),
    "hg_metrics_row": (I32, [P, P, I32, P, P, P, P, I32, I32, P, P]),
    "hg_set_kernel_timers": (I32, [P]),
    "hg_sample_layer_scratch_bytes": (I64, [I64, I64]),
    "hg_sample_layer": (I32, [P, P, P, I64, P, P, I64, I32, P, P, P, P, P, P, P, P, P, P, P, P, I64, P]),
    "hg_prune_scratch_bytes": (I64, [I64]),
    "hg_prune_block": (I32, [P, I64, P, I64, P, P, P, P, P, P, P, P, P, P, P, P, P, I64, P]),
    "hg_cache_lookup": (I32, [P, I64, P, P, I64, P, P, P, P, F64, P, P, P, P]),
    "hg_load_features_scratch_bytes": (I64, [I64]),
    "hg_load_features": (I32, [P, I64, P, P, P, P, P, I32, I32, P, P, P, I64, P]),
    "hg_load_features_sharded": (I32, [P, I64, P, P, P, P, P, P, I32, I32, I32, I32, P, P, P, P]),
    "hg_device_alloc": (I32, [I64, P]),
    "hg_device_free": (I32, [P]),
    "hg_ipc_handle_bytes": (I64, []),
    "hg_ipc_export": (I32, [P, P]),
    "hg_ipc_open": (I32, [P, P]),
    "hg_ipc_close": (I32, [P]),
    "hg_gat_scores": (I32, [P, I64, P, P, I32, I32, P, P, P, P, P]),
    "hg_gat_aggregate": (I32, [P, I64, P, P, P, P, P, P, P, I32, I32, P, I32, P, P, P, P]),
    "hg_gat_bwd_dst": (I32, [P, I64, P, P, P, P, P, P, P, P, P, P, P, I32, I32, I32, P, P, P, P, P]),
    "hg_gat_bwd_src": (I32, [P, I64, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, I32, I32, P, P, P, P]),
    "hg_gat_param_scratch_bytes": (I64, [I32]),
    "hg_gat_param_grads": (I32, [I64, I64, I32, P, P, P, P, P, P]),
    "hg_gat_scatter_norms": (I32, [P, I64, P, P, I32, P, P, P]),
    "hg_aggregate_fwd": (I32, [I32, P, I64, P, P, P, P, P, P, P, I32, P, P, P]),
    "hg_aggregate_fwd_rows": (I32, [I32, P, I64, P, P, P, P, P, P, P, I32, I32, P, P, P]),
    "hg_resolve_feature_rows": (I32, [P, I64, P, P, P, P, P, P, P, I32, I32, I32, I32, P, P, P, P]),
    "hg_scatter_rows": (I32, [P, I64, P, P, I32, I32, P, P]),
    "hg_inject_rows": (I32, [P, I64, P, P, P, I32, P, P]),
    "hg_resolve_hit_rows": (I32, [P, I64, P, P, P, P, I32, P, P, P]),
    "hg_cross_entropy": (I32, [P, P, I32, I32, P, P, P, P]),
    "hg_gather_dz": (I32, [P, I64, P, P, P, I32, I32, P, P]),
    "hg_gather_rows_ts": (I32, [P, I64, P, P, I32, I32, P, P]),
    "hg_csc_scratch_bytes": (I64, [I64, I64]),
    "hg_build_csc": (I32, [P, P, P, P, P, I64, I64, P, P, P, P, P, I64, P]),
    "hg_transpose_agg": (I32, [I32, P, I64, P, P, P, P, P, P, P, P, P, P, P, P, I32, I32, P, P, P, P,
                               P, P, I64, P, P, I32, P]),
    "hg_row_norms": (I32, [P, I64, I32, P, P]),
    "hg_sgd": (I32, [P, P, I64, F32, P]),
    "hg_p2p_allreduce_sgd": (I32, [P, P, I64, P, P, P, P, I32, P, F32, P]),
    "hg_cache_update_scratch_bytes": (I64, [I64]),
    "hg_cache_rank": (I32, [P, I32, F64, P, P, P, P, P, P, P, P, I64, P]),
    "hg_cache_write": (I32, [I32, I32, I32, P, F64, I32, P, P, P, P, P, P, P, P, I64, P]),
    "hg_cache_sweep": (I32, [P, I64, P]),
    "hg_cache_request_reset": (I32, [P, P, P]),
    "hg_cache_lookup_sharded": (I32, [P, I64, P, P, I64, I32, P, P, P, P, F64, P, P, P, P, P, P]),
    "hg_inject_rows_sharded": (I32, [P, I64, P, P, P, I32, P, P]),
    "hg_cache_request": (I32, [P, I32, F64, P, P, P, P, P, I32, P, P, P, P, P, P, I64, P]),
    "hg_cache_apply_scratch_bytes": (I64, [I64]),
    "hg_cache_invalidate": (I32, [I32, P, P, I64, I64, I64, P, P, P, P]),
    "hg_cache_apply": (I32, [P, P, P, P, I64, I32, I64, I64, F64, I32, I64, I64, I64, P, P, P, P, P, P, I64, P]),
    "hg_peer_signal": (I32, [P, P, P]),
    "hg_peer_wait": (I32, [P, I32, P, P]),
    "hg_degree_order_scratch_bytes": (I64, [I64]),
    "hg_feature_region": (I32, [P, P, I64, I64, P, P, P, I64, P]),
    "hg_synth_power_law": (I64, [I64, I32, P, P, P]),
    "hg_build_csr2_scratch_bytes": (I64, [I64, I64]),
    "hg_build_csr2": (I32, [P, P, I64, I64, P, P, P, P, I64, P]),
    "hg_parse_int_lines": (I32, [S, I64, P, P, P, P, P, I32]),
    "hg_parse_edge_list": (I32, [S, P, P, P, P, P, P, P, I32]),
    "hg_ts_bytes": (I64, [I64, I32]),
    "hg_ts_pack": (I32, [P, I64, I32, I32, I32, I64, P, P]),
    "hg_ts_linear_fwd": (I32, [P, I64, P, I32, P, I32, P, I32, P, P]),
    "hg_ts_linear_dgrad": (I32, [P, I64, P, I32, P, I32, P, P]),
    "hg_ts_linear_wgrad": (I32, [P, I64, P, I32, P, I32, P, P, I32, P]),
}

_lib = None
_lock = threading.Lock()


class HgError(RuntimeError):
    pass


def load():
    """The loaded library (no GPU needed to load it)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise HgError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def require_cuda():
    if not torch.cuda.is_available():
        raise HgError("paper_2301_07482_b200 needs a CUDA device (sm_100a); there is no CPU fallback")


_prof = None   # {entry point: [(start_event, end_event, args)]} while profiling


def enable_profile(names):
    """Record CUDA events around the named entry points (on the current
    stream, which is the stream every caller in this package passes)."""
    global _prof
    _prof = {n: [] for n in names}


def disable_profile():
    global _prof
    p, _prof = _prof, None
    return p


def call(name, *args):
    """Invoke an int-status entry point and raise on failure."""
    lib = load()
    if _prof is not None and name in _prof:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = getattr(lib, name)(*args)
        e1.record()
        _prof[name].append((e0, e1, args))
    else:
        st = getattr(lib, name)(*args)
    if st != 0:
        raise HgError(f"{name} failed ({st}): {lib.hg_last_error().decode()}")
    return st


def query(name, *args):
    return getattr(load(), name)(*args)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
