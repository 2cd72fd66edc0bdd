"""Feature-gather DRAM-traffic probe (run under ncu): the same row gather
into outputs allocated different ways, to separate algorithmic bytes from
allocator / alignment effects. Not part of the product path."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2301_07482_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
N, n_src, n_live = 2_400_000, 650_000, 310_000
g = torch.Generator(device="cpu").manual_seed(0)
live = torch.sort(torch.randperm(n_src, generator=g)[:n_live])[0].to(torch.int32).to(dev)
src_nodes = torch.randint(0, N, (n_src,), generator=g, dtype=torch.int32).to(dev)
cnt = torch.tensor([n_live], dtype=torch.int32, device=dev)
gctr = torch.zeros(8, dtype=torch.int64, device=dev)
sp = _lib.stream_ptr()
cudart = ctypes.CDLL("libcudart.so")
ws = torch.empty(int(_lib.query("hg_load_features_scratch_bytes", n_src)), dtype=torch.uint8, device=dev)


def run(dim, out_ptr, tag):
    feats = torch.randn(N, dim, device=dev)
    for _ in range(3):
        _lib.call("hg_load_features", _lib.ptr(cnt), n_src, _lib.ptr(live), _lib.ptr(src_nodes), None,
                  _lib.ptr(feats), _lib.ptr(feats), dim, 0, out_ptr, _lib.ptr(gctr), _lib.ptr(ws), ws.numel(), sp)
    torch.cuda.synchronize()
    print(tag, "done", flush=True)


h = torch.empty((n_src, 100), device=dev)
run(100, h.data_ptr(), "torch_d100")
p = ctypes.c_void_p()
assert cudart.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(n_src * 100 * 4)) == 0
run(100, p.value, "cudaMalloc_d100")
h128 = torch.empty((n_src, 128), device=dev)
run(128, h128.data_ptr(), "torch_d128")
