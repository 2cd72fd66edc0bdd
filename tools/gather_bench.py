"""Feature-gather microbenchmark (hg_load_features alone): random sorted
live rows of a frontier, random node ids, a static region covering 10% of the
nodes; CUDA-event time per launch and algorithmic GB/s
(rows x (row read + fp32 row write + 12 B of indices)). Not a product path."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2301_07482_b200 import _lib  # noqa: E402

dev = torch.device("cuda")


def case(N, dim, dtype, n_src, n_live, region_frac=0.1, reps=20):
    g = torch.Generator(device="cpu").manual_seed(0)
    live = torch.sort(torch.randperm(n_src, generator=g)[:n_live])[0].to(torch.int32).to(dev)
    src_nodes = torch.randint(0, N, (n_src,), generator=g, dtype=torch.int32).to(dev)
    feats = torch.randn(N, dim, device=dev).to(dtype)
    nreg = int(N * region_frac)
    fro = torch.full((N,), -1, dtype=torch.int32, device=dev)
    reg_ids = torch.randperm(N, device=dev)[:nreg]
    fro[reg_ids] = torch.arange(nreg, dtype=torch.int32, device=dev)
    region = feats[reg_ids].contiguous()
    cnt = torch.tensor([n_live], dtype=torch.int32, device=dev)
    gctr = torch.zeros(8, dtype=torch.int64, device=dev)
    h = torch.empty((n_src, dim), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    code = 1 if dtype == torch.float16 else 0
    sp = _lib.stream_ptr()
    ts = []
    for r in range(reps + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("hg_load_features", _lib.ptr(cnt), n_src, _lib.ptr(live), _lib.ptr(src_nodes), _lib.ptr(fro),
                  _lib.ptr(region), _lib.ptr(feats), dim, code, _lib.ptr(h), _lib.ptr(gctr), None, 0, sp)
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1) / 1e3)
    # parity: every live row equals its source row (fp32)
    ids = src_nodes[live.long()].long()
    assert torch.equal(h[live.long()], feats[ids].float()), "gather mismatch"
    t = sorted(ts)[len(ts) // 2]
    isz = feats.element_size()
    byts = n_live * (dim * isz + dim * 4 + 12)
    print(f"N={N} d={dim} {str(dtype)[6:]} live={n_live}: {t*1e6:7.1f} us  {byts/t/1e9:7.1f} GB/s "
          f"({byts/1e6:.1f} MB)", flush=True)


case(2_400_000, 100, torch.float32, 650_000, 310_000)
case(2_400_000, 100, torch.float32, 650_000, 650_000)
case(111_000_000, 128, torch.float16, 900_000, 450_000)
case(111_000_000, 128, torch.float16, 900_000, 900_000)
case(30_000_000, 768, torch.float16, 600_000, 300_000)
