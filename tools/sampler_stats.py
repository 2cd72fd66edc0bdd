"""Per-layer sampler workload at a benchmark shape: frontier rows, candidate
in-edges, degree distribution of the frontier (what k_select processes).
Not a product path."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2301_07482_b200 as hg  # noqa: E402
from paper_2301_07482_b200.data import csr2_from_edges_device  # noqa: E402

cfgd = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
src, dst, feats, labels, train = bench.make_data(cfgd)
g = csr2_from_edges_device(src, dst, cfgd["n"], "cuda")
del src, dst
deg_all = (g.end - g.start).cpu().numpy()
plan = hg.SamplePlan(bench.FANOUTS, bench.BATCH, 0)
batches = hg.split_batches(train, bench.BATCH, np.random.default_rng(0))
for b in range(3):
    sub = hg.sample_layered(g, batches[b], plan, hg.batch_rng(0, b))
    print(f"batch {b}")
    for li, blk in enumerate(reversed(sub.layers)):      # outermost first = sampling order
        fr = blk.dst_nodes.cpu().numpy().astype(np.int64)
        d = deg_all[fr]
        fan = bench.FANOUTS[li]
        bins = [0, 8, 16, 32, 64, 128, 512, 2048, 1 << 40]
        h = np.histogram(d, bins=bins)[0]
        cand = np.histogram(d, bins=bins, weights=d)[0]
        print(f"  layer {li} fanout {fan}: F={len(fr)} candidates={int(d.sum())} chunks32={int(np.ceil(d / 32).sum())} "
              f"max={int(d.max())}")
        for lo, hi, n, c in zip(bins[:-1], bins[1:], h, cand):
            if n:
                print(f"     deg ({lo},{hi}]: rows {n:8d} ({100 * n / len(fr):5.1f}%)  candidates {int(c):10d} "
                      f"({100 * c / d.sum():5.1f}%)")
