"""Diagnostic (GPU): distribution of the layer-1/2 gradient norms of the C2
step over the cache-rank buckets (kNB buckets over the occupied fp64 bit
range, as hg_cache.cu's bucket sort cuts them). Prints bucket-size quantiles."""
import numpy as np
import torch

import bench
import paper_2301_07482_b200 as hg
from paper_2301_07482_b200.data import csr2_from_edges_device

cfgd = bench.CONFIGS["c2"]
dev = torch.device("cuda", 0)
src, dst, feats, labels, train = bench.make_data(cfgd)
graph = csr2_from_edges_device(src, dst, cfgd["n"], dev)
tcfg = hg.TrainConfig(fanouts=bench.FANOUTS, hidden=bench.HIDDEN, batch_size=bench.BATCH, eta=bench.ETA,
                      kind=hg.LayerKind.SAGE_MEAN, p_grad=bench.P_GRAD, t_stale=bench.T_STALE, seed=0, epochs=1)
tr = hg.Trainer(graph, torch.from_numpy(feats).to(dev), labels, train, tcfg, cfgd["classes"])
batches = hg.make_batches(train, tcfg)
for i in range(30):
    tr.train_iteration(i, 0, tr.sample(i, batches[i]))
    if i % 10 != 9:
        continue
    for l in (1, 2):
        x = tr.last[3][l].cpu().numpy()
        bits = x.view(np.uint64)
        lo, hi = int(bits.min()), int(bits.max())
        for nb in (16384, 65536):
            r = hi - lo
            nbits = r.bit_length()
            shift = max(0, nbits - int(np.log2(nb)))
            b = np.minimum((bits - np.uint64(lo)) >> np.uint64(shift), nb - 1)
            cnt = np.bincount(b.astype(np.int64), minlength=nb)
            occ = cnt[cnt > 0]
            print(f"step {i} layer {l} n {len(x)} nb {nb} occupied {len(occ)} max {cnt.max()} "
                  f"q50/90/99 {np.percentile(occ, [50, 90, 99])} items in buckets>32: {cnt[cnt > 32].sum()} "
                  f">256: {cnt[cnt > 256].sum()} log10 range {np.log10(x.max() / max(x.min(), 1e-300)):.1f}")
