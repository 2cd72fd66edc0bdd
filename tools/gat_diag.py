import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2301_07482_b200 as hg
from oracle.datagen import csr2_from_edges, power_law_dataset
from oracle.step import GAT, OTrainConfig, OTrainer
ds = power_law_dataset(3000, np.random.default_rng(0), m=4, feature_dim=16)
g = csr2_from_edges(ds.src, ds.dst, ds.num_nodes)
c = dict(fanouts=(10, 5, 3), hidden=32, batch_size=128, epochs=1, eta=0.05, p_grad=0.9, t_stale=5, seed=3, heads=4)
tr = hg.Trainer(g, ds.features, ds.labels, ds.train_ids, hg.TrainConfig(kind=hg.LayerKind.GAT, **c), ds.num_classes)
otr = OTrainer(g, ds.features, ds.labels, ds.train_ids, OTrainConfig(kind=GAT, **c), ds.num_classes)
seeds = hg.make_batches(ds.train_ids, tr.cfg)[0]
tr.train_iteration(0, 0, tr.sample(0, seeds)); otr.train_iteration(0, 0, otr.sample(0, seeds))
rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
pr, tapes, grads, norms = tr.last
opr, otape, ong, onorms, ograds = otr.last
for l in range(3):
    rows = opr.compute_rows[l]
    h = tapes[l].h_out.cpu().numpy()[rows]; oh = otape.h_layers[l][rows]
    print("layer", l, "h_out rel", rel(h, oh), "relu flips", int(((h > 0) != (oh > 0)).sum()), "of", h.size)
    for n in ("weight", "bias", "att_src", "att_dst"):
        print("   grad", n, rel(getattr(grads[l], n).cpu().numpy(), getattr(ograds[l], n)))
    t = tapes[l]; ot = otape.entries[l]
    H = t.heads
    print("   el rel", rel(t.el.cpu().numpy()[opr.layer_live[l]], (ot.z.reshape(ot.z.shape[0], H, -1) * otr.network.layers[l].att_src.reshape(H, -1)).sum(-1)[opr.layer_live[l]]))
for l in (1, 2):
    print("norms", l, rel(norms[l].cpu().numpy(), onorms[l]))
# intermediates of the backward vs the oracle's formulas (oracle/gat.py layer_backward)
for l in range(3):
    t, ot = tapes[l], otape.entries[l]
    rows = opr.compute_rows[l]
    H = t.heads
    F = ot.z.shape[2]
    d_out = ong[l][rows]
    gq = d_out if ot.relu is None else np.where(ot.relu, d_out, 0)
    gh = gq.reshape(-1, H, F)
    da = np.einsum("ehf,ehf->eh", gh[ot.seg], ot.z[ot.src])
    cc = np.zeros((len(rows), H), np.float32); np.add.at(cc, ot.seg, ot.alpha * da)
    de = ot.alpha * (da - cc[ot.seg]); ds_ = np.where(ot.pre > 0, de, np.float32(0.2) * de)
    der = np.zeros((len(rows), H), np.float32); np.add.at(der, ot.seg, ds_)
    gz, gcc, gder, gdl = [x.cpu().numpy() for x in t.bwd]
    print("L", l, "gz", rel(gz[:len(rows)], gq), "cc", rel(gcc[:len(rows)], cc), "der", rel(gder[:len(rows)], der),
          "alpha-sum-check", float(np.abs(np.bincount(ot.seg, ot.alpha[:, 0]) - 1).max()))
    bad = np.argsort(-np.abs(gder[:len(rows)] - der).max(1))[:5]
    for r in bad:
        deg = int((ot.seg == r).sum())
        print("     row", r, "deg+self", deg, "gpu", gder[r], "ora", der[r], "cc", gcc[r], cc[r])
