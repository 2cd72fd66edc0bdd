"""CPU oracle for the ReFresh per-iteration data path — TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference `histgnn`
algorithms (/root/reference/pkg/src/histgnn, a pure-Python CPU package) for
the one hot path this repository accelerates: layered sampling, cache-aware
pruning, the historical-embedding cache, the feature gather, the SAGE/GCN
block convolutions with their hand backward, and the training iteration that
strings them together. Every function cites the reference file:line it
restates.

Who may use it: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` leg — and there only as the checker or
the timed CPU baseline. The product package `paper_2301_07482_b200` never
imports it; the product fails loudly when its CUDA library is missing.

Pinning: the oracle is checked bit-exactly (integers) and to fp tolerance
(floats) against golden vectors produced by importing the reference itself in
the build container (`tests/golden/make_golden.py` → `tests/golden/*.npz`,
numpy version recorded inside each fixture) — see `tests/test_oracle_golden.py`.
"""

from .datagen import Dataset, power_law_dataset, sbm_dataset, csr2_from_edges
from .rng import pcg64_seed_state, pcg64_keys53, PCG_MULT
from .sampling import OBlock, OSubgraph, sample_layered, batch_rng, split_batches
from .histcache import OCachePolicy, OHistCache
from .step import (
    ONetwork,
    init_network,
    prune_with_cache,
    load_input,
    forward_pass,
    backward,
    cross_entropy,
    node_grad_norms,
    sgd_step,
    OTrainer,
    make_batches,
    run_plain_loop,
)

__all__ = [
    "Dataset", "power_law_dataset", "sbm_dataset", "csr2_from_edges",
    "pcg64_seed_state", "pcg64_keys53", "PCG_MULT",
    "OBlock", "OSubgraph", "sample_layered", "batch_rng", "split_batches",
    "OCachePolicy", "OHistCache",
    "ONetwork", "init_network", "prune_with_cache", "load_input", "forward_pass",
    "backward", "cross_entropy", "node_grad_norms", "sgd_step", "OTrainer",
    "make_batches", "run_plain_loop",
]
