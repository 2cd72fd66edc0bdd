"""Reference-typed facade over the device path: `histgnn`'s module layout and
value conventions (int64 numpy ids, numpy offsets / rows, copies on return),
with every computation still running in libhgb200.so.

The main package (`paper_2301_07482_b200.sampler`, `.trainer`, ...) hands
back device tensors so that a training loop never leaves the GPU. Code
written against the reference indexes numpy arrays with the results
(`block.src_nodes[block.adj.neighbors(r)]`, `np.sort(pruned.injected[b][0])`,
`sub.layers[i].src_nodes is sub.layers[i - 1].dst_nodes`), so this
subpackage converts at the boundary:

  histgnn.graphs   -> compat.graphs   (host Csr2Graph; device mirror on demand)
  histgnn.sampler  -> compat.sampler  (sample_layered / SubgraphProducer on the GPU)
  histgnn.cache    -> compat.cache    (the device HistCache, numpy views)
  histgnn.nn       -> compat.nn       (reference-shaped LayerParams / Network)
  histgnn.trainer  -> compat.trainer  (prune_with_cache / Trainer on the GPU)
  histgnn.data     -> compat.data     (dataset format; native multi-threaded parsers)

A reference user (or the reference's own test-suite, `tools/
run_reference_tests.py`) changes only the import line.
"""

from . import cache, data, graphs, nn, sampler, trainer  # noqa: F401
