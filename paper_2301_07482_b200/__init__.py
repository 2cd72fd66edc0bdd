"""paper_2301_07482_b200 — B200-native per-iteration data path of ReFresh
(arXiv 2301.07482), a drop-in for the reference `histgnn` trainer API.

Public modules mirror the reference: graphs, sampler, cache, nn, trainer.
All compute runs in libhgb200.so (sm_100a CUDA, C-ABI, include/hgb200.h);
there is no CPU fallback.
"""

__version__ = "1.0.0"

from . import _lib  # noqa: F401
from .cache import CachePolicy, HistCache  # noqa: F401
from .graphs import CooGraph, Csr2Graph, build_csr2, csr2_from_arrays  # noqa: F401
from .nn import LayerKind, backward, cross_entropy, forward_pass, init_network, node_grad_norms, sgd_step  # noqa: F401
from .sharding import ShardedFeatures  # noqa: F401
from .sampler import (LayerBlock, LayeredSubgraph, SamplePlan, SubgraphProducer, batch_rng,  # noqa: F401
                      sample_layered, split_batches)
from .trainer import (EmbeddingLog, IterMetrics, cosine_rows, epoch_mean_estimation_error, PrunedBatch, TrainConfig, Trainer, evaluate, full_graph_logits, io_saving,  # noqa: F401
                      make_batches,  # noqa: F401
                      prune_with_cache, run_plain_loop, write_metrics_csv)
