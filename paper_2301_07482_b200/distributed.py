"""Data-parallel plumbing for the per-iteration path.

One process per GPU. Rank r of P trains global batch indices P*s + r at step
s, so every batch's sampled subgraph is bit-identical to the single-GPU run
(per-batch PCG64 streams, histgnn/sampler.py:104-106). The one exchange step
is the gradient all-reduce of the single flat parameter bucket (all layers in
one contiguous fp32 buffer, nn.Network.flat) before SGD; NCCL over NVLink on
the GPU box, gloo in the CPU tests. Feature / cache ownership follows the
reference's contiguous partition (histgnn/comms.py:329-337).
"""

from __future__ import annotations

import numpy as np


def rank_batch_indices(num_batches: int, rank: int, world: int) -> list:
    """Global batch indices rank `rank` trains, in step order."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    steps = num_batches // world          # every rank takes the same number of steps
    return [world * s + rank for s in range(steps)]


def owner_ranges(num_nodes: int, world: int) -> np.ndarray:
    """Contiguous owner ranges [bounds[r], bounds[r+1]) like
    comms.partition_features: the first num_nodes % world owners get one
    extra row."""
    base, extra = divmod(num_nodes, world)
    sizes = np.full(world, base, dtype=np.int64)
    sizes[:extra] += 1
    return np.concatenate([[0], np.cumsum(sizes)])


def owner_of(ids, bounds: np.ndarray) -> np.ndarray:
    return np.searchsorted(bounds, np.asarray(ids), side="right") - 1


def make_allreduce_hook(world: int, group=None):
    """Trainer.grad_hook that averages the flat gradient bucket over ranks
    (one all-reduce per step, fixed reduction order inside the backend)."""
    import torch.distributed as dist

    def hook(grads):
        flat = grads.flat
        dist.all_reduce(flat, group=group)
        flat.div_(world)

    # NCCL collectives are stream-ordered device work and can be captured in
    # the step's CUDA graph (engine.StepEngine); gloo's host-side all-reduce
    # cannot, so a gloo hook keeps the step eager
    hook.graph_safe = dist.get_backend(group) == "nccl"
    return hook


class P2PAllReduce:
    """Fused data-parallel exchange + SGD over peer memory (hg_p2p_allreduce_sgd).

    Replaces `make_allreduce_hook` + `sgd_step`: every rank copies its flat
    gradient bucket into its own CUDA-IPC exchange slot and raises a flag; each
    rank then reads all P slots (NVLink loads on a multi-GPU box), sums them in
    rank order, divides by P and applies SGD to its parameters in the same
    kernel, so every rank holds identical weights without an NCCL launch. Two
    kernel launches, capturable in the step's CUDA graph. A collective
    constructor (every rank of `group` calls it with the same bucket size)."""

    fused_sgd = True
    graph_safe = True

    def __init__(self, numel: int, rank: int, world: int, device, group=None, timeout_s: float = 120.0):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib
        from .sharding import _DevBuf
        _lib.require_cuda()
        self.n, self.rank, self.world = int(numel), int(rank), int(world)
        self.device = torch.device(device)
        slot_bytes = 2 * self.n * 4
        flag_off = (slot_bytes + 255) // 256 * 256
        p = ctypes.c_void_p()
        _lib.call("hg_device_alloc", flag_off + 256, ctypes.byref(p))
        self._owned = p.value
        torch.as_tensor(_DevBuf(p.value, (flag_off + 256,), "|u1"), device=self.device).zero_()
        torch.cuda.synchronize(self.device)
        lib = _lib.load()
        hb = int(lib.hg_ipc_handle_bytes())
        h = ctypes.create_string_buffer(hb)
        _lib.call("hg_ipc_export", p, h)
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h.raw), group=group)
        bases, self._opened = [], []
        for r in range(self.world):
            if r == self.rank:
                bases.append(p.value)
                continue
            q = ctypes.c_void_p()
            _lib.call("hg_ipc_open", ctypes.create_string_buffer(handles[r], hb), ctypes.byref(q))
            bases.append(q.value)
            self._opened.append(q.value)
        self.my_slots, self.my_flag = p.value, p.value + flag_off
        self.slots_dev = torch.tensor(bases, dtype=torch.int64, device=self.device)
        self.flags_dev = torch.tensor([b + flag_off for b in bases], dtype=torch.int64, device=self.device)
        self.state = torch.zeros(8, dtype=torch.int64, device=self.device)
        self.state[4] = int(timeout_s * 1e9)     # peer-wait limit (hg_collective.cu)
        dist.barrier(group=group)

    def __call__(self, grads):
        raise TypeError("P2PAllReduce fuses the exchange with SGD: call .sgd(network, grads, eta)")

    def sgd(self, network, grads, eta: float) -> None:
        from . import _lib
        if grads.flat.numel() != self.n:
            raise ValueError(f"bucket of {grads.flat.numel()} floats, exchange sized for {self.n}")
        _lib.call("hg_p2p_allreduce_sgd", _lib.ptr(network.flat), _lib.ptr(grads.flat), self.n, self.my_slots,
                  self.my_flag, _lib.ptr(self.slots_dev), _lib.ptr(self.flags_dev), self.world, _lib.ptr(self.state),
                  float(np.float32(eta)), _lib.stream_ptr())

    @property
    def timed_out(self) -> bool:
        return bool(int(self.state[3].item()))

    def check(self) -> None:
        """Raise if a peer missed an exchange (the kernel skipped the update)."""
        if self.timed_out:
            raise RuntimeError("P2P gradient exchange timed out waiting for a peer rank; parameters were not "
                               "updated from that step on")

    def close(self, group=None) -> None:
        """Unmap peers and free the exchange area (collective: barriers
        first so no peer still reads it)."""
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib
        torch.cuda.synchronize(self.device)
        dist.barrier(group=group)
        for q in self._opened:
            _lib.call("hg_ipc_close", ctypes.c_void_p(q))
        self._opened = []
        dist.barrier(group=group)
        if self._owned is not None:
            _lib.call("hg_device_free", ctypes.c_void_p(self._owned))
            self._owned = None


def apply_sgd(hook, network, grads, eta: float) -> None:
    """The optimizer step of a (possibly data-parallel) iteration: a fused
    exchange hook does both; a plain hook all-reduces, then hg_sgd."""
    from .nn import sgd_step
    if hook is not None and getattr(hook, "fused_sgd", False):
        hook.sgd(network, grads, eta)
        return
    if hook is not None:
        hook(grads)
    sgd_step(network, grads, eta)


INDEX_BYTES_PER_ID = 8     # histgnn/comms.py:26 (two-sided: the requester ships its id list)


def transfer_accounting(owner_rows, rank: int, row_bytes: int) -> dict:
    """The feature-fetch accounting of histgnn/comms.py:283-323 (simulate_fetch)
    computed from the rows this rank really read from each owner's shard
    (ShardedFeatures.owner_rows deltas): one transfer per remote owner with
    rows (requests_for_batch / merge_transfers, comms.py:187-194,326-337),
    payload = rows x row_bytes; one-sided reads move only the payload, the
    two-sided protocol adds the id list (8 B per id) and one synchronisation
    per transfer. Round scheduling / completion time model a PCIe switch tree
    and are not applicable to NVSwitch."""
    rows = [int(x) for x in (owner_rows.tolist() if hasattr(owner_rows, "tolist") else owner_rows)]
    transfers = [(o, rank, n) for o, n in enumerate(rows) if o != rank and n > 0]
    payload = sum(n for _, _, n in transfers) * int(row_bytes)
    index = sum(n for _, _, n in transfers) * INDEX_BYTES_PER_ID
    return {"transfers": [{"src": s, "dst": d, "num_ids": n} for s, d, n in transfers],
            "one_sided": {"payload_bytes": payload, "index_bytes": 0, "sync_events": 0, "total_bytes": payload},
            "two_sided": {"payload_bytes": payload, "index_bytes": index, "sync_events": len(transfers),
                          "total_bytes": payload + index},
            "local_rows": rows[rank] if 0 <= rank < len(rows) else 0}
