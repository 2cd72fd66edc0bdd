"""Feature-fetch accounting (TEST INFRASTRUCTURE ONLY): a restatement of
histgnn/comms.py's partition and transfer bookkeeping that the device's
per-owner read counters (ShardedFeatures.owner_rows) are checked against.

- partition_features  comms.py:326-337  contiguous split, first N % P owners
                                        one extra row; owner[node] -> device
- requests_for_batch  comms.py:340-349  one transfer per remote owner
- merge_transfers     comms.py:187-194  sum duplicate (src, dst), drop local
- fetch_bytes         comms.py:283-323  payload = ids x bytes_per_row;
                                        two-sided adds 8 B per id and one sync
                                        per transfer (the round schedule models
                                        a PCIe tree and is not restated)
"""

from __future__ import annotations

import numpy as np

INDEX_BYTES_PER_ID = 8


def partition_features(num_nodes: int, num_devices: int) -> np.ndarray:
    if num_devices < 1:
        raise ValueError("need at least one device")
    base, extra = divmod(num_nodes, num_devices)
    return np.repeat(np.arange(num_devices), [base + (i < extra) for i in range(num_devices)])


def requests_for_batch(owner: np.ndarray, ids, requester: int) -> list:
    own = owner[np.asarray(ids, np.int64)]
    devs, counts = np.unique(own, return_counts=True)
    return [(int(d), requester, int(c)) for d, c in zip(devs, counts) if d != requester]


def merge_transfers(requests) -> list:
    acc = {}
    for s, d, n in requests:
        if s != d and n:
            acc[(s, d)] = acc.get((s, d), 0) + n
    return [(s, d, n) for (s, d), n in sorted(acc.items())]


def fetch_bytes(transfers, two_sided: bool, bytes_per_row: int) -> dict:
    ids = sum(n for _, _, n in transfers)
    idx = ids * INDEX_BYTES_PER_ID if two_sided else 0
    return {"payload_bytes": ids * bytes_per_row, "index_bytes": idx,
            "sync_events": len(transfers) if two_sided else 0, "total_bytes": ids * bytes_per_row + idx}
