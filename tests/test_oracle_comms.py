"""The fetch-accounting restatement (oracle/comms.py) pinned to the
reference's own cases (pkg/tests/test_comms.py:166-230) and to the product's
host helper (distributed.transfer_accounting)."""

import numpy as np
import pytest

from oracle.comms import fetch_bytes, merge_transfers, partition_features, requests_for_batch


def test_partition_matches_reference_cases():
    owner = partition_features(10, 4)
    assert [int((owner == d).sum()) for d in range(4)] == [3, 3, 2, 2]
    np.testing.assert_array_equal(partition_features(7, 7), np.arange(7))
    with pytest.raises(ValueError):
        partition_features(5, 0)


def test_requests_and_merge_match_reference_cases():
    owner = partition_features(10, 4)
    assert requests_for_batch(owner, np.array([0, 3, 4, 9]), 1) == [(0, 1, 1), (3, 1, 1)]
    assert requests_for_batch(owner, np.array([3, 4]), 1) == []
    assert merge_transfers([(0, 1, 5), (0, 1, 7), (2, 2, 9), (1, 0, 0)]) == [(0, 1, 12)]


def test_two_sided_adds_index_bytes_and_syncs():
    tr = [(0, 2, 100)]                                # test_comms.py:185-196: 100 ids x 4 B
    one, two = fetch_bytes(tr, False, 4), fetch_bytes(tr, True, 4)
    assert one["total_bytes"] == 400 and one["index_bytes"] == 0 and one["sync_events"] == 0
    assert two["total_bytes"] == 1200 and two["sync_events"] == 1


def test_product_accounting_equals_the_restatement():
    from paper_2301_07482_b200.distributed import owner_ranges, transfer_accounting
    rng = np.random.default_rng(0)
    for n, P in [(1000, 4), (37, 3), (64, 8)]:
        owner = partition_features(n, P)
        b = owner_ranges(n, P)
        np.testing.assert_array_equal(owner, np.repeat(np.arange(P), np.diff(b)))
        for requester in range(P):
            ids = rng.choice(n, size=n // 3, replace=False)
            counts = np.bincount(owner[ids], minlength=P)
            acc = transfer_accounting(counts, requester, 512)
            want = merge_transfers(requests_for_batch(owner, ids, requester))
            assert [(t["src"], t["dst"], t["num_ids"]) for t in acc["transfers"]] == want
            for mode, two in (("one_sided", False), ("two_sided", True)):
                assert acc[mode] == fetch_bytes(want, two, 512)
