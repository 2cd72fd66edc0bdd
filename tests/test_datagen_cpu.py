"""The native power-law generator (hg_synth_power_law, host C++) against the
reference generator restated in oracle/datagen.py (histgnn/data.py:243-270,
itself pinned to the reference's golden datasets in test_oracle_golden.py):
edges, features, labels and split bit-identical for the same Generator, and
the Generator left in the same state. No GPU needed (host function)."""

import numpy as np
import pytest

from oracle.datagen import power_law_dataset
from paper_2301_07482_b200.data import synth_edges, synth_power_law_host


@pytest.mark.parametrize("n,m,d,seed", [(2, 1, 4, 0), (50, 1, 4, 1), (300, 3, 8, 2), (3000, 4, 16, 7),
                                        (20000, 10, 8, 0), (5000, 13, 3, 11)])
def test_native_generator_matches_reference_restatement(n, m, d, seed):
    ref = power_law_dataset(n, np.random.default_rng(seed), m=m, feature_dim=d, classes=5)
    got = synth_power_law_host(n, np.random.default_rng(seed), m=m, feature_dim=d, classes=5)
    assert np.array_equal(got[0], ref.src) and np.array_equal(got[1], ref.dst)
    assert np.array_equal(got[2], ref.features)
    assert np.array_equal(got[3], ref.labels)
    for a, b in zip(got[4:], (ref.train_ids, ref.val_ids, ref.test_ids)):
        assert np.array_equal(a, b)


def test_generator_state_continues_the_stream():
    r1, r2 = np.random.default_rng(3), np.random.default_rng(3)
    power_law_dataset(1000, r1, m=5, feature_dim=1)
    synth_power_law_host(1000, r2, m=5, feature_dim=1)
    assert r1.bit_generator.state == r2.bit_generator.state
    assert np.array_equal(r1.random(17), r2.random(17))


def test_buffered_half_word_is_honoured():
    # an odd number of 32-bit draws before the call leaves has_uint32 set
    r1, r2 = np.random.default_rng(5), np.random.default_rng(5)
    r1.integers(1000)
    r2.integers(1000)
    assert r2.bit_generator.state["has_uint32"] == 1
    ref = power_law_dataset(400, r1, m=3, feature_dim=2)
    src, dst = synth_edges(400, 3, r2)
    assert np.array_equal(src, ref.src[:len(src)]) and np.array_equal(dst, ref.dst)


def test_invalid_shapes_raise_value_error():
    with pytest.raises(ValueError):
        synth_edges(3, 3, 0)
    with pytest.raises(ValueError):
        synth_edges(10, 0, 0)
