"""Native dataset parsers (csrc/hg_ingest.cu, ingest.py) against the Python
restatement of the reference's readers (oracle/ingest.py; histgnn/data.py:
109-151, graphs.py:186-218): same arrays, same error text (file:line), on
files large enough to be split over many parser threads. Host code only."""

import os

import numpy as np
import pytest

from oracle import ingest as ref
from paper_2301_07482_b200 import _lib

pytestmark = pytest.mark.skipif(not os.path.exists(_lib.LIB_PATH), reason="libhgb200.so not built")


def _err(fn, *a, **k):
    with pytest.raises(ValueError) as e:
        fn(*a, **k)
    return str(e.value)


def test_edge_list_matches_reference_reader(tmp_path):
    from paper_2301_07482_b200.ingest import read_edge_list
    rng = np.random.default_rng(0)
    n, m = 5000, 400_000                      # ~4 MB: split over several threads
    src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
    lines = []
    for i, (s, d) in enumerate(zip(src, dst)):
        if i % 997 == 0:
            lines.append("# a comment line")
        if i % 1013 == 0:
            lines.append("   ")
        lines.append(f"{s} {d}" + ("  # trailing" if i % 7 == 0 else "") + ("\t" if i % 11 == 0 else ""))
    p = tmp_path / "edges.txt"
    p.write_text("\n".join(lines) + "\n")
    for threads in (1, 8):
        s, d, nn = read_edge_list(p, nthreads=threads)
        rs, rd, rn = ref.read_edge_list(p)
        assert nn == rn
        np.testing.assert_array_equal(s, rs)
        np.testing.assert_array_equal(d, rd)


@pytest.mark.parametrize("bad,line", [("1 2 3", "expected 'src dst'"), ("1 x", "non-integer"), ("-1 2", "negative"),
                                      ("7", "expected 'src dst'")])
def test_edge_list_errors_name_the_first_bad_line(tmp_path, bad, line):
    from paper_2301_07482_b200.ingest import read_edge_list
    body = [f"{i % 50} {(i * 7) % 50}" for i in range(300_000)]
    body[123_456] = bad                       # deep inside a later chunk
    body[200_000] = "9 9 9"                   # a second, later error
    p = tmp_path / "edges.txt"
    p.write_text("\n".join(body) + "\n")
    got = _err(read_edge_list, p, nthreads=8)
    assert got == _err(ref.read_edge_list, p)
    assert f"edges.txt:123457:" in got and line in got


def test_edge_list_range_against_node_count(tmp_path):
    from paper_2301_07482_b200.ingest import read_edge_list
    p = tmp_path / "edges.txt"
    p.write_text("0 1\n0 3\n")
    assert _err(read_edge_list, p, num_nodes=3) == _err(ref.read_edge_list, p, num_nodes=3)
    p.write_text("")
    s, d, n = read_edge_list(p)
    assert len(s) == 0 and n == 0


def test_int_lines_match_reference_reader(tmp_path):
    from paper_2301_07482_b200.ingest import read_int_lines
    rng = np.random.default_rng(1)
    v = rng.integers(0, 1000, 600_000)
    text = "\n".join((f"  {x} " if i % 5 == 0 else (f"+{x}" if i % 13 == 0 else str(x))) + ("\n" if i % 17 == 0 else "")
                     for i, x in enumerate(v))
    p = tmp_path / "labels.txt"
    p.write_text(text + "\n")
    np.testing.assert_array_equal(read_int_lines(p, "class id", nthreads=8), ref.read_int_lines(p, "class id"))
    p.write_text("1_000\n2\n")
    np.testing.assert_array_equal(read_int_lines(p, "node id"), [1000, 2])


@pytest.mark.parametrize("bad", ["banana", "-4", "9", "1__0", "3.0"])
def test_int_line_errors_match_reference_wording(tmp_path, bad):
    from paper_2301_07482_b200.ingest import read_int_lines
    body = [str(i % 5) for i in range(250_000)]
    body[200_001] = bad
    p = tmp_path / "test.txt"
    p.write_text("\n".join(body) + "\n")
    assert _err(read_int_lines, p, "node id", upper=5, nthreads=8) == _err(ref.read_int_lines, p, "node id", upper=5)


def test_reference_ingest_cases(tmp_path):
    """The reference's own ingest cases (pkg/tests/test_data.py:80-130)."""
    from paper_2301_07482_b200.compat.data import Dataset, ingest, load_features, save_dataset, save_features
    from paper_2301_07482_b200.compat.graphs import CooGraph
    ds = Dataset(CooGraph(np.array([0, 1, 2]), np.array([1, 2, 0]), 3),
                 np.array([[0.5, -1.25], [3.0, 0.0], [-0.0, 7.5]], np.float32), np.array([1, 0, 1]), [0], [1], [2])
    save_dataset(tmp_path, ds)
    back = ingest(tmp_path)
    assert back.features.tobytes() == ds.features.tobytes()
    np.testing.assert_array_equal(back.graph.src, ds.graph.src)
    np.testing.assert_array_equal(back.graph.dst, ds.graph.dst)
    assert back.num_classes == 2 and list(back.test_ids) == [2]
    save_features(tmp_path / "features.bin", ds.features[:2])
    msg = _err(ingest, tmp_path)
    assert "features.bin" in msg and "2" in msg and "3" in msg
    save_dataset(tmp_path, ds)
    (tmp_path / "labels.txt").write_text("0\nbanana\n1\n")
    assert "labels.txt:2" in _err(ingest, tmp_path)
    save_dataset(tmp_path, ds)
    (tmp_path / "edges.txt").write_text("0 1\n0 3\n")
    assert "edges.txt" in _err(ingest, tmp_path)
    (tmp_path / "features.bin").write_bytes(b"\x01\x02\x03")
    assert "truncated" in _err(load_features, tmp_path / "features.bin")
    os.remove(tmp_path / "val.txt")
    with pytest.raises(FileNotFoundError, match="val.txt"):
        ingest(tmp_path)
