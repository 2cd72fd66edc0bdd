#!/usr/bin/env python
"""Run the reference's own test-suite (`/root/reference/pkg/tests`) against
the drop-in, changing only the import lines.

  python tools/run_reference_tests.py stage   # here: needs /root/reference
  python tools/run_reference_tests.py run     # on the GPU box (pytest, GPU)

`stage` copies the selected reference test modules into
`baseline/_ref/reference_tests/` (git-ignored, travels to the GPU box with
the installed reference) and rewrites every `from histgnn.<m> import ...`
with m in {graphs, sampler, cache, nn, trainer, data}: the names the drop-in's
reference-typed facade (`paper_2301_07482_b200.compat.<m>`) provides come
from it, anything else (e.g. `normalize_adjacency`, the layer-math
functions, the synthetic generators) stays on the reference. The
communication simulator and SGC stay on the reference untouched: they are
test inputs / out-of-scope subsystems.

`run` executes them with pytest and deselects the cases outside the hot
path (listed with the reason in DESELECT).
"""

from __future__ import annotations

import ast
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/pkg/tests"
REF_PKG = os.path.join(ROOT, "baseline", "_ref")
OUT = os.path.join(REF_PKG, "reference_tests")
MODULES = ("test_sampler.py", "test_cache.py", "test_trainer.py", "test_graphs.py", "test_data.py",
           "test_acceptance.py")
FACADE = ("graphs", "sampler", "cache", "nn", "trainer", "data")

# node-id fragment -> reason (kept out of the run; everything else must pass)
DESELECT = {
    "test_graphs.py::test_normalize": "GCN normalisation is computed inside the aggregation kernels "
                                      "(no adjacency matrix object on the hot path)",
    "test_graphs.py::test_edge_list": "edge-list file I/O is dataset ingest (SURVEY §8(f).2), not the step",
    "test_acceptance.py::test_criterion_05": "float64 finite differences of the layer math; the device network "
                                             "computes in fp32 (gradients pinned at 1e-3 vs the reference in "
                                             "tests/test_gpu_prune_nn.py)",
    "test_acceptance.py::test_criterion_06": "SGC convergence model (histgnn.sgc): out of scope (SURVEY §2)",
    "test_acceptance.py::test_criterion_10": "PCIe communication simulator (histgnn.comms): out of scope",
}

_IMPORT = re.compile(r"^from histgnn\.(\w+) import (\([^)]*\)|[^\n]*)", re.M)


def _rewrite(src: str) -> str:
    sys.path.insert(0, ROOT)
    import importlib

    def sub(m):
        mod, names = m.group(1), m.group(2)
        if mod not in FACADE:
            return m.group(0)
        facade = importlib.import_module(f"paper_2301_07482_b200.compat.{mod}")
        listed = [n.strip() for n in names.strip("()").replace("\n", " ").split(",") if n.strip()]
        ours = [n for n in listed if hasattr(facade, n.split(" as ")[0].strip())]
        theirs = [n for n in listed if n not in ours]
        lines = []
        if ours:
            lines.append(f"from paper_2301_07482_b200.compat.{mod} import {', '.join(ours)}")
        if theirs:
            lines.append(f"from histgnn.{mod} import {', '.join(theirs)}")
        return "\n".join(lines)

    out = _IMPORT.sub(sub, src)
    ast.parse(out)
    return out


CONFTEST = '''"""Staged by tools/run_reference_tests.py: the repo root (the drop-in) and
baseline/_ref (the reference's data generators) on sys.path."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.dirname(HERE)
ROOT = os.path.dirname(os.path.dirname(REF))
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)
'''


def stage() -> None:
    if not os.path.isdir(REF_TESTS):
        raise SystemExit(f"{REF_TESTS} not found (stage runs where the reference is)")
    if not os.path.isdir(os.path.join(REF_PKG, "histgnn")):
        raise SystemExit("install the reference into baseline/_ref first (see DESIGN.md)")
    os.makedirs(OUT, exist_ok=True)
    for name in MODULES:
        with open(os.path.join(REF_TESTS, name)) as fh:
            src = fh.read()
        with open(os.path.join(OUT, name), "w") as fh:
            fh.write(_rewrite(src))
    with open(os.path.join(OUT, "conftest.py"), "w") as fh:
        fh.write(CONFTEST)
    with open(os.path.join(OUT, "pytest.ini"), "w") as fh:
        fh.write("[pytest]\naddopts = -p no:cacheprovider\n")
    print(f"staged {len(MODULES)} reference test modules into {OUT}")


def deselect_args() -> list:
    return ["-k", " and ".join(f"not {frag.split('::')[1]}" for frag in DESELECT)]


def run(extra=()) -> int:
    if not os.path.isdir(OUT):
        raise SystemExit("not staged: run `python tools/run_reference_tests.py stage` where /root/reference exists")
    cmd = [sys.executable, "-m", "pytest", OUT, "-q", "-rs", "-c", os.path.join(OUT, "pytest.ini"),
           "--rootdir", OUT] + deselect_args() + list(extra)
    return subprocess.call(cmd, cwd=OUT)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "run"
    if what == "stage":
        stage()
    else:
        sys.exit(run(sys.argv[2:]))
