"""The reference's own hot-path tests, unmodified, against the drop-in.

/root/reference/pkg/tests (copied with the pip --target install of the
reference into baseline/_ref/, which travels to the GPU box) are run in a
subprocess with tests/ref_dropin_plugin.py swapping
graphtables.table_to_graph / pagerank / triangle_count for this package's
(INTEGRATION.md §3):

* test_convert.py (all: replay equality, duplicates, empty tables, type
  errors, read-only views, mutability, worker independence, round trips);
* test_algorithms.py::TestPageRank and ::TestTriangles (known answers,
  dense-matrix and cubic-enumeration oracles, worker exactness);
* test_acceptance.py:159-270 (graph algorithms vs oracles, PageRank
  tolerances, conversion round trips, and the sort-first throughput
  criterion: 10 M rows in < 10 s).
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parent.parent
REF = REPO / "baseline" / "_ref"
REF_TESTS = REF / "graphtables_tests"

SELECTION = [
    "test_convert.py",
    "test_algorithms.py::TestPageRank",
    "test_algorithms.py::TestTriangles",
    "test_acceptance.py::test_graph_algorithms_match_oracles",
    "test_acceptance.py::test_pagerank_tolerances",
    "test_acceptance.py::test_conversion_round_trips_and_worker_independence",
    "test_acceptance.py::test_sort_first_throughput",
]


def test_reference_hot_path_tests_pass_on_the_drop_in(tmp_path):
    if not (REF / "graphtables").exists() or not REF_TESTS.exists():
        pytest.skip("reference not installed in baseline/_ref (pip --target install + tests copy)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join(
        [str(REF), str(REPO), str(REPO / "tests"), str(REF_TESTS), env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-rA", "-p", "ref_dropin_plugin", "-p",
           "no:cacheprovider", "--rootdir", str(tmp_path), *[str(REF_TESTS / s) for s in SELECTION]]
    proc = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1200)
    out = proc.stdout + proc.stderr
    log = REPO / "gpurun_out" / "reference_suite_on_dropin.log"
    try:
        log.parent.mkdir(exist_ok=True)
        log.write_text(out)
    except OSError:
        pass
    assert proc.returncode == 0, out[-6000:]
    assert "drop-in: graphtables.table_to_graph" in out
