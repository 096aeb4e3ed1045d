"""Run the REFERENCE's own test files against the GPU path.

The reference package is copied (untracked) to baseline/_ref/pkg; with
paper_2306_10410_b200.integration.patch_reference applied (via the
ref_patch_plugin pytest plugin) its seam (_parallel first-hit / compaction /
scatter) and its name-imported apply_permutation / coo_to_csr / spmv_pull run
on libboba_b200.  The selected tests are the ones SURVEY.md §4 lists as the
hot path's parity suite, plus the reference's benchmark-record tests (its
run_bench / compare_records drive the patched path).  The copy is made by
tools/install_reference.sh (gitignored, shipped to the GPU box).
"""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF_PKG = os.path.join(ROOT, "baseline", "_ref", "pkg")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(REF_PKG), reason="baseline/_ref/pkg not present")]

SELECT = [
    "tests/test_ordering.py::TestBobaSequential",
    "tests/test_ordering.py::TestBobaParallel",
    "tests/test_ordering.py::TestEveryOrderingIsAPermutation",
    "tests/test_ordering.py::TestEstimators",
    "tests/test_graph.py::TestCooToCsr",
    "tests/test_graph.py::TestApplyPermutation",
    "tests/test_graph.py::TestDegrees",
    "tests/test_kernels.py::TestSpmv",
    "tests/test_kernels.py::TestPageRank",
    # the reference's own run_bench / compare_records on the patched
    # path (checksums identical across orderings, end-to-end sums, row contract)
    "tests/test_bench_cli.py::TestRunBench",
    "tests/test_bench_cli.py::TestCompare",
]


def test_reference_hot_path_tests_pass_on_gpu(tmp_path):
    env = dict(os.environ)
    env.update(BOBA_REPO_ROOT=ROOT, BOBA_REF_SRC=os.path.join(REF_PKG, "src"),
               NUMBA_CACHE_DIR=str(tmp_path / "numba"), PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), os.path.join(REF_PKG, "src"), ROOT]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "ref_patch_plugin",
           "-x", *SELECT]
    r = subprocess.run(cmd, cwd=REF_PKG, env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert " passed" in r.stdout
