"""The reference's OWN tests (oracle/_ref/tests, unmodified) run against this
framework through tools/fmmb_ref_bridge.py: test_lists.py, test_pseudosort.py,
test_morton.py, test_scan.py, test_container.py, test_fmm.py (near field and
direct sums through the bound plugin), test_boxtype.py, test_partition.py and acceptance criteria 1-3."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("target", [
    "tests/test_lists.py",
    "tests/test_pseudosort.py",
    "tests/test_morton.py",
    "tests/test_scan.py",
    "tests/test_container.py",
    "tests/test_fmm.py",
    "tests/test_boxtype.py",
    "tests/test_partition.py",
    "tests/test_acceptance.py::test_criterion_1_list_correctness",
    "tests/test_acceptance.py::test_criterion_2_single_count_coverage",
    "tests/test_acceptance.py::test_criterion_3_pseudo_sort_contract",
])
def test_reference_suite_on_b200(gpu, target):
    if not os.path.isdir(os.path.join(REF, "tests")):
        pytest.skip("oracle/_ref not built")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(REF, "tests"),
                                         os.path.join(ROOT, "tools"), ROOT])
    out = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-p", "fmmb_ref_bridge", "-p",
         "no:cacheprovider", "--rootdir", REF, target],
        cwd=REF, env=env, capture_output=True, text=True, timeout=900)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    assert "build_all calls routed to the B200 build" in out.stdout
