"""Shared test setup.

Markers: `gpu` tests need a CUDA device and libfmmb200.so; everything else
runs on CPU.  The reference CPU implementation (the checker) is the
unmodified fmmkit built into oracle/_ref by oracle/build_ref.sh; the C
restatement in oracle/ is loaded through oracle/oracle.py.  Both are test
infrastructure only.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and libfmmb200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def have_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def reference():
    """The unmodified reference package (CPU checker), or skip."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import fmmkit  # noqa: F401
    except ImportError:
        pytest.skip("reference build oracle/_ref missing (run oracle/build_ref.sh)")
    import fmmkit

    return fmmkit


@pytest.fixture(scope="session")
def ref():
    return reference()


@pytest.fixture(scope="session")
def gpu():
    if not have_gpu():
        pytest.skip("no CUDA device")
    import paper_1301_1704_b200 as fb

    fb._lib.load()
    return fb
