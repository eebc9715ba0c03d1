"""Reentrancy of the drop-in (SURVEY 8(b) "Threading": the reference's
compiled kernels are nogil and reentrant).  Several host threads call
build_all / sort_points on the SAME device (one shared library handle)
concurrently; every result is bit-identical to the serial one."""

import threading

import numpy as np
import pytest

from paper_1301_1704_b200.workloads import generate
from tests.parity import compare_structures

pytestmark = pytest.mark.gpu


def _run_threads(fns):
    out = [None] * len(fns)
    errs = []
    start = threading.Barrier(len(fns))

    def body(i):
        try:
            start.wait()
            out[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=body, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    return out


def test_concurrent_build_all_matches_serial(gpu):
    cases = [generate(40000 + 7000 * k, 30000 + 5000 * k, "uniform" if k % 2 else "sphere", 70 + k)
             + (4 + k % 3,) for k in range(4)]
    serial = [gpu.build_all(s, q, r, max_level=L) for s, q, r, L in cases]
    for _ in range(3):
        got = _run_threads([lambda c=c: gpu.build_all(c[0], c[1], c[2], max_level=c[3])
                            for c in cases * 2])
        for k, g in enumerate(got):
            errors = compare_structures(g, serial[k % len(cases)])
            assert not errors, errors


def test_concurrent_device_builds_and_sorts(gpu):
    import torch

    dev = torch.device("cuda", 0)
    s, q, r = generate(2**17, 2**17, "uniform", 5)
    ts, tq, tr = (torch.from_numpy(a).to(dev) for a in (s, q, r))
    want = gpu.build_all(s, q, r, max_level=6)
    want_sort = gpu.sort_points(s, q, 6)

    def build():
        st = gpu.build_all_device(ts, tq, tr, 6)
        torch.cuda.current_stream(dev).synchronize()
        return st.to_numpy()

    def sort():
        return gpu.sort_points(s, q, 6)

    got = _run_threads([build, sort, build, sort, build, sort])
    for k, g in enumerate(got):
        if k % 2 == 0:
            assert not compare_structures(g, want)
        else:
            for f in ("points", "charges", "permutation", "bookmarks", "non_empty_index", "boxes"):
                assert np.array_equal(getattr(g, f), getattr(want_sort, f)), f
