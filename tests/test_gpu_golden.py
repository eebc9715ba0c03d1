"""GPU build vs the committed golden vectors of the reference (no reference
needed at run time): bit-exact arrays, dtypes and shapes."""

import numpy as np
import pytest

from tests import golden_io as gio

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(gio.small_cases()))
def test_build_all_small_golden(gpu, name):
    case = gio.small_cases()[name]
    src, q, recv, L = gio.case_inputs(case)
    st = gpu.build_all(src, q, recv, max_level=L)
    errors = gio.compare_flat(gio.flatten(st), gio.expected_outputs(case))
    assert not errors, errors


@pytest.mark.parametrize("name", sorted(gio.hashes()))
def test_build_all_large_golden_hashes(gpu, name):
    spec = gio.hashes()[name]
    src, q, recv, L = gio.large_inputs(spec)
    st = gpu.build_all(src, q, recv, max_level=L)
    got = {k: gio.sha(v) for k, v in gio.flatten(st).items()}
    bad = sorted(k for k in spec["arrays"] if got.get(k) != spec["arrays"][k])
    assert not bad and set(got) == set(spec["arrays"]), bad


def test_encode_points_golden_edges(gpu):
    from paper_1301_1704_b200 import kernels as K

    e = gio.encode_edges()
    pts = e["pts"]
    for L in (0, 1, 3, 7, 9, 20):
        got = K.encode_points(pts[:, 0], pts[:, 1], pts[:, 2], L)
        assert got.dtype == np.uint64
        assert np.array_equal(got, e[f"L{L}"]), L
