"""Error behaviour of the drop-in API matches the reference's exception types."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_level_and_budget_errors(gpu):
    pts = np.random.default_rng(0).random((10, 3))
    with pytest.raises(gpu.CapacityError):
        gpu.build_all(pts, None, pts, max_level=21)
    with pytest.raises(gpu.CapacityError, match="budget"):
        gpu.sort_points(np.array([[0.5, 0.5, 0.5]]), None, 8, histogram_budget_bytes=1024)
    with pytest.raises(gpu.DomainError):
        gpu.sort_points(pts, None, 3, mode="bogus")
    with pytest.raises(gpu.DomainError):
        gpu.build_all(pts, None, pts)


def test_negative_coordinates_are_domain_errors(gpu):
    pts = np.random.default_rng(1).random((100, 3))
    pts[17, 1] = -0.3  # reference: out-of-bounds histogram index (UB)
    with pytest.raises(gpu.DomainError):
        gpu.build_all(pts, None, pts[:50], max_level=3)
    with pytest.raises(gpu.DomainError):
        gpu.sort_points(pts, None, 3)


def test_tiny_negative_truncates_like_reference(gpu, ref):
    """(long long)(-1e-9 * 2^L) == 0: the compiled reference keeps such points
    in box 0, and so do we."""
    pts = np.random.default_rng(2).random((50, 3))
    pts[3, 0] = -1e-9
    want = ref.build_all(pts, None, pts, max_level=3)
    got = gpu.build_all(pts, None, pts, max_level=3)
    from tests.parity import compare_structures

    assert not compare_structures(got, want)


def test_atomic_mode_equals_deterministic(gpu):
    pts = np.random.default_rng(12).random((20000, 3))
    a = gpu.sort_points(pts, None, 4, mode="deterministic")
    for w in (1, 2, 8):
        b = gpu.sort_points(pts, None, 4, mode="atomic", workers=w)
        assert np.array_equal(a.points, b.points) and np.array_equal(a.bookmarks, b.bookmarks)
