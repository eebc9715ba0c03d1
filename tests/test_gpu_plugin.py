"""The kernel plugin (drop-in for fmmkit.backend.kernels) vs the CPU oracle /
the compiled reference kernels, including numpy/torch in-out conventions."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_1301_1704_b200.workloads import generate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K(gpu):
    from paper_1301_1704_b200 import kernels

    return kernels


def test_bit_dilation_roundtrip(K):
    rng = np.random.default_rng(1)
    v = rng.integers(0, 2**21, size=10000, dtype=np.uint64)
    s = K.spread_bits(v)
    assert s.dtype == np.uint64
    assert np.array_equal(K.compact_bits(s), v)
    ix, iy, iz = (rng.integers(0, 2**21, size=5000, dtype=np.uint64) for _ in range(3))
    idx = K.interleave_coords(ix, iy, iz)
    bx, by, bz = K.deinterleave_indices(idx)
    assert np.array_equal(bx, ix) and np.array_equal(by, iy) and np.array_equal(bz, iz)
    # reference examples (tests/test_morton.py:35-46): (1,1,1)->7, (2,1,0)@L2->10
    assert K.interleave_coords(np.array([1], np.uint64), np.array([1], np.uint64),
                               np.array([1], np.uint64))[0] == 7
    assert K.interleave_coords(np.array([2], np.uint64), np.array([1], np.uint64),
                               np.array([0], np.uint64))[0] == 10


def test_encode_strided_columns_match_oracle(K):
    src, _, _ = generate(20000, 1, "sphere", 3)
    for L in (0, 4, 9, 20):
        got = K.encode_points(src[:, 0], src[:, 1], src[:, 2], L)
        assert np.array_equal(got, orc.encode(src, L))
    # box index of (0.55, 0.3, 0.05) at level 2 is 10 (tests/test_morton.py:76-80)
    assert K.encode_points(np.array([0.55]), np.array([0.3]), np.array([0.05]), 2)[0] == 10


def test_assign_box_ranks_matches_sequential_counter(K):
    src, _, _ = generate(30000, 1, "uniform", 4)
    boxes = orc.encode(src, 3)
    bins, ranks = K.assign_box_ranks(boxes, 8**3)
    ob = np.empty(8**3, dtype=np.int64)
    orr = np.empty(boxes.size, dtype=np.int64)
    orc.load().orc_assign_ranks(boxes.ctypes.data, boxes.size, ob.ctypes.data, 8**3,
                                orr.ctypes.data)
    assert bins.dtype == np.int64 and ranks.dtype == np.int64
    assert np.array_equal(bins, ob) and np.array_equal(ranks, orr)
    b2, r2 = K.assign_box_ranks_atomic(boxes, 8**3, 8)
    assert np.array_equal(b2, ob)


@pytest.mark.parametrize("L", [1, 2, 3, 5, 7])
def test_segments_match_oracle(K, L):
    s = orc.sort_points(generate(6000, 1, "uniform", L)[0], None, L)
    r = orc.sort_points(generate(1, 5000, "sphere", L + 10)[2], None, L)
    a = K.adjacent_segments(r.non_empty_index, s.non_empty_index, L)
    b = orc.adjacent_segments(r.non_empty_index, s.non_empty_index, L)
    assert all(np.array_equal(x, y) and x.dtype == y.dtype for x, y in zip(a, b))
    a = K.stencil_segments(r.non_empty_index, s.non_empty_index, L)
    b = orc.stencil_segments(r.non_empty_index, s.non_empty_index, L)
    assert all(np.array_equal(x, y) and x.dtype == y.dtype for x, y in zip(a, b))


def test_segments_arbitrary_inputs(K):
    """Unsorted receivers and duplicated sources follow the reference's
    per-box bisect semantics (_ckernels.pyx:172-287)."""
    rng = np.random.default_rng(9)
    src = np.sort(rng.integers(0, 8**4, size=600).astype(np.uint64))  # duplicates
    recv = rng.integers(0, 8**4, size=300).astype(np.uint64)  # unsorted
    for fn, ofn in ((K.adjacent_segments, orc.adjacent_segments),
                    (K.stencil_segments, orc.stencil_segments)):
        a, b = fn(recv, src, 4), ofn(recv, src, 4)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_empty_and_low_level_segments(K):
    e = np.empty(0, dtype=np.uint64)
    bm, lst = K.adjacent_segments(e, np.array([1, 2], np.uint64), 3)
    assert bm.tolist() == [0] and lst.size == 0
    bm, rk, cd = K.stencil_segments(np.array([5], np.uint64), np.array([1, 2], np.uint64), 1)
    assert bm.tolist() == [0, 0] and rk.size == 0 and cd.dtype == np.int16


def test_propagate_and_scan(K):
    keys = orc.sort_points(generate(5000, 1, "uniform", 2)[0], None, 6).non_empty_index
    assert np.array_equal(K.propagate_to_parents(keys), orc.propagate(keys))
    shuffled = np.random.default_rng(3).permutation(keys)
    assert np.array_equal(K.propagate_to_parents(shuffled), np.unique(keys >> np.uint64(3)))
    v = np.random.default_rng(4).integers(0, 1000, size=100001)
    out, tot = K.exclusive_scan(v)
    assert tot == v.sum() and out[0] == 0 and np.array_equal(out[1:], np.cumsum(v)[:-1])
    with pytest.raises(ValueError):
        K.exclusive_scan(np.array([1, -1]))


def test_device_in_device_out(K):
    v = torch.arange(100, dtype=torch.int64, device="cuda").view(torch.uint64)
    s = K.spread_bits(v)
    assert isinstance(s, torch.Tensor) and s.is_cuda


def test_install_into_reference(ref, K):
    """The reference's own API runs on this plugin (swap of cli.py:263-266)."""
    import fmmkit.backend as bm

    saved = bm.kernels
    try:
        K.install(ref)
        assert ref.backend_name() == "compiled"
        src, q, recv = generate(3000, 3000, "uniform", 60)
        st = ref.build_all(src, q, recv, max_level=4)
    finally:
        bm.kernels = saved
    want = ref.build_all(src, q, recv, max_level=4)
    from tests.parity import compare_structures

    assert not compare_structures(st, want)


def test_build_bookmarks_and_reorder_match_oracle(K):
    """kernels.build_bookmarks / kernels.reorder (pseudosort.py:68-78, 105-135)
    on the device vs the C restatement, numpy and CUDA in/out."""
    src, q, _ = generate(40000, 1, "sphere", 11)
    for L in (1, 3, 5):
        boxes = orc.encode(src, L)
        bins, ranks = K.assign_box_ranks(boxes, 8**L)
        bm, ne = K.build_bookmarks(bins)
        obm, one = orc.build_bookmarks(bins)
        assert bm.dtype == np.int64 and ne.dtype == np.uint64
        assert np.array_equal(bm, obm) and np.array_equal(ne, one)
        got = K.reorder(src, q, bins, boxes, ranks, L)
        want = orc.reorder(src, q, bins, boxes, ranks)
        for f in ("points", "charges", "permutation", "bookmarks", "non_empty_index", "boxes"):
            a, b = np.asarray(getattr(got, f)), getattr(want, f)
            assert a.dtype == b.dtype and np.array_equal(a, b), (L, f)
        nq = K.reorder(src, None, bins, boxes, ranks, L)
        assert nq.charges is None and np.array_equal(nq.points, want.points)
    # device in -> device out
    dev = torch.device("cuda", 0)
    bins_d = torch.tensor([0, 3, 0, 0, 2, 1], dtype=torch.int64, device=dev)
    bm, ne = K.build_bookmarks(bins_d)
    assert bm.is_cuda and bm.cpu().tolist() == [0, 3, 5, 6]
    assert ne.view(torch.int64).cpu().tolist() == [1, 4, 5]
    # empty and all-zero histograms
    bm, ne = K.build_bookmarks(np.zeros(0, np.int64))
    assert bm.tolist() == [0] and ne.size == 0
    bm, ne = K.build_bookmarks(np.zeros(9, np.int64))
    assert bm.tolist() == [0] and ne.size == 0


def test_reorder_rejects_bad_sort_index(K):
    from paper_1301_1704_b200.errors import DomainError

    pts = np.random.default_rng(0).random((10, 3))
    boxes = np.zeros(10, np.uint64)
    with pytest.raises(DomainError):
        K.reorder(pts, None, np.array([10], np.int64), boxes[:5], np.arange(5), 0)
    with pytest.raises(DomainError):  # box index outside the histogram
        K.reorder(pts, None, np.array([10], np.int64), boxes + 3, np.arange(10), 0)
    with pytest.raises(DomainError):
        K.build_bookmarks(np.array([1, -2, 3], np.int64))
