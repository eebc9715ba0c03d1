"""build_all on the GPU vs the reference CPU build_all: every output array
bit-identical (values, dtypes, shapes) on the same inputs."""

import numpy as np
import pytest

from paper_1301_1704_b200.workloads import generate
from tests.parity import compare_structures

pytestmark = pytest.mark.gpu

CASES = [
    # (n_src, n_recv, level, dist, seed)
    (3000, 3000, 4, "uniform", 60),
    (4096, 4096, 5, "sphere", 27),
    (2**16, 2**16, 4, "uniform", 1),  # c1
    (1000, 700, 3, "uniform", 5),
    (1, 1, 3, "uniform", 9),
    (500, 0, 3, "uniform", 3),
    (0, 400, 3, "uniform", 4),
    (0, 0, 3, "uniform", 4),
    (300, 200, 0, "uniform", 7),
    (300, 200, 1, "uniform", 7),
    (300, 200, 2, "uniform", 7),
    (20000, 15000, 6, "sphere", 11),
    (2**18, 2**18, 7, "uniform", 2),
    (2**17, 2**17, 9, "sphere", 3),
    (5000, 5000, 10, "sphere", 8),
    (3000, 2000, 11, "uniform", 12),
]


@pytest.fixture(params=["auto", "onesweep", "bucket_hist", "serial"])
def sort_path(request, gpu):
    """Every sort-phase strategy: bucket sort (speculative regions, overflow
    rerun) with the local pass overlapped on the side stream, Onesweep, the
    histogram-sized bucket path, and the bucket path serialised on one stream."""
    if request.param == "serial":
        gpu._lib.set_overlap(False)
        gpu._lib.set_sort_path("auto")
    else:
        gpu._lib.set_sort_path(request.param)
    yield request.param
    gpu._lib.set_sort_path("auto")
    gpu._lib.set_overlap(True)


@pytest.mark.parametrize("n,m,level,dist,seed", CASES)
def test_build_all_matches_reference(gpu, ref, sort_path, n, m, level, dist, seed):
    src, q, _ = generate(n, 1, dist, seed)
    _, _, recv = generate(1, m, dist, seed + 1000)
    budget = max(2 << 30, 8 ** level * 8)
    want = ref.build_all(src, q, recv, max_level=level, histogram_budget_bytes=budget)
    got = gpu.build_all(src, q, recv, max_level=level, histogram_budget_bytes=budget)
    errors = compare_structures(got, want)
    assert not errors, "\n".join(errors)
    if sort_path == "onesweep" and n + m > 0 and gpu.lists._bitmap_path_ok(level, n + m):
        assert got.sort_path == "onesweep"


def test_bucket_overflow_reruns_on_onesweep(gpu, ref):
    """A dense cluster overflows the bucket sort's shared-memory capacity: the
    build reruns on the Onesweep path and still matches the reference."""
    rng = np.random.default_rng(5)
    src = 0.3 + 1e-4 * rng.random((60000, 3))  # one finest box at L=5
    recv = rng.random((5000, 3))
    q = rng.normal(size=60000)
    want = ref.build_all(src, q, recv, max_level=5)
    got = gpu.build_all(src, q, recv, max_level=5)
    assert got.sort_path == "onesweep"
    assert not compare_structures(got, want)


def test_crowded_box_inside_bucket(gpu, ref):
    """A box with more points than the in-box ranking handles (> 64) inside a
    bucket that still fits shared memory: the bucket falls back to the
    in-smem LSD passes; the rest of the build stays on the bucket path."""
    src, q, recv = generate(2**16, 2**16, "uniform", 31)
    src = np.concatenate([src, np.repeat(src[:1], 200, axis=0)])
    q = np.concatenate([q, np.arange(200.0)])
    want = ref.build_all(src, q, recv, max_level=5)
    got = gpu.build_all(src, q, recv, max_level=5)
    assert got.sort_path == "bucket"
    assert not compare_structures(got, want)


def test_overfull_bucket_is_refined(gpu, ref):
    """A coarse bucket with 3x the shared-memory capacity: the speculative
    regions overflow, the histogram pass refines the bucket into sub-bin
    groups, and the build stays on the bucket path (twice: the second build
    of the same shape starts with the histogram pass)."""
    src, q, recv = generate(2**16, 2**16, "uniform", 41)
    extra = np.random.default_rng(2).random((3000, 3)) * 0.25  # one level-2 box
    src = np.concatenate([src, extra])
    q = np.concatenate([q, np.ones(3000)])
    want = ref.build_all(src, q, recv, max_level=5)
    for _ in range(2):
        got = gpu.build_all(src, q, recv, max_level=5)
        assert got.sort_path == "bucket"
        assert not compare_structures(got, want)


def test_uniform_build_takes_bucket_path(gpu, ref):
    src, q, recv = generate(2**17, 2**17, "uniform", 21)
    want = ref.build_all(src, q, recv, max_level=6)
    got = gpu.build_all(src, q, recv, max_level=6)
    assert got.sort_path == "bucket"
    assert not compare_structures(got, want)


def test_build_all_receivers_without_charges(gpu, ref):
    src, _, recv = generate(2000, 2000, "uniform", 13)
    want = ref.build_all(src, None, recv, max_level=4)
    got = gpu.build_all(src, None, recv, max_level=4)
    assert got.sorted_src.charges is None
    assert not compare_structures(got, want)


def test_boundary_coordinates(gpu, ref):
    one = 1.0
    below = np.nextafter(1.0, 0.0)
    pts = np.array([
        [0.0, 0.0, 0.0], [one, one, one], [below, below, below], [2.0**-30, 0.5, one],
        [0.5, 0.25, 0.75], [one, 0.0, below], [-0.0, 0.3, 0.3], [0.999999, 1e-300, 0.5],
    ])
    for level in (0, 1, 3, 7, 9):
        want = ref.build_all(pts, np.arange(8.0), pts[::-1].copy(), max_level=level)
        got = gpu.build_all(pts, np.arange(8.0), pts[::-1].copy(), max_level=level)
        assert not compare_structures(got, want), level


def _reference_sparse(ref, src, q, recv, level):
    """The reference's build_all at levels whose dense 8^L histogram cannot be
    allocated (L >= 12): the same steps with the histogram rank replaced by
    the stable argsort it equals (the reference's own oracle,
    tests/test_pseudosort.py:94-104); encode, the level directory, E2 and E4
    are the reference's own functions (lists.py:69-130, compiled kernels)."""
    from types import SimpleNamespace

    k = ref.backend.kernels

    def sort(pts, charges):
        boxes = k.encode_points(pts[:, 0], pts[:, 1], pts[:, 2], level)
        perm = np.argsort(boxes, kind="stable").astype(np.int64)
        sb = boxes[perm]
        head = np.ones(sb.shape[0], dtype=bool)
        head[1:] = sb[1:] != sb[:-1]
        starts = np.flatnonzero(head).astype(np.int64)
        bm = np.append(starts, np.int64(sb.shape[0]))
        return SimpleNamespace(level=level, points=pts[perm],
                               charges=None if charges is None else charges[perm],
                               permutation=perm, bookmarks=bm, non_empty_index=sb[starts],
                               boxes=sb)

    ss, sr = sort(src, q), sort(recv, None)
    table = ref.lists.build_neighbor_table(ss.non_empty_index, sr.non_empty_index, level)
    directory = ref.lists.build_level_directory(ss.non_empty_index, sr.non_empty_index, level)
    stencils = ref.lists.build_translation_stencils(directory)
    return SimpleNamespace(max_level=level, sorted_src=ss, sorted_recv=sr, neighbor_table=table,
                           directory=directory, stencils=stencils)


@pytest.mark.parametrize("n,m,level,seed", [(3000, 2500, 13, 5), (2000, 1800, 20, 6),
                                            (40000, 30000, 13, 7)])
def test_build_all_deep_levels(gpu, ref, n, m, level, seed):
    """The sparse build (levels above the occupancy-bitmap limit,
    lists._build_all_sparse) against the reference's own steps."""
    src, q, _ = generate(n, 1, "sphere", seed)
    _, _, recv = generate(1, m, "sphere", seed + 1000)
    want = _reference_sparse(ref, src, q, recv, level)
    got = gpu.build_all(src, q, recv, max_level=level, histogram_budget_bytes=8 ** level * 8)
    errors = compare_structures(got, want)
    assert not errors, "\n".join(errors)
    bs = got.build_seconds
    assert set(bs) >= {"sort_sources", "sort_receivers", "neighbor_table", "level_directory",
                       "stencils"} and all(v >= 0 for v in bs.values())


def test_index_embedding_edges_match_reference(gpu, ref):
    """Source records carry their index in the coordinates' exponent fields
    when every coordinate lies in [2^-8, 1) (bucket.cuh rec_embed): points on
    and around the range edges -- 0, -0.0, subnormals, 2^-8 and its neighbours,
    1 - ulp, exactly 1.0, values above 1 (clamped by the encoder) -- mixed
    with ordinary points must come out bit-identical to the reference."""
    rng = np.random.default_rng(5)
    n, m, L = 6000, 4000, 5
    src = rng.random((n, 3))
    recv = rng.random((m, 3))
    q = rng.normal(size=n)
    edge = np.array([0.0, -0.0, 5e-324, 2.0**-8, np.nextafter(2.0**-8, 0), np.nextafter(2.0**-8, 1),
                     2.0**-9, 0.5, np.nextafter(1.0, 0), 1.0, 1.5, 7.25, 2.0**-7, 0.999])
    k = 0
    for i in range(0, n, 7):  # every 7th source gets edge values on 1-3 axes
        for a in range(1 + i % 3):
            src[i, (a + i) % 3] = edge[k % edge.size]
            k += 1
    for i in range(0, m, 11):
        recv[i, i % 3] = edge[k % edge.size]
        k += 1
    want = ref.build_all(src, q, recv, max_level=L)
    for path in ("auto", "bucket_hist"):
        gpu._lib.set_sort_path(path)
        try:
            got = gpu.build_all(src, q, recv, max_level=L)
        finally:
            gpu._lib.set_sort_path("auto")
        errors = compare_structures(got, want)
        assert not errors, "\n".join(errors)
