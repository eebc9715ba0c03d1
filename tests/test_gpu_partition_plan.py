"""Receiver-load partition plan: choose_partition with
the per-level loads, prefix and cuts on the device gives plans identical to
the reference's (partition.py:74-127, run from oracle/_ref as the checker)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inputs(ref, n, L, seed, skew):
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 3)) ** skew
    boxes = ref.box_indices_of_points(pts, L)
    return np.unique(boxes, return_counts=True)


def _same(a, b):
    assert (a.nodes, a.units_per_node, a.partition_level, a.critical_level, a.balanced) == \
        (b.nodes, b.units_per_node, b.partition_level, b.critical_level, b.balanced)
    assert a.load_ratio == b.load_ratio
    assert a.box_proc_id.dtype == b.box_proc_id.dtype
    assert np.array_equal(a.box_proc_id, b.box_proc_id)
    assert np.array_equal(a.unit_ranges, b.unit_ranges)


@pytest.mark.parametrize("n,L,seed,skew,nodes,upn,tol", [
    (20000, 5, 0, 1.0, 2, 1, 0.2), (20000, 5, 1, 3.0, 4, 2, 0.2), (50000, 6, 2, 2.0, 8, 1, 0.05),
    (3000, 4, 3, 1.5, 3, 2, 0.2), (100000, 7, 4, 4.0, 8, 4, 0.01), (500, 3, 5, 1.0, 1, 1, 0.2)])
def test_plans_identical(gpu, ref, n, L, seed, skew, nodes, upn, tol):
    uniq, counts = _inputs(ref, n, L, seed, skew)
    _same(gpu.choose_partition(uniq, counts, L, nodes, upn, tol),
          ref.choose_partition(uniq, counts, L, nodes, upn, tol))


def test_errors_and_round_trip(gpu, ref, tmp_path):
    from paper_1301_1704_b200 import partition as P

    uniq, counts = _inputs(ref, 64, 2, 6, 1.0)
    with pytest.raises(gpu.DomainError):
        gpu.choose_partition(uniq, counts, 2, 0, 1)
    with pytest.raises(gpu.InfeasiblePartitionError):
        gpu.choose_partition(uniq[:3], counts[:3], 2, 4, 1)
    plan = gpu.choose_partition(uniq, counts, 2, 2, 2)
    P.dump_plan(plan, tmp_path / "p.fmms")
    ref.partition.dump_plan(ref.choose_partition(uniq, counts, 2, 2, 2), tmp_path / "r.fmms")
    assert (tmp_path / "p.fmms").read_bytes() == (tmp_path / "r.fmms").read_bytes()
    _same(P.load_plan(tmp_path / "p.fmms"), ref.partition.load_plan(tmp_path / "r.fmms"))
