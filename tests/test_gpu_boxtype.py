"""Box-type classification on the device equals the
reference's classify (boxtype.py:103-144, run from oracle/_ref as the
checker) for the scenarios of the reference's test_boxtype.py and for
load-balanced plans from its choose_partition."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _plan(ref, box_proc_id, nodes, upn, l_par, l_crit=None):
    from fmmkit.partition import PartitionPlan

    bp = np.asarray(box_proc_id, dtype=np.int32)
    bounds = np.searchsorted(bp, np.arange(nodes * upn + 1), side="left")
    return PartitionPlan(nodes=nodes, units_per_node=upn, partition_level=l_par,
                         critical_level=l_crit if l_crit is not None else max(l_par - 1, 2),
                         box_proc_id=bp, unit_ranges=np.stack([bounds[:-1], bounds[1:]], 1),
                         balanced=True, load_ratio=1.0)


def _levels_from_points(pts, L):
    from fmmkit import box_indices_of_points

    uniq = np.unique(box_indices_of_points(pts, L))
    levels = {L: uniq}
    for l in range(L - 1, 1, -1):
        levels[l] = np.unique(levels[l + 1] >> np.uint64(3))
    return levels, uniq


def _check(gpu, ref, node, levels, plan):
    want = ref.classify(node, levels, plan)
    got = gpu.classify(node, levels, plan)
    for l in levels:
        assert got.types[l].dtype == np.int8
        assert np.array_equal(got.types[l], want.types[l]), (node, l)


def test_reference_scenarios(gpu, ref):
    dense = {l: np.arange(8 ** l, dtype=np.uint64) for l in range(2, 5)}
    _check(gpu, ref, 0, dense, _plan(ref, np.zeros(64), 1, 1, 2))
    bp = np.zeros(512, dtype=np.int32)
    bp[300:] = 1
    for node in (0, 1):
        _check(gpu, ref, node, {l: dense[l] for l in (2, 3)}, _plan(ref, bp, 2, 1, 3))


@pytest.mark.parametrize("nodes,upn,seed,L", [(2, 1, 0, 4), (4, 1, 1, 4), (4, 2, 2, 5),
                                              (3, 2, 3, 5), (8, 1, 4, 6)])
def test_matches_reference_on_balanced_plans(gpu, ref, nodes, upn, seed, L):
    rng = np.random.default_rng(seed)
    pts = rng.random((20000, 3)) ** (1 + 0.5 * rng.random())
    levels, uniq = _levels_from_points(pts, L)
    counts = np.ones(uniq.shape[0], dtype=np.int64)
    plan = ref.choose_partition(uniq, counts, L, nodes, upn)
    for node in range(nodes):
        _check(gpu, ref, node, levels, plan)


def test_device_inputs_and_errors(gpu, ref):
    bp = np.repeat(np.arange(4, dtype=np.int32), 128)
    plan = _plan(ref, bp, 4, 1, 3, 2)
    dense = {l: np.arange(8 ** l, dtype=np.uint64) for l in (2, 3, 4)}
    want = ref.classify(2, dense, plan)
    dev = {l: torch.from_numpy(v.astype(np.int64)).cuda().to(torch.uint64) for l, v in dense.items()}
    got = gpu.classify(2, dev, plan)
    for l in dense:
        assert got.types[l].is_cuda
        assert np.array_equal(got.types[l].cpu().numpy(), want.types[l])
    with pytest.raises(gpu.DomainError):
        gpu.classify(0, {1: np.arange(8, dtype=np.uint64)}, plan)


def test_dump_load_typed(gpu, ref, tmp_path):
    bp = np.zeros(512, dtype=np.int32)
    bp[300:] = 1
    plan = _plan(ref, bp, 2, 1, 3)
    dense = {l: np.arange(8 ** l, dtype=np.uint64) for l in (2, 3)}
    typed = gpu.classify(1, dense, plan)
    from paper_1301_1704_b200 import boxtype as bt

    bt.dump_typed(typed, tmp_path / "t.fmms")
    ref.boxtype.dump_typed(ref.classify(1, dense, plan), tmp_path / "r.fmms")
    assert (tmp_path / "t.fmms").read_bytes() == (tmp_path / "r.fmms").read_bytes()
    back = bt.load_typed(tmp_path / "t.fmms", plan)
    for l in dense:
        assert np.array_equal(back.types[l], typed.types[l])
