"""The CPU oracle (oracle/, test infrastructure) is pinned to the reference:
bit-exact against the committed golden vectors, and against the live
reference when oracle/_ref is importable."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1301_1704_b200.workloads import generate
from tests import golden_io as gio
from tests.parity import compare_structures


@pytest.mark.parametrize("name", sorted(gio.small_cases()))
def test_oracle_matches_golden_small(name):
    case = gio.small_cases()[name]
    src, q, recv, L = gio.case_inputs(case)
    st = orc.build_all(src, q, recv, L)
    errors = gio.compare_flat(gio.flatten(st), gio.expected_outputs(case))
    assert not errors, errors


@pytest.mark.parametrize("name", ["c1", "u20_L3"])
def test_oracle_matches_golden_hashes(name):
    spec = gio.hashes()[name]
    src, q, recv, L = gio.large_inputs(spec)
    st = orc.build_all(src, q, recv, L)
    got = {k: gio.sha(v) for k, v in gio.flatten(st).items()}
    assert got == spec["arrays"]


def test_oracle_encode_edges():
    e = gio.encode_edges()
    for L in (0, 1, 3, 7, 9, 20):
        assert np.array_equal(orc.encode(e["pts"], L), e[f"L{L}"]), L


def test_oracle_matches_live_reference(ref):
    for n, m, L, dist, seed in [(2000, 1500, 4, "uniform", 41), (1500, 2500, 6, "sphere", 42),
                                (300, 300, 2, "uniform", 43)]:
        src, q, _ = generate(n, 1, dist, seed)
        _, _, recv = generate(1, m, dist, seed + 1)
        want = ref.build_all(src, q, recv, max_level=L)
        got = orc.build_all(src, q, recv, L)
        errors = compare_structures(got, want)
        assert not errors, errors


def test_generate_matches_reference_cli(ref):
    from fmmkit.cli import RunSpec, generate as ref_generate

    for dist in ("uniform", "sphere"):
        a = generate(1000, 700, dist, 5)
        b = ref_generate(RunSpec(n_sources=1000, n_receivers=700, dist=dist, seed=5))
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("name", sorted(gio.small_cases()))
def test_oracle_near_field_matches_golden(name):
    """orc_near_field (C restatement of _ckernels.pyx:290-323) on the
    reference's own sorted outputs reproduces the reference's phi."""
    case = gio.small_cases()[name]
    nf = gio.nearfield()
    out = gio.expected_outputs(case)
    q = out.get("src.charges", np.ones(out["src.points"].shape[0]))
    phi = orc.near_field(out["src.points"], q, out["src.bookmarks"], out["neighbor_bookmark"],
                         out["neighbor_list"], out["recv.points"], out["recv.bookmarks"])
    assert np.array_equal(phi.view(np.uint64), nf[f"{name}/phi"].view(np.uint64))


def test_oracle_direct_matches_golden():
    nf = gio.nearfield()
    for name in ("u3_L3", "s5_L5"):
        src, q, recv, _ = gio.case_inputs(gio.small_cases()[name])
        assert np.array_equal(orc.direct(src, q, recv).view(np.uint64),
                              nf[f"{name}/direct"].view(np.uint64))
    src, q, recv = nf["clustered/in.src"], nf["clustered/in.q"], nf["clustered/in.recv"]
    assert np.array_equal(orc.direct(src, q, recv).view(np.uint64),
                          nf["clustered/direct"].view(np.uint64))
