"""Near-field consumer on the device: bit-identical to
the reference's compiled near_field / direct_potentials
(_ckernels.pyx:290-350), checked against the committed golden vectors
(tests/golden/make_golden_nearfield.py, generated from the unmodified
reference) and against the C restatement (oracle/fmm_oracle.c)."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_1301_1704_b200.workloads import generate
from tests import golden_io as gio

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nf():
    return gio.nearfield()


def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.dtype == b.dtype == np.float64 and a.shape == b.shape
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("name", sorted(gio.small_cases()))
def test_small_cases_bitwise(gpu, nf, name):
    src, q, recv, L = gio.case_inputs(gio.small_cases()[name])
    st = gpu.build_all(src, q, recv, max_level=L)
    _eq(gpu.near_field_potentials(st), nf[f"{name}/phi"])


@pytest.mark.parametrize("name", ["u3_L3", "s5_L5"])
def test_direct_sum_bitwise(gpu, nf, name):
    src, q, recv, _ = gio.case_inputs(gio.small_cases()[name])
    _eq(gpu.direct_sum(src, q, recv), nf[f"{name}/direct"])


def test_clustered_and_coincident(gpu, nf):
    """Hundreds of points per box (receiver groups > 32 lanes), duplicated
    points (dist == 0 pairs skipped), a box-free level-0 build."""
    src, q, recv = nf["clustered/in.src"], nf["clustered/in.q"], nf["clustered/in.recv"]
    for L in (0, 2):
        st = gpu.build_all(src, q, recv, max_level=L)
        _eq(gpu.near_field_potentials(st), nf[f"clustered/L{L}/phi"])
    _eq(gpu.direct_sum(src, q, recv), nf["clustered/direct"])


def test_single_box_near_equals_direct(gpu):
    """test_backends.py:112-126: at max_level=0 the near field is the direct
    sum over the sorted arrays, bit for bit."""
    src, q, recv = generate(400, 400, "uniform", 11)
    st = gpu.build_all(src, q, recv, max_level=0)
    near = gpu.near_field_potentials(st)
    ref = gpu.direct_sum(st.sorted_src.points, st.sorted_src.charges, st.sorted_recv.points)
    _eq(near, ref)


@pytest.mark.parametrize("case", ["c1", "u20_L7", "s20_L9", "u20_L3"])
def test_large_cases_sha(gpu, case):
    """Full near field of the larger golden cases, device-built structures
    consumed in place; sha256 of phi equals the reference's."""
    src, q, recv, L = gio.large_inputs(gio.hashes()[case])
    dev = torch.device("cuda", 0)
    st = gpu.build_all_device(torch.from_numpy(src).to(dev),
                              torch.from_numpy(q).to(dev) if q is not None else None,
                              torch.from_numpy(recv).to(dev), L)
    phi = gpu.near_field_potentials(st)
    assert isinstance(phi, torch.Tensor) and phi.is_cuda
    assert gio.sha(phi.cpu().numpy()) == gio.nearfield_hashes()[case]


def test_matches_c_oracle_random_lists(gpu):
    """Synthetic neighbour lists wider than a warp (40 segments, repeats,
    empty boxes) against the C restatement."""
    rng = np.random.default_rng(5)
    ks, kr = 50, 30
    sizes = rng.integers(0, 12, ks)
    sbm = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ns = int(sbm[-1])
    spts = rng.random((ns, 3))
    q = rng.normal(size=ns)
    rsz = rng.integers(0, 40, kr)
    rbm = np.concatenate([[0], np.cumsum(rsz)]).astype(np.int64)
    nr = int(rbm[-1])
    rpts = rng.random((nr, 3))
    rpts[:5] = spts[:5]  # coincident pairs
    nseg = rng.integers(0, 41, kr)
    nbm = np.concatenate([[0], np.cumsum(nseg)]).astype(np.int64)
    nlist = rng.integers(0, ks, int(nbm[-1])).astype(np.int64)
    want = orc.near_field(spts, q, sbm, nbm, nlist, rpts, rbm)
    k = gpu.kernels
    got = k.near_field(spts[:, 0], spts[:, 1], spts[:, 2], q, sbm, nbm, nlist,
                       rpts[:, 0], rpts[:, 1], rpts[:, 2], rbm)
    _eq(got, want)
    # device inputs -> device output, strided columns
    d = torch.device("cuda", 0)
    ts, tr = torch.from_numpy(spts).to(d), torch.from_numpy(rpts).to(d)
    got_d = k.near_field(ts[:, 0], ts[:, 1], ts[:, 2], torch.from_numpy(q).to(d),
                         torch.from_numpy(sbm).to(d), torch.from_numpy(nbm).to(d),
                         torch.from_numpy(nlist).to(d), tr[:, 0], tr[:, 1], tr[:, 2],
                         torch.from_numpy(rbm).to(d))
    assert got_d.is_cuda
    _eq(got_d.cpu().numpy(), want)


def test_empty_and_errors(gpu):
    k = gpu.kernels
    e = np.empty(0)
    z = np.zeros(1, dtype=np.int64)
    assert k.near_field(e, e, e, e, z, z, np.empty(0, np.int64), e, e, e, z).shape == (0,)
    phi = k.near_field(e, e, e, e, z, np.zeros(3, np.int64), np.empty(0, np.int64),
                       np.ones(4), np.ones(4), np.ones(4), np.array([0, 2, 4]))
    assert np.array_equal(phi, np.zeros(4))
    with pytest.raises(gpu.DomainError):
        k.near_field(e, e, e, e, z, np.zeros(2, np.int64), np.empty(0, np.int64), e, e, e, z)
    assert k.direct_potentials(e, e, e, e, np.ones(3), np.ones(3), np.ones(3)).tolist() == [0.0] * 3
