"""Full-size workloads (BASELINE configs c2/c3): size-independent properties
on the device outputs (the oracle would take minutes at this size)."""

import numpy as np
import pytest
import torch

from paper_1301_1704_b200.workloads import WORKLOADS, generate

pytestmark = pytest.mark.gpu


def _take(u64, idx):
    return u64.view(torch.int64)[idx].view(torch.uint64)


def _check(st, src, recv, L):
    dev = st.sorted_src.points.device
    for ps, pts in ((st.sorted_src, src), (st.sorted_recv, recv)):
        n = pts.shape[0]
        perm = ps.permutation
        # permutation is a permutation and the gather is exact
        assert torch.equal(torch.sort(perm).values, torch.arange(n, device=dev))
        assert torch.equal(ps.points, pts[perm])
        keys = ps.boxes.view(torch.int64)
        assert bool((keys[1:] >= keys[:-1]).all())  # grouped ascending
        # stable: equal keys keep input order
        same = keys[1:] == keys[:-1]
        assert bool((perm[1:][same] > perm[:-1][same]).all())
        bm = ps.bookmarks
        ne = ps.non_empty_index.view(torch.int64)
        assert int(bm[0]) == 0 and int(bm[-1]) == n
        assert bool((ne[1:] > ne[:-1]).all())
        assert torch.equal(keys[bm[:-1]], ne)
    # E2 rows: ascending ranks, neighbours within one box step
    nb, nl = st.neighbor_table.neighbor_bookmark, st.neighbor_table.neighbor_list
    assert int(nb[-1]) == nl.numel()
    rows = torch.repeat_interleave(torch.arange(nb.numel() - 1, device=dev), nb[1:] - nb[:-1])
    within = nl[1:] > nl[:-1]
    assert bool(within[(rows[1:] == rows[:-1])].all())
    from paper_1301_1704_b200 import kernels as K

    sk = st.sorted_src.non_empty_index
    rk = st.sorted_recv.non_empty_index
    sc = torch.stack([t.view(torch.int64) for t in K.deinterleave_indices(_take(sk, nl))], 1)
    rc = torch.stack([t.view(torch.int64) for t in K.deinterleave_indices(_take(rk, rows))], 1)
    assert int((sc - rc).abs().max()) <= 1
    # E4 at every level: offset codes decode to the coordinate difference and
    # the stencil excludes the own neighbourhood
    for l in range(2, L + 1):
        bm, ranks, codes = st.stencils.bookmark[l], st.stencils.ranks[l], st.stencils.codes[l]
        r = torch.repeat_interleave(torch.arange(bm.numel() - 1, device=dev), bm[1:] - bm[:-1])
        s_keys = _take(st.directory.src_boxes[l], ranks)
        r_keys = _take(st.directory.recv_boxes[l], r)
        sc = torch.stack([t.view(torch.int64) for t in K.deinterleave_indices(s_keys)], 1)
        rc = torch.stack([t.view(torch.int64) for t in K.deinterleave_indices(r_keys)], 1)
        d = sc - rc
        assert int(d.abs().amax(1).min()) >= 2 and int(d.abs().max()) <= 3
        code = (d[:, 0] + 3) + 7 * (d[:, 1] + 3) + 49 * (d[:, 2] + 3)
        assert torch.equal(code.to(torch.int16), codes)
        assert bool(((sc >> 1) - (rc >> 1)).abs().amax(1).le(1).all())


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_size_properties(gpu, name):
    wl = WORKLOADS[name]
    src, q, recv = generate(wl.n, wl.n, wl.dist, wl.seed)
    dev = torch.device("cuda", 0)
    s, qq, r = (torch.from_numpy(a).to(dev) for a in (src, q, recv))
    st = gpu.build_all_device(s, qq, r, wl.level)
    _check(st, s, r, wl.level)
    assert torch.equal(st.sorted_src.charges, qq[st.sorted_src.permutation])


def _flat(st):
    out = {}
    for side in ("sorted_src", "sorted_recv"):
        ps = getattr(st, side)
        for f in ("points", "charges", "permutation", "bookmarks", "non_empty_index", "boxes"):
            v = getattr(ps, f)
            if v is not None:
                out[f"{side}.{f}"] = v
    out["nb"] = st.neighbor_table.neighbor_bookmark
    out["nl"] = st.neighbor_table.neighbor_list
    for l, v in st.directory.src_boxes.items():
        out[f"ds{l}"] = v
    for l, v in st.directory.recv_boxes.items():
        out[f"dr{l}"] = v
    for l in st.stencils.ranks:
        out[f"sb{l}"] = st.stencils.bookmark[l]
        out[f"sr{l}"] = st.stencils.ranks[l]
        out[f"sc{l}"] = st.stencils.codes[l]
    return out


def test_wide_index_embedding_matches_onesweep(gpu):
    """n + m = 2^26 + 2^20: the combined index needs 27 bits, so the source
    records embed it with 2-bit exponents (coordinates in [2^-4, 1), the rest
    take the side store) -- every output array equals the Onesweep path's,
    which never builds records."""
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(17)
    n, m, L = 2**26, 2**20, 7
    src = torch.rand((n, 3), generator=g, device=dev, dtype=torch.float64)
    src[::97, 1] *= 0.05  # plenty of coordinates below 2^-4 (side-store escapes)
    recv = torch.rand((m, 3), generator=g, device=dev, dtype=torch.float64)
    q = torch.randn(n, generator=g, device=dev, dtype=torch.float64)
    a = _flat(gpu.build_all_device(src, q, recv, L))
    gpu._lib.set_sort_path("onesweep")
    try:
        b = _flat(gpu.build_all_device(src, q, recv, L))
    finally:
        gpu._lib.set_sort_path("auto")
    assert a.keys() == b.keys()
    for k in a:
        assert a[k].dtype == b[k].dtype and a[k].shape == b[k].shape, k
        assert torch.equal(a[k].view(torch.uint8), b[k].view(torch.uint8)), k


def test_phase_trace_and_partitioned_timer(gpu):
    """The FMMB_TRACE timeline API answers (empty when the handle was created
    without it) and the partitioned build's PhaseTimer reports every phase."""
    from paper_1301_1704_b200 import distributed as D

    dev = torch.device("cuda", 0)
    assert isinstance(gpu._lib.trace(dev), list)
    src, q, recv = (torch.from_numpy(a).to(dev) for a in generate(20000, 15000, "uniform", 3))
    comm = D.SimComm(2)
    half = (src.shape[0] // 2, recv.shape[0] // 2)
    shards = [(src[:half[0]], q[:half[0]], recv[:half[1]]),
              (src[half[0]:], q[half[0]:], recv[half[1]:])]
    timer = D.PhaseTimer()
    out = D.build_all_distributed(shards, 5, comm, timer=timer)
    ph = timer.ms()
    for k in ("partition (histogram, all-reduce, cut)", "pack", "exchange (all-to-all)",
              "local sort", "occupancy all-reduce", "owned lists", "offsets (all-gather)"):
        assert k in ph and ph[k] >= 0.0, k
    assert len(out) == 2 and sum(int(s.exchanged["sent_bytes"]) for s in out) > 0
