"""Multi-process (gloo, world size 2 and 3) tests of the partitioned build's
host side: the TorchComm collectives and the driver's partition, exchange and
offset logic, with the per-rank device steps restated on the CPU oracle
(tests/dist_oracle_ops.py).  The concatenated shards must equal the
single-node oracle build bit for bit."""

import os
import pickle
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, ws, port):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    return dist


def _comm_worker(rank, ws, port, outdir):
    sys.path.insert(0, ROOT)
    dist = _init(rank, ws, port)
    from paper_1301_1704_b200.distributed import TorchComm

    c = TorchComm()
    x = [torch.arange(3 + rank, dtype=torch.float64).reshape(-1, 1).repeat(1, 3) + 10 * rank]
    chunks = [[x[0][:1 + d] for d in range(ws)]]
    got = c.all_to_all(chunks)[0]
    bits = torch.tensor([1 << rank, -(1 << 63) if rank == ws - 1 else 0], dtype=torch.int64)
    red = c.allreduce_sum([bits])[0]
    gat = c.all_gather([torch.tensor([rank, 2 * rank], dtype=torch.int64)])[0]
    with open(os.path.join(outdir, f"{rank}.pkl"), "wb") as f:
        pickle.dump(([g.numpy() for g in got], red.numpy(), [g.numpy() for g in gat]), f)
    dist.destroy_process_group()


def test_torchcomm_gloo_collectives():
    ws = 3
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_comm_worker, args=(ws, _port(), d), nprocs=ws)
        res = [pickle.load(open(os.path.join(d, f"{r}.pkl"), "rb")) for r in range(ws)]
    for r, (got, red, gat) in enumerate(res):
        for s in range(ws):  # rank s sent its first 1 + r rows to rank r
            want = np.arange(3 + s, dtype=np.float64)[: 1 + r, None].repeat(3, 1) + 10 * s
            assert np.array_equal(got[s], want)
        assert red[0] == sum(1 << k for k in range(ws))  # disjoint bits: SUM == OR
        assert red[1] == np.int64(-(1 << 63))
        assert [list(g) for g in gat] == [[k, 2 * k] for k in range(ws)]


def _build_worker(rank, ws, port, outdir, n, m, level, dist_name):
    sys.path.insert(0, ROOT)
    dist = _init(rank, ws, port)
    from paper_1301_1704_b200.distributed import TorchComm, build_all_distributed
    from paper_1301_1704_b200.workloads import generate
    from tests.dist_oracle_ops import OracleOps

    src, q, recv = generate(n, m, dist_name, 3)
    cs = np.linspace(0, n, ws + 1).astype(int)
    cr = np.linspace(0, m, ws + 1).astype(int)
    t = torch.from_numpy
    shard = (t(src[cs[rank]:cs[rank + 1]].copy()), t(q[cs[rank]:cs[rank + 1]].copy()),
             t(recv[cr[rank]:cr[rank + 1]].copy()))
    (out,) = build_all_distributed([shard], level, TorchComm(), ops=OracleOps())
    with open(os.path.join(outdir, f"{rank}.pkl"), "wb") as f:
        pickle.dump(out.to_numpy(), f)
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,n,m,level,dist_name", [
    (2, 3000, 2500, 4, "uniform"),
    (3, 4000, 4000, 5, "sphere"),
])
def test_partitioned_driver_gloo_matches_oracle(ws, n, m, level, dist_name):
    sys.path.insert(0, ROOT)
    from oracle import oracle as orc
    from paper_1301_1704_b200.distributed import concat_shards
    from paper_1301_1704_b200.workloads import generate

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_build_worker, args=(ws, _port(), d, n, m, level, dist_name), nprocs=ws)
        shards = [pickle.load(open(os.path.join(d, f"{r}.pkl"), "rb")) for r in range(ws)]
    got = concat_shards(shards)
    src, q, recv = generate(n, m, dist_name, 3)
    want = orc.build_all(src, q, recv, level)

    def same(a, b, what):
        a = a.numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
        b = np.asarray(b)
        assert a.shape == b.shape and np.array_equal(a.astype(b.dtype), b), what

    for side in ("sorted_src", "sorted_recv"):
        for f in ("points", "permutation", "bookmarks", "non_empty_index", "boxes"):
            same(getattr(getattr(got, side), f), getattr(getattr(want, side), f), f"{side}.{f}")
    same(got.sorted_src.charges, want.sorted_src.charges, "charges")
    same(got.neighbor_table.neighbor_bookmark, want.neighbor_table.neighbor_bookmark, "nbm")
    same(got.neighbor_table.neighbor_list, want.neighbor_table.neighbor_list, "nlist")
    for l in range(2, level + 1):
        same(got.directory.src_boxes[l], want.directory.src_boxes[l], f"dsrc{l}")
        same(got.directory.recv_boxes[l], want.directory.recv_boxes[l], f"drecv{l}")
        same(got.stencils.bookmark[l], want.stencils.bookmark[l], f"sbm{l}")
        same(got.stencils.ranks[l], want.stencils.ranks[l], f"srk{l}")
        same(got.stencils.codes[l], want.stencils.codes[l], f"scd{l}")
    # the partition moved points between ranks and every rank owns a range
    assert sum(s.exchanged["sent_points"] for s in shards) > 0
    assert shards[0].key_window[0] == 0 and shards[-1].key_window[1] == 8 ** level


def test_cut_bins_balanced_and_monotone():
    sys.path.insert(0, ROOT)
    from paper_1301_1704_b200.distributed import cut_bins, key_windows

    rng = np.random.default_rng(0)
    h = torch.from_numpy(rng.integers(0, 50, size=4096))
    for p in (1, 2, 3, 8):
        br = cut_bins(h, p)
        assert bool((br[1:] >= br[:-1]).all()) and int(br.min()) == 0 and int(br.max()) == p - 1
        loads = [int(h[br == g].sum()) for g in range(p)]
        assert max(loads) - min(loads) <= 2 * int(h.max())
        w = key_windows(br, p, 4, 12)
        assert w[0][0] == 0 and w[-1][1] == 8**4
        assert all(w[g][1] == w[g + 1][0] for g in range(p - 1))
    assert int(cut_bins(torch.zeros(16, dtype=torch.int64), 4).max()) == 0
