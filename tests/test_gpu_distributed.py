"""Partitioned (multi-GPU) build, all ranks simulated on one GPU (SimComm):
the concatenation of the rank shards equals the single-GPU build bit for
bit."""

import numpy as np
import pytest
import torch

from paper_1301_1704_b200.workloads import generate
from tests.parity import compare_structures

pytestmark = pytest.mark.gpu


def _shards(arr, p):
    cut = np.linspace(0, arr.shape[0], p + 1).astype(int)
    return [arr[cut[i]:cut[i + 1]] for i in range(p)]


@pytest.mark.parametrize("p,n,m,level,dist,charges", [
    (2, 20000, 15000, 4, "uniform", True),
    (3, 30000, 30000, 5, "uniform", True),
    (4, 2**17, 2**17, 6, "uniform", True),
    (4, 20000, 25000, 6, "sphere", True),
    (8, 50000, 40000, 5, "sphere", False),
    (2, 5000, 0, 3, "uniform", True),
    (3, 0, 4000, 3, "uniform", True),
])
@pytest.mark.parametrize("exchange", ["a2a", "peer"])
def test_partitioned_build_matches_single(gpu, p, n, m, level, dist, charges, exchange):
    """a2a: pack into send buffers + all-to-all; peer: the fused pack that
    stores every point straight into its destination rank's arrays."""
    from paper_1301_1704_b200 import distributed as D

    src, q, _ = generate(n, 1, dist, 17)
    _, _, recv = generate(1, m, dist, 18)
    if not charges:
        q = None
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    shards = [(t(s), t(qq) if q is not None else None, t(r)) for s, qq, r in
              zip(_shards(src, p), _shards(q if q is not None else np.zeros(n), p),
                  _shards(recv, p))]
    out = D.build_all_distributed(shards, level, D.SimComm(p), exchange=exchange)
    got = D.concat_shards(out)
    want = gpu.build_all(t(src), t(q) if q is not None else None, t(recv), max_level=level)
    errors = compare_structures(got.to_numpy(), want.to_numpy())
    assert not errors, "\n".join(errors)


def test_partition_is_balanced_and_contiguous(gpu):
    from paper_1301_1704_b200 import distributed as D

    src, q, recv = generate(2**16, 2**16, "uniform", 5)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    shards = [(t(s), t(qq), t(r)) for s, qq, r in
              zip(_shards(src, 4), _shards(q, 4), _shards(recv, 4))]
    out = D.build_all_distributed(shards, 6, D.SimComm(4))
    counts = [int(o.sorted_src.points.shape[0] + o.sorted_recv.points.shape[0]) for o in out]
    assert sum(counts) == 2**17
    assert max(counts) <= 1.05 * (2**17 / 4)
    wins = [o.key_window for o in out]
    assert wins[0][0] == 0 and wins[-1][1] == 8**6
    assert all(wins[i][1] == wins[i + 1][0] for i in range(3))


def test_peer_exchange_two_processes_over_ipc(gpu):
    """Two ranks in two processes sharing the GPU: the fused pack stores into
    the other process's receive arrays through CUDA IPC; the concatenated
    shards equal the single-GPU build for both exchanges."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", "29657",
         os.path.join(root, "tools", "peer_ipc_check.py")],
        cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "peer OK" in out.stdout and "a2a OK" in out.stdout
