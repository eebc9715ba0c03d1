"""Two processes on one GPU: the fused pack + exchange over CUDA IPC (gloo for
the control plane) must give shards whose concatenation equals the
single-GPU build (run under torchrun --nproc-per-node 2)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1301_1704_b200 as fb  # noqa: E402
from paper_1301_1704_b200 import distributed as D  # noqa: E402
from paper_1301_1704_b200.workloads import generate  # noqa: E402
from tests.parity import compare_structures  # noqa: E402

dist.init_process_group("gloo")
rank, ws = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n, m, L = 60000, 50000, 5
src, q, _ = generate(n, 1, "sphere", 5)
_, _, recv = generate(1, m, "sphere", 6)
cut = lambda a: np.array_split(a, ws)[rank]  # noqa: E731
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
shard = [(t(cut(src)), t(cut(q)), t(cut(recv)))]
for exchange in ("peer", "a2a"):
    out = D.build_all_distributed(shard, L, D.TorchComm(), exchange=exchange)[0].to_numpy()
    allo = [None] * ws
    dist.all_gather_object(allo, out)
    if rank == 0:
        got = D.concat_shards(allo)
        want = fb.build_all(src, q, recv, max_level=L)
        errors = compare_structures(got, want)
        print(exchange, "OK" if not errors else errors[:3], flush=True)
        assert not errors
dist.barrier()
dist.destroy_process_group()
