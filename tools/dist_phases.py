"""Per-phase wall time of the partitioned build (paper_1301_1704_b200.distributed)
on one rank per process: every device op / collective is synchronised and
timed, so the split between kernels, collectives and host glue shows.

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tools/dist_phases.py c2 5
(ranks may share one GPU: local_rank % device_count)"""
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1301_1704_b200 import distributed as D  # noqa: E402
from paper_1301_1704_b200.pseudosort import choose_max_level  # noqa: E402
from paper_1301_1704_b200.workloads import WORKLOADS, generate  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ws = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
T = collections.defaultdict(float)


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] += time.perf_counter() - t0
        return r
    return w


comm = D.TorchComm()
ops = D.DeviceOps()
for n in ("allreduce_sum", "all_to_all", "all_gather", "exchange_counts", "peer_tables",
          "peer_barrier"):
    setattr(comm, n, timed("comm." + n, getattr(comm, n)))
for n in ("part_histogram", "part_pack", "dist_sort", "dist_lists", "part_counts",
          "part_pack_peer"):
    setattr(ops, n, timed("ops." + n, getattr(ops, n)))
L = choose_max_level(wl.n * ws, 16)
src, q, recv = generate(wl.n, wl.n, wl.dist, wl.seed + rank)
src, q, recv = (torch.from_numpy(a).to(dev) for a in (src, q, recv))
for _ in range(2):
    D.build_all_distributed([(src, q, recv)], L, comm, ops=ops)
T.clear()
torch.cuda.synchronize()
dist.barrier()
t0 = time.perf_counter()
for _ in range(reps):
    sh = D.build_all_distributed([(src, q, recv)], L, comm, ops=ops)
    sh = None
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / reps
if rank == 0:
    out = {k: round(v / reps * 1e3, 3) for k, v in sorted(T.items())}
    out["total_ms"] = round(tot * 1e3, 3)
    out["glue_ms"] = round(tot * 1e3 - sum(out[k] for k in T), 3)
    print(json.dumps({"P": ws, "workload": wl.name, "L": L, **out}))
dist.destroy_process_group()
