"""Device-resident near-field pass on a built workload:
CUDA-event time of kernels.near_field over the structures build_all_device
returned, interactions/s and FP64 issue rate.

    python tools/bench_nearfield.py [c1|c2|c3|c4] [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1301_1704_b200 as fb  # noqa: E402
from paper_1301_1704_b200.workloads import WORKLOADS, generate  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
src, q, recv = generate(wl.n, wl.n, wl.dist, wl.seed)
src, q, recv = (torch.from_numpy(a).to(dev) for a in (src, q, recv))
st = fb.build_all_device(src, q, recv, wl.level)
ss, sr, nt = st.sorted_src, st.sorted_recv, st.neighbor_table
sizes = torch.diff(ss.bookmarks)
cs = torch.nn.functional.pad(torch.cumsum(sizes[nt.neighbor_list], 0), (1, 0))
S = cs[nt.neighbor_bookmark[1:]] - cs[nt.neighbor_bookmark[:-1]]
R = torch.diff(sr.bookmarks)
inter = int((R * S).sum())
phi = fb.near_field_potentials(st)  # warm
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    phi = fb.near_field_potentials(st)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e-3)
t = sorted(ts)[len(ts) // 2]
print(json.dumps({"workload": wl.name, "interactions": inter, "ms": t * 1e3,
                  "interactions_per_s": inter / t, "receivers": int(sr.points.shape[0]),
                  "all_ms": [x * 1e3 for x in ts]}))
