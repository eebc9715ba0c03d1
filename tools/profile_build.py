"""One warm build then N profiled builds of a workload (for ncu)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1301_1704_b200 as fb
from paper_1301_1704_b200.workloads import WORKLOADS, generate
wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
fb._lib.set_sort_path(os.environ.get('FMMB_SORT_PATH', 'auto'))
src, q, recv = generate(wl.n, wl.n, wl.dist, wl.seed)
src, q, recv = (torch.from_numpy(a).cuda() for a in (src, q, recv))
st = fb.build_all_device(src, q, recv, wl.level); st = None
torch.cuda.synchronize()
for _ in range(reps):
    st = fb.build_all_device(src, q, recv, wl.level)
    print({k: round(v * 1e3, 3) for k, v in st.build_seconds.items()}, st.n_launches, st.sort_path)
    st = None
torch.cuda.synchronize()
