"""c4 as bench.py runs it (two perturbed point sets alternating), with sort paths and phases."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1301_1704_b200 as fb
from paper_1301_1704_b200.workloads import WORKLOADS, generate, perturb
wl = WORKLOADS["c4"]
src, q, recv = generate(wl.n, wl.n, wl.dist, wl.seed)
rng = np.random.default_rng(123)
pert = [(torch.from_numpy(perturb(src, rng)).cuda(), torch.from_numpy(perturb(recv, rng)).cuda()) for _ in range(2)]
qd = torch.from_numpy(q).cuda()
for k in range(6):
    s_in, r_in = pert[k % 2]
    st = fb.build_all_device(s_in, qd, r_in, wl.level)
    print(k, {kk: round(v * 1e3, 3) for kk, v in st.build_seconds.items()}, st.n_launches, st.sort_path, flush=True)
    st = None
