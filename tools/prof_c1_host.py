"""Host-side profile of the c1 build call (cProfile over 500 synchronised
calls of build_all_device); prints the top functions by own time."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1301_1704_b200 as fb  # noqa: E402
from paper_1301_1704_b200.workloads import WORKLOADS, generate  # noqa: E402

wl = WORKLOADS["c1"]
s, q, r = generate(wl.n, wl.n, wl.dist, wl.seed)
dev = torch.device("cuda", 0)
s, q, r = (torch.from_numpy(a).to(dev) for a in (s, q, r))
for _ in range(20):
    st = fb.build_all_device(s, q, r, wl.level)
    st = None
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    st = fb.build_all_device(s, q, r, wl.level)
    st = None
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
