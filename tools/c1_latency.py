"""c1 (2^16 + 2^16, L=4) per-call latency of build_all_device: wall clock per
synchronised call (with and without phase events) next to the device time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1301_1704_b200 as fb  # noqa: E402
from paper_1301_1704_b200.workloads import WORKLOADS, generate  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c1"]
s, q, r = generate(wl.n, wl.n, wl.dist, wl.seed)
dev = torch.device("cuda", 0)
s, q, r = (torch.from_numpy(a).to(dev) for a in (s, q, r))
for timing in (True, False):
    for _ in range(20):
        st = fb.build_all_device(s, q, r, wl.level, timing=timing)
    torch.cuda.synchronize()
    reps = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        st = fb.build_all_device(s, q, r, wl.level, timing=timing)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    print(f"timing={timing}: {wall * 1e3:.3f} ms per call (wall), {e0.elapsed_time(e1) / reps:.3f} ms "
          f"(events), device phases {sum(float(v) for k, v in st.build_seconds.items() if k in ('sort_sources', 'level_directory', 'stencils')) * 1e3 if timing else 0:.3f} ms")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    st = fb.build_all_device(s, q, r, wl.level, timing=True)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
