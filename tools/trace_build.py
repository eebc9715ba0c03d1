"""Phase timeline of the fused build on both streams (FMMB_TRACE=1 events).

    FMMB_TRACE=1 python tools/trace_build.py c2 [reps]

Prints, for the last of `reps` device-resident builds, every phase boundary
in ms since the build's start event, tagged with the stream that ran it
(s = caller's stream, side = the sort stream).  CUDA events only; no
profiler.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FMMB_TRACE", "1")

import torch  # noqa: E402

import paper_1301_1704_b200 as fb  # noqa: E402
from paper_1301_1704_b200.workloads import WORKLOADS, c4_step_inputs, generate  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = WORKLOADS[name]
if name == "c4":
    s, q, r = c4_step_inputs(wl.n, wl.seed, 1)
else:
    s, q, r = generate(wl.n, wl.n, wl.dist, wl.seed)
dev = torch.device("cuda", 0)
s, q, r = (torch.from_numpy(a).to(dev) for a in (s, q, r))
for _ in range(reps):
    st = fb.build_all_device(s, q, r, wl.level)
    st = None
torch.cuda.synchronize()
tl = fb._lib.trace(dev)
print(f"{name}: last of {reps} builds")
prev = {}
for ph, t in tl:
    stream = "side" if "side" in ph or ph in ("local pass", "charge gather") else "s"
    dt = t - prev.get(stream, 0.0)
    prev[stream] = t
    print(f"  {t:8.3f} ms  (+{dt:6.3f} on {stream:4s})  {ph}")
