"""c4 dynamic rebuild: a 100-step trajectory of full data-structure rebuilds.

Each step moves both point sets on the device (x <- remainder(x + N(0, 1e-3),
1), workloads.perturb_device; timed separately from the rebuild) and then
runs the full fused build (build_all_device).  Per-step device times come
from CUDA events on the build stream.  One sampled step's inputs are copied
to the host and rebuilt by the reference CPU path (compiled fmmkit in
oracle/_ref, else the C oracle port); every output array of that step must
be bit-identical.

    python tools/c4_trajectory.py [--steps 100] [--check-step 37] [--no-check]

Prints one JSON line (per-step ms, median / p90, particles/s, parity).
Workload driver only: the reference / oracle is the checker here, never on
the timed path.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--check-step", type=int, default=37)
    p.add_argument("--no-check", action="store_true")
    p.add_argument("--seed", type=int, default=123)
    a = p.parse_args()

    import numpy as np
    import torch

    import paper_1301_1704_b200 as fb
    from paper_1301_1704_b200.workloads import WORKLOADS, generate, perturb_device

    sys.path.insert(0, os.path.join(ROOT))
    import bench

    wl = WORKLOADS["c4"]
    dev = torch.device("cuda", 0)
    src_np, q_np, recv_np = generate(wl.n, wl.n, wl.dist, wl.seed)
    src = torch.from_numpy(src_np).to(dev)
    q = torch.from_numpy(q_np).to(dev)
    recv = torch.from_numpy(recv_np).to(dev)
    stream = torch.cuda.current_stream(dev)
    n_part = 2 * wl.n
    # warm-up rebuilds on the unperturbed state (allocator, handle)
    for _ in range(3):
        st = fb.build_all_device(src, q, recv, wl.level, timing=False)
        st = None
    torch.cuda.synchronize()

    move_ms, build_ms, sample = [], [], None
    for k in range(a.steps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        perturb_device(src, a.seed, 2 * k + 2)
        perturb_device(recv, a.seed, 2 * k + 3)
        e1.record(stream)
        st = fb.build_all_device(src, q, recv, wl.level, timing=False)
        e2.record(stream)
        if not a.no_check and k == a.check_step:
            sample = (src.cpu().numpy(), recv.cpu().numpy(), st.to_numpy())
        st = None
        e2.synchronize()
        move_ms.append(e0.elapsed_time(e1))
        build_ms.append(e1.elapsed_time(e2))

    parity = None
    ref_s = None
    if sample is not None:
        s_in, r_in, ours = sample
        run, kind = bench.reference_build_fn()
        t0 = time.perf_counter()
        ref = run(s_in, q_np, r_in, wl.level)
        ref_s = time.perf_counter() - t0
        parity = bench.compare_outputs(ours, ref) | {"against": kind, "step": a.check_step}
        edge = int((s_in == 1.0).sum() + (r_in == 1.0).sum())
        parity["coords_equal_to_1.0"] = edge

    srt = sorted(build_ms)
    line = {
        "workload": f"c4: N=M={wl.n} uniform (seed {wl.seed}), L={wl.level}, "
                    f"{a.steps} rebuild steps, device perturbation seed {a.seed}",
        "build_ms_median": statistics.median(build_ms),
        "build_ms_p90": srt[int(0.9 * (len(srt) - 1))],
        "build_ms_min": srt[0], "build_ms_max": srt[-1],
        "move_ms_median": statistics.median(move_ms),
        "step_ms_median": statistics.median([m + b for m, b in zip(move_ms, build_ms)]),
        "particles_per_s_build": n_part / (statistics.median(build_ms) * 1e-3),
        "particles_per_s_step": n_part / (statistics.median(
            [m + b for m, b in zip(move_ms, build_ms)]) * 1e-3),
        "trajectory_s": sum(move_ms + build_ms) * 1e-3,
        "reference_step_s": ref_s,
        "parity_vs_reference": parity,
        "build_ms": [round(v, 4) for v in build_ms],
    }
    print(json.dumps(line), flush=True)
    if parity is not None and not parity["bit_exact"]:
        sys.exit(1)


if __name__ == "__main__":
    main()
