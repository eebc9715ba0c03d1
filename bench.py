#!/usr/bin/env python
"""Benchmark of the B200 FMM data-structure build (BASELINE.json metric:
particles/s for the full build, fraction of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2]
    python bench.py --impl reference ...      # the reference CPU path

A step is one full `build_all` (sort both sets, bookmarks, level directory,
E2 neighbour table, E4 stencils at every level) over one batch of synthetic
input (`fmmkit.cli.generate`'s Philox streams).  `value` is device-resident
throughput (inputs already in HBM, outputs left in HBM); `e2e` goes through
the public API with pinned host inputs and numpy outputs (H2D + D2H inside
the timed region).  Inputs (0.94 GB at c2) exceed the 126 MB L2, so no flush
is needed between steps.

Multi-GPU (torchrun, N>1): ONE problem partitioned by Morton-key ranges
over NCCL (paper_1301_1704_b200.distributed: histogram all-reduce, all-to-all
of the points, all-reduce of the occupancy bitmaps, owned lists per rank).
Weak scaling: every rank contributes a c2-sized shard (N = M = 2^24 per GPU,
uniform, seed 1 + rank), the global level is choose_max_level(N_global, 16)
(the reference's cluster-size rule, pseudosort.py:22-29): L = 7, 7, 8, 8 at
1, 2, 4, 8 GPUs.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particles/sec for full FMM data-structure build"
NVLINK_GBS = 900.0  # NVLink 5 per direction per B200 (nominal)
UNIT = "particles/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default=None, choices=["c1", "c2", "c3", "c4", "c5"],
                   help="default: c2 on one GPU, c5 shards (2^27 + 2^27 per GPU, L=8) for N > 1")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--partitioned", action="store_true",
                   help="run the Morton-range partitioned path even at one process (P = 1)")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-nf", action="store_true", help="skip the near-field consumer timing")
    p.add_argument("--sort-path", default="auto",
                   choices=["auto", "bucket", "onesweep", "bucket_hist"])
    return p.parse_args()


# ------------------------------------------------------------------ ranks
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------- cpu reference
def workload_inputs(name: str):
    """The exact numpy inputs of a workload (the GPU arm uploads the same
    arrays): c1-c3 from fmmkit.cli.generate's streams, c4 = one perturbed
    rebuild step (workloads.c4_step_inputs, the c4 golden case)."""
    from paper_1301_1704_b200.workloads import WORKLOADS, c4_step_inputs, generate

    wl = WORKLOADS[name]
    if name == "c4":
        src, q, recv = c4_step_inputs(wl.n, wl.seed, 1)
    else:
        src, q, recv = generate(wl.n, wl.n, wl.dist, wl.seed)
    return src, q, recv, wl.level


def reference_build_fn():
    """(build_all callable, kind): the unmodified reference compiled from its
    sources into oracle/_ref (fmmkit, compiled backend, deterministic mode),
    else the C restatement of the same algorithm (oracle/)."""
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    try:
        sys.path.insert(0, ref_dir)
        import fmmkit  # noqa: F401  (oracle/_ref: the unmodified reference)

        assert fmmkit.backend_name() == "compiled"
        return (lambda s, q, r, L: fmmkit.build_all(s, q, r, max_level=L)), "reference"
    except Exception:
        sys.path.pop(0)
        from oracle import oracle as orc

        return (lambda s, q, r, L: orc.build_all(s, q, r, L)), "port"


def cpu_reference_rate(workload: str, steps: int = 1, budget_s: float = 90.0, inputs=None):
    """The reference CPU build_all on the IDENTICAL inputs of the workload
    (BASELINE.md section 3): up to `steps` timed builds, stopping once
    `budget_s` of build time is spent (at least one).  The deterministic
    reference build is single-threaded, so cores = 1.
    Returns (particles/s, kind, cores, sample, per-build seconds, last result)."""
    src, q, recv, L = inputs if inputs is not None else workload_inputs(workload)
    run, kind = reference_build_fn()
    times = []
    res = None
    while True:
        res = None
        t0 = time.perf_counter()
        res = run(src, q, recv, L)
        times.append(time.perf_counter() - t0)
        if len(times) >= steps or sum(times) > budget_s:
            break
    n_part = src.shape[0] + recv.shape[0]
    med = statistics.median(times)
    sample = (f"the full {workload} workload (identical arrays: N={src.shape[0]}, "
              f"M={recv.shape[0]}, max_level={L}), "
              f"{'compiled fmmkit (oracle/_ref)' if kind == 'reference' else 'C oracle port'}, "
              f"deterministic mode (single-threaded; os.cpu_count()={os.cpu_count()}), "
              f"median of {len(times)} build(s)")
    return n_part / med, kind, 1, sample, times, res


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    wl = "c2" if args.workload in ("c5",) else args.workload
    # one c2 reference build takes ~30 s: time up to --steps builds within a
    # ~2-minute budget (no warm-up: nothing to warm in a 30-s CPU build)
    rate, kind, cores, sample, times, _ = cpu_reference_rate(wl, steps=max(1, args.steps),
                                                             budget_s=100.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(times), "warmup": 0,
        "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(wl, 1),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "build_seconds": [round(t, 3) for t in times],
    }
    print(json.dumps(line), flush=True)


def workload_config(name: str, ws: int) -> dict:
    from paper_1301_1704_b200.workloads import WORKLOADS

    wl = WORKLOADS[name]
    extra = ", one perturbed rebuild step per timed step" if name == "c4" else ""
    return {
        "workload": f"{wl.name}: N=M={wl.n} {wl.dist}, max_level={wl.level}, seed={wl.seed}{extra}",
        "global_batch_particles": 2 * wl.n * ws,
        "parallelism": "single GPU" if ws == 1 else f"{ws} independent replicas",
        "l2": "inputs larger than the 126 MB L2 (c2: 0.94 GB); no flush",
    }


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax.append(float(parts[1]))
                except ValueError:
                    continue
                for name, v in zip(self.NAMES, parts[2:6]):
                    if v.lower().startswith("active"):
                        reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# -------------------------------------------------------------- our arm
def flat_outputs(st) -> dict:
    """Every output array of an FmmStructures (numpy), keyed like the golden files."""
    out = {}
    for side, ps in (("src", st.sorted_src), ("recv", st.sorted_recv)):
        for f in ("points", "charges", "permutation", "bookmarks", "non_empty_index", "boxes"):
            v = getattr(ps, f)
            if v is not None:
                out[f"{side}.{f}"] = np.asarray(v)
    out["neighbor_bookmark"] = np.asarray(st.neighbor_table.neighbor_bookmark)
    out["neighbor_list"] = np.asarray(st.neighbor_table.neighbor_list)
    for l, v in st.directory.src_boxes.items():
        out[f"dir_src.{l}"] = np.asarray(v)
    for l, v in st.directory.recv_boxes.items():
        out[f"dir_recv.{l}"] = np.asarray(v)
    for f in ("bookmark", "ranks", "codes"):
        for l, v in getattr(st.stencils, f).items():
            out[f"st_{f}.{l}"] = np.asarray(v)
    return out


def compare_outputs(got, want) -> dict:
    """Bit-equality of every output array (values, dtypes, shapes)."""
    g, w = flat_outputs(got), flat_outputs(want)
    bad = sorted(k for k in set(g) | set(w)
                 if k not in g or k not in w or g[k].dtype != w[k].dtype
                 or g[k].shape != w[k].shape or not np.array_equal(g[k], w[k]))
    return {"bit_exact": not bad, "arrays": len(w), "mismatched": bad[:8],
            "bytes": int(sum(v.nbytes for v in w.values()))}


def run_ours(args):
    import torch

    import paper_1301_1704_b200 as fb
    from paper_1301_1704_b200 import roofline
    from paper_1301_1704_b200.workloads import perturb_device

    torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    fb._lib.set_sort_path(args.sort_path, dev)
    src_np, q_np, recv_np, L = workload_inputs(args.workload)
    src = torch.from_numpy(src_np).to(dev)
    q = torch.from_numpy(q_np).to(dev)
    recv = torch.from_numpy(recv_np).to(dev)
    n_part = src.shape[0] + recv.shape[0]
    stream = torch.cuda.current_stream(dev)
    c4 = args.workload == "c4"
    pstep = [0]  # c4 trajectory step (perturbation key)

    def step():
        if c4:  # dynamic rebuild: the particles move, then the full rebuild
            pstep[0] += 1
            perturb_device(src, 123, 2 * pstep[0])
            perturb_device(recv, 123, 2 * pstep[0] + 1)
        return fb.build_all_device(src, q, recv, L)

    # warm-up (also sizes the caching allocator for the outputs)
    st = None
    for _ in range(max(args.warmup, 3)):
        st = None
        st = step()
    counts = roofline.build_counts(st)
    balg = roofline.build_bytes(counts)
    wbytes = roofline.list_write_bytes(counts)
    st = None
    torch.cuda.synchronize()

    clocks = ClockSampler(dev.index)
    clocks.start()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    phases = []
    launches = 0
    ev0.record(stream)
    for _ in range(args.steps):
        st = step()
        phases.append(st.build_seconds)
        launches += st.n_launches + (2 if c4 else 0)  # + the two k_perturb launches
        st = None
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    elapsed = ev0.elapsed_time(ev1) * 1e-3
    value = n_part * args.steps / elapsed
    ms_step = elapsed / args.steps * 1e3

    keys = ("sort_sources", "level_directory", "lists_count", "size_readback", "lists_write")
    ph = {k: statistics.median([float(p[k]) for p in phases]) * 1e3 for k in keys}
    build_ms = statistics.median([sum(float(p[k]) for k in keys) for p in phases]) * 1e3
    peak, peak_src = roofline.measured_hbm_gbs(ROOT)
    traffic = None  # DRAM bytes per launch of the dominant kernel, from the committed ncu capture
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            t = json.load(f).get("k_lists_write", {})
        if t.get("workload") == args.workload:
            traffic = int(t["dram_bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        pass
    write_s = ph["lists_write"] * 1e-3
    achieved = wbytes / write_s / 1e9
    build_gbs = balg / (elapsed / args.steps) / 1e9

    # ---- end to end: pinned host inputs -> public API -> numpy outputs
    e2e = None
    ours_np = None
    if not args.no_e2e:
        h_src = torch.from_numpy(src_np).pin_memory()
        h_q = torch.from_numpy(q_np).pin_memory()
        h_recv = torch.from_numpy(recv_np).pin_memory()
        h2d = (h_src.numel() + h_q.numel() + h_recv.numel()) * 8
        res = fb.build_all(h_src, h_q, h_recv, max_level=L)  # warm (pins output buffers)
        d2h = _numpy_bytes(res)
        res = None
        times = []
        for _ in range(max(1, args.e2e_steps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = fb.build_all(h_src, h_q, h_recv, max_level=L)
            times.append(time.perf_counter() - t0)
            ours_np = res
            res = None
        e2e = {"value": n_part / statistics.median(times), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": statistics.median(times) * 1e3}

    # ---- the near-field pass consuming the device-built
    # structures in place (not part of the build metric; reported beside it)
    nf = None
    if not args.no_nf and not c4:
        st = fb.build_all_device(src, q, recv, L)
        ss, sr, nt = st.sorted_src, st.sorted_recv, st.neighbor_table
        cs = torch.nn.functional.pad(torch.cumsum(torch.diff(ss.bookmarks)[nt.neighbor_list], 0),
                                     (1, 0))
        pairs = int(((cs[nt.neighbor_bookmark[1:]] - cs[nt.neighbor_bookmark[:-1]])
                     * torch.diff(sr.bookmarks)).sum())
        fb.near_field_potentials(st)
        nts = []
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fb.near_field_potentials(st)
            e1.record(stream)
            torch.cuda.synchronize()
            nts.append(e0.elapsed_time(e1) * 1e-3)
        t_nf = statistics.median(nts)
        nf = {"kernel": "k_near_field", "pair_interactions": pairs, "ms": t_nf * 1e3,
              "interactions_per_s": pairs / t_nf, "dtype": "f64 (bit-exact vs compiled reference)"}
        st = None

    # ---- the reference CPU build on the identical arrays, and bit-equality
    # of every output array with this run's end-to-end result
    cpu = None
    parity = None
    if not args.no_cpu:
        rate, kind, cores, sample, _, ref_res = cpu_reference_rate(
            args.workload, steps=1, inputs=(src_np, q_np, recv_np, L))
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
        if ours_np is not None:
            parity = compare_outputs(ours_np, ref_res) | {"against": kind}
        ref_res = None
    ours_np = None

    cfg = workload_config(args.workload, 1)
    if c4:
        cfg["step"] = ("device perturbation x <- mod(x + N(0,1e-3), 1) of both sets "
                       "(timed, fused k_perturb pass each) + full rebuild; trajectory seed 123")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64/u64 (integer keys, f64 points)",
        "data": "synthetic (fmmkit.cli.generate Philox streams)",
        "config": cfg,
        "roofline": {
            "bound": "hbm", "kernel": "k_lists_write (E2+E4 list write)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": peak_src, "traffic": traffic,
            "alg_bytes_per_launch": wbytes, "avg_launch_ms": ph["lists_write"],
        },
        "build_roofline": {
            "alg_bytes_per_step": balg, "achieved_gbs": build_gbs,
            "frac_of_measured": build_gbs / peak,
            "frac_of_nominal_8tbs": build_gbs / roofline.NOMINAL_HBM_GBS,
        },
        "build_ms_per_step": build_ms,
        "phases_ms": ph,
        "counts": {k: counts[k] for k in ("ks", "kr", "e2")} | {
            "stencil_entries": int(sum(counts["s_l"].values()))},
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity_vs_reference": parity,
        "gpu_launches": int(launches),
        "near_field": nf,
    }
    print(json.dumps(line), flush=True)


def _numpy_bytes(st) -> int:
    tot = 0
    for ps in (st.sorted_src, st.sorted_recv):
        for f in ("points", "charges", "permutation", "bookmarks", "non_empty_index", "boxes"):
            v = getattr(ps, f)
            if v is not None:
                tot += v.nbytes
    tot += st.neighbor_table.neighbor_bookmark.nbytes + st.neighbor_table.neighbor_list.nbytes
    L = st.max_level
    for l in range(2, L):
        tot += st.directory.src_boxes[l].nbytes + st.directory.recv_boxes[l].nbytes
    for l in st.stencils.ranks:
        tot += (st.stencils.bookmark[l].nbytes + st.stencils.ranks[l].nbytes
                + st.stencils.codes[l].nbytes)
    return tot


def run_partitioned(args):
    """N > 1: the Morton-range partitioned build of one problem (NCCL)."""
    import torch
    import torch.distributed as dist

    from paper_1301_1704_b200 import distributed as D
    from paper_1301_1704_b200 import roofline
    from paper_1301_1704_b200.pseudosort import choose_max_level
    from paper_1301_1704_b200.workloads import WORKLOADS, generate

    ws, rank, local = dist_env()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("FMMB_DIST_BACKEND", "nccl")  # gloo: host-staged (testing)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    wl = WORKLOADS[args.workload]
    if wl.name == "c5":  # 2^27 + 2^27 per GPU (c5 = 2^30 + 2^30 at 8 GPUs), fixed L = 8
        n_per = wl.n // 8
        L = wl.level
        # generated per shard on the device (torch Philox, seed 1 + rank): a
        # 2^30 host generation is 24 GB per array
        g = torch.Generator(device=dev)
        g.manual_seed(wl.seed + rank)
        src = torch.rand((n_per, 3), generator=g, device=dev, dtype=torch.float64)
        recv = torch.rand((n_per, 3), generator=g, device=dev, dtype=torch.float64)
        q = torch.randn(n_per, generator=g, device=dev, dtype=torch.float64)
        src_np = q_np = recv_np = None
    else:
        n_per = wl.n
        L = choose_max_level(n_per * ws, 16)
        src_np, q_np, recv_np = generate(n_per, n_per, wl.dist, wl.seed + rank)
        src = torch.from_numpy(src_np).to(dev)
        q = torch.from_numpy(q_np).to(dev)
        recv = torch.from_numpy(recv_np).to(dev)
    n_glob = n_per * ws
    comm = D.TorchComm()
    ops = D.DeviceOps()
    timer = [None]

    def step():
        return D.build_all_distributed([(src, q, recv)], L, comm, ops=ops, timer=timer[0])[0]

    sh = None
    for _ in range(max(args.warmup, 3)):
        sh = None
        sh = step()
    pts = int(sh.sorted_src.points.shape[0] + sh.sorted_recv.points.shape[0])
    sent = int(sh.exchanged["sent_points"])
    sent_bytes = int(sh.exchanged.get("sent_bytes", 0))
    lists_bytes = 8 * int(sh.neighbor_table.neighbor_list.shape[0]) + sum(
        10 * int(v.shape[0]) for v in sh.stencils.ranks.values())
    sh = None
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ops.launches = 0
    timer[0] = D.PhaseTimer()
    ev0.record(stream)
    for _ in range(args.steps):
        sh = step()
        sh = None
    ev1.record(stream)
    launches = ops.launches
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([ev0.elapsed_time(ev1) * 1e-3], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    agg = torch.tensor([pts, sent, lists_bytes, sent_bytes], device=dev, dtype=torch.int64)
    dist.all_reduce(agg)
    pts_all, sent_all, lists_all, sent_bytes_all = (int(x) for x in agg.tolist())
    # per-phase device time (events on this rank's stream), max over ranks
    ph = timer[0].ms()
    names = sorted(ph)
    pt = torch.tensor([ph[k] / args.steps for k in names], device=dev, dtype=torch.float64)
    dist.all_reduce(pt, op=dist.ReduceOp.MAX)
    phases = {k: float(v) for k, v in zip(names, pt.tolist())}
    ex_ms = sum(v for k, v in phases.items() if k.startswith("exchange"))
    sent_max = torch.tensor([sent_bytes], device=dev, dtype=torch.int64)
    dist.all_reduce(sent_max, op=dist.ReduceOp.MAX)
    sent_max = int(sent_max.item())
    ms_step = elapsed / args.steps * 1e3
    value = 2 * n_glob * args.steps / elapsed
    # per-GPU algorithmic bytes: inputs + sorted outputs (SURVEY 8(d), 80/64 B per
    # src/recv point) + the lists this rank owns, against its share of the step
    per_gpu_bytes = (80 + 64) / 2 * pts_all / ws + lists_all / ws
    achieved = per_gpu_bytes / (elapsed / args.steps) / 1e9
    peak, peak_src = roofline.measured_hbm_gbs(ROOT)
    e2e = None
    e2e_note = None
    if not args.no_e2e:
        e_src, e_q, e_recv, e_L, e_n = src, q, recv, L, n_glob
        # host outputs of one rank ~ 200 B per particle; with every local
        # rank holding them, stay within ~1/3 of the host's available RAM
        # (a c5 shard is ~60 GB of numpy outputs per rank): else measure the
        # end-to-end path on c2-size shards (2^24 + 2^24 per rank)
        try:
            avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
        except (ValueError, OSError):
            avail = 0
        local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
        need = 200 * 2 * n_per * local_ranks * 2
        if avail and need > avail / 3 and n_per > 2**24:
            g2 = torch.Generator(device=dev)
            g2.manual_seed(7 + rank)
            e_n = 2**24
            e_src = torch.rand((e_n, 3), generator=g2, device=dev, dtype=torch.float64)
            e_recv = torch.rand((e_n, 3), generator=g2, device=dev, dtype=torch.float64)
            e_q = torch.randn(e_n, generator=g2, device=dev, dtype=torch.float64)
            e_L = choose_max_level(e_n * ws, 16)
            e_n = e_n * ws
            e2e_note = (f"c2-size shards (N=M=2^24 per rank, max_level={e_L}): the {wl.name} "
                        f"host outputs ({need / 1e9:.0f} GB on this node) exceed 1/3 of the "
                        f"available host RAM ({avail / 1e9:.0f} GB)")
        h_src = e_src.cpu().pin_memory()
        h_q = e_q.cpu().pin_memory()
        h_recv = e_recv.cpu().pin_memory()
        times = []
        d2h = 0
        for _ in range(max(1, args.e2e_steps)):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            shard = [(h_src.to(dev, non_blocking=True), h_q.to(dev, non_blocking=True),
                      h_recv.to(dev, non_blocking=True))]
            out = D.build_all_distributed(shard, e_L, comm)[0].to_numpy()
            dt = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            times.append(float(dt.item()))
            d2h = _numpy_bytes_shard(out)
            out = None
        h2d = (h_src.numel() + h_q.numel() + h_recv.numel()) * 8
        e2e = {"value": 2 * e_n / statistics.median(times), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d * ws), "d2h_bytes_per_step": int(d2h * ws),
               "ms_per_step": statistics.median(times) * 1e3}
        if e2e_note:
            e2e["workload"] = e2e_note
    cpu = None
    if rank == 0 and not args.no_cpu:
        # the reference CPU build of c2 on identical arrays (rank 0 only, after
        # the timed region); the c5 problem (2^31 points) does not fit the
        # host, so its CPU rate is extrapolated at c2's per-particle rate
        rate, kind, cores, sample, _, _ = cpu_reference_rate("c2", steps=1)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": sample + "; extrapolated to this workload at the same "
                                  "per-particle rate (the global problem exceeds host memory)"}
    dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f64/u64 (integer keys, f64 points)",
            "data": "synthetic (fmmkit.cli.generate Philox streams, seed 1 + rank)",
            "config": {
                "workload": f"{wl.name} shard per GPU: N=M={n_per} {wl.dist} per rank, "
                            f"global N=M={n_glob}, max_level={L} (cluster size 16)",
                "global_batch_particles": 2 * n_glob,
                "parallelism": f"{ws}-way Morton-range partition ({backend} all-reduce + all-to-all)",
                "l2": "inputs larger than the 126 MB L2; no flush",
            },
            "roofline": {
                "bound": "hbm", "kernel": "whole partitioned step per GPU",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": peak_src, "traffic": None,
            },
            "exchange": {
                "points_sent": sent_all, "bytes_sent": sent_bytes_all,
                "max_bytes_sent_per_gpu": sent_max, "ms": ex_ms,
                "nvlink_roofline": {
                    "bound": "nvlink", "unit": "GB/s",
                    "achieved": (sent_max / (ex_ms * 1e-3) / 1e9) if ex_ms > 0 else None,
                    "peak": NVLINK_GBS, "peak_source": "nominal NVLink 5, per direction per GPU",
                    "frac": (sent_max / (ex_ms * 1e-3) / 1e9 / NVLINK_GBS) if ex_ms > 0 else None},
            },
            "phases_ms": phases,
            "max_memory_gb_rank0": torch.cuda.max_memory_allocated(dev) / 1e9,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _numpy_bytes_shard(sh) -> int:
    tot = 0
    for ps in (sh.sorted_src, sh.sorted_recv):
        for f in ("points", "charges", "permutation", "bookmarks", "non_empty_index", "boxes"):
            v = getattr(ps, f)
            if v is not None:
                tot += v.nbytes
    tot += sh.neighbor_table.neighbor_bookmark.nbytes + sh.neighbor_table.neighbor_list.nbytes
    for l in sh.stencils.ranks:
        tot += (sh.stencils.bookmark[l].nbytes + sh.stencils.ranks[l].nbytes
                + sh.stencils.codes[l].nbytes)
    return tot


def main():
    args = parse()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.workload is None:
        args.workload = "c2" if ws == 1 and not args.partitioned else "c5"
    if args.impl == "reference":
        run_reference_arm(args)
    elif ws > 1 or args.partitioned:
        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531"), ("RANK", "0"),
                     ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0")):
            os.environ.setdefault(k, v)
        run_partitioned(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
