"""Loaders for the committed golden vectors (tests/golden/, produced by the
unmodified reference via tests/golden/make_golden.py)."""

import hashlib
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def small_cases() -> dict:
    z = np.load(os.path.join(HERE, "small_cases.npz"))
    cases = {}
    for key in z.files:
        name, field = key.split("/", 1)
        cases.setdefault(name, {})[field] = z[key]
    return cases


def encode_edges() -> dict:
    z = np.load(os.path.join(HERE, "encode_edges.npz"))
    return {k: z[k] for k in z.files}


def hashes() -> dict:
    with open(os.path.join(HERE, "hashes.json")) as f:
        return json.load(f)


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def flatten(st) -> dict:
    out = {}
    for side, ps in (("src", st.sorted_src), ("recv", st.sorted_recv)):
        for f in ("points", "permutation", "bookmarks", "non_empty_index", "boxes"):
            out[f"{side}.{f}"] = np.asarray(getattr(ps, f))
        if ps.charges is not None:
            out[f"{side}.charges"] = np.asarray(ps.charges)
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


def compare_flat(got: dict, want: dict) -> list:
    errors = []
    if set(got) != set(want):
        errors.append(f"field sets differ: {sorted(set(got) ^ set(want))}")
    for k in sorted(set(got) & set(want)):
        a, b = got[k], want[k]
        if a.dtype != b.dtype or a.shape != b.shape or not np.array_equal(a, b):
            errors.append(f"{k}: {a.dtype}{a.shape} vs {b.dtype}{b.shape}")
    return errors


def case_inputs(case: dict):
    src = case["in.src"]
    q = case.get("in.q")
    recv = case["in.recv"]
    return src, q, recv, int(case["level"])


def expected_outputs(case: dict) -> dict:
    return {k: v for k, v in case.items() if not k.startswith("in.") and k != "level"}


def large_inputs(spec: dict):
    from paper_1301_1704_b200.workloads import generate

    src, q, _ = generate(spec["n"], 1, spec["dist"], spec["seed"])
    _, _, recv = generate(1, spec["m"], spec["dist"], spec["seed"] + 1000)
    return src, (q if spec["charges"] else None), recv, spec["level"]


def nearfield() -> dict:
    """phi of the near-field consumer (tests/golden/make_golden_nearfield.py)."""
    z = np.load(os.path.join(HERE, "nearfield.npz"))
    return {k: z[k] for k in z.files}


def nearfield_hashes() -> dict:
    with open(os.path.join(HERE, "nearfield_hashes.json")) as f:
        return json.load(f)


def northstar_inputs(name: str):
    """Inputs of the north-star golden cases (make_golden_northstar.py): the
    bench's c2 / c3 arrays, and one perturbed c4 rebuild step."""
    from paper_1301_1704_b200.workloads import WORKLOADS, c4_step_inputs, generate

    wl = WORKLOADS[name]
    if name == "c4":
        src, q, recv = c4_step_inputs(wl.n, wl.seed, 1)
    else:
        src, q, recv = generate(wl.n, wl.n, wl.dist, wl.seed)
    return src, q, recv, wl.level
