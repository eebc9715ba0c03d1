"""Generate the golden vectors of the build path FROM THE UNMODIFIED REFERENCE.

    python tests/golden/make_golden.py     # needs oracle/_ref (oracle/build_ref.sh)
                                           # or FMMB_REFERENCE_SRC=/root/reference/pkg/src

Writes (committed):
  small_cases.npz   full input + output arrays of small build_all cases
  encode_edges.npz  encode_points on boundary / out-of-domain coordinates
  hashes.json       sha256 of every output array of the larger cases
                    (inputs regenerate bit-identically from workloads.generate)
The reference runs here (CPU container) only; the GPU box compares against
these files (and against oracle/_ref when it travels along).
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("FMMB_REFERENCE_SRC", os.path.join(ROOT, "oracle", "_ref")))

import fmmkit  # noqa: E402  (the reference)

from paper_1301_1704_b200.workloads import generate  # noqa: E402

# (name, n_src, n_recv, level, dist, seed, with_charges)
SMALL = [
    ("u3_L3", 600, 500, 3, "uniform", 21, True),
    ("s5_L5", 700, 700, 5, "sphere", 27, True),
    ("u_L0", 50, 40, 0, "uniform", 3, True),
    ("u_L1", 60, 70, 1, "uniform", 4, False),
    ("u_L2", 80, 90, 2, "uniform", 5, True),
    ("src_only", 120, 0, 3, "uniform", 6, True),
    ("recv_only", 0, 130, 3, "uniform", 7, False),
    ("single", 1, 1, 3, "uniform", 8, True),
    ("u9_sparse", 300, 300, 9, "uniform", 9, True),
]
LARGE = [
    ("c1", 2**16, 2**16, 4, "uniform", 1, True),
    ("u20_L7", 2**20, 2**20, 7, "uniform", 1, True),
    ("s20_L9", 2**20, 2**20, 9, "sphere", 1, True),
    ("u20_L3", 2**20, 2**20, 3, "uniform", 30, False),
]


def inputs(n, m, dist, seed):
    src, q, _ = generate(n, 1, dist, seed)
    _, _, recv = generate(1, m, dist, seed + 1000)
    return src, q, recv


def flatten(st) -> dict:
    out = {}
    for side, ps in (("src", st.sorted_src), ("recv", st.sorted_recv)):
        for f in ("points", "permutation", "bookmarks", "non_empty_index", "boxes"):
            out[f"{side}.{f}"] = getattr(ps, f)
        if ps.charges is not None:
            out[f"{side}.charges"] = ps.charges
    out["neighbor_bookmark"] = st.neighbor_table.neighbor_bookmark
    out["neighbor_list"] = st.neighbor_table.neighbor_list
    for l, v in st.directory.src_boxes.items():
        out[f"dir_src.{l}"] = v
    for l, v in st.directory.recv_boxes.items():
        out[f"dir_recv.{l}"] = v
    for f in ("bookmark", "ranks", "codes"):
        for l, v in getattr(st.stencils, f).items():
            out[f"st_{f}.{l}"] = v
    return out


def sha(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def main():
    assert fmmkit.backend_name() == "compiled", fmmkit.backend_name()
    arrays = {}
    for name, n, m, L, dist, seed, wq in SMALL:
        src, q, recv = inputs(n, m, dist, seed)
        st = fmmkit.build_all(src, q if wq else None, recv, max_level=L)
        arrays[f"{name}/in.src"] = src
        if wq:
            arrays[f"{name}/in.q"] = q
        arrays[f"{name}/in.recv"] = recv
        arrays[f"{name}/level"] = np.array(L)
        for k, v in flatten(st).items():
            arrays[f"{name}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)

    one = 1.0
    below = np.nextafter(1.0, 0.0)
    edge = np.array([0.0, one, below, 2.0**-30, 0.5, 1.5, -0.0, 1e-300, 0.999999999,
                     -0.1, -0.7, -1e-9, np.nan, np.inf, -np.inf, 1e300, 0.25, 0.75])
    g = np.meshgrid(edge, edge[::-1], edge[::3], indexing="ij")
    pts = np.stack([x.reshape(-1) for x in g], axis=1)
    enc = {"pts": pts}
    ck = fmmkit.backend.get_kernels("compiled")
    for L in (0, 1, 3, 7, 9, 20):
        enc[f"L{L}"] = ck.encode_points(pts[:, 0], pts[:, 1], pts[:, 2], L)
    np.savez_compressed(os.path.join(HERE, "encode_edges.npz"), **enc)

    hashes = {}
    for name, n, m, L, dist, seed, wq in LARGE:
        src, q, recv = inputs(n, m, dist, seed)
        st = fmmkit.build_all(src, q if wq else None, recv, max_level=L)
        hashes[name] = {"n": n, "m": m, "level": L, "dist": dist, "seed": seed,
                        "charges": wq, "arrays": {k: sha(v) for k, v in flatten(st).items()}}
        print(name, "done", flush=True)
    with open(os.path.join(HERE, "hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
