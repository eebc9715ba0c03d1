"""Golden vectors of the near-field consumer FROM THE
UNMODIFIED REFERENCE (compiled backend):

    python tests/golden/make_golden_nearfield.py   # needs oracle/_ref

Writes (committed):
  nearfield.npz      phi = fmmkit.near_field_potentials(build_all(...)) for the
                     small cases of make_golden.py (inputs regenerate from
                     workloads.generate), direct_sum on two of them, and a
                     clustered case (hundreds of points per box, coincident
                     pairs) with its inputs
  nearfield_hashes.json  sha256 of phi for the larger cases
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, os.environ.get("FMMB_REFERENCE_SRC", os.path.join(ROOT, "oracle", "_ref")))

import fmmkit  # noqa: E402  (the reference)

from make_golden import LARGE, SMALL, inputs, sha  # noqa: E402


def clustered():
    """Two tight clusters (L=2: hundreds of points per box) with duplicated
    points, so coincident pairs (dist == 0) are skipped."""
    rng = np.random.default_rng(77)
    a = 0.1 + 0.05 * rng.random((300, 3))
    b = 0.6 + 0.1 * rng.random((200, 3))
    src = np.concatenate([a, b, a[:40]])
    recv = np.concatenate([b[:100], a[100:250], 0.9 * rng.random((60, 3))])
    q = rng.normal(size=src.shape[0])
    return src, q, recv


def main():
    assert fmmkit.backend_name() == "compiled", fmmkit.backend_name()
    out = {}
    for name, n, m, L, dist, seed, wq in SMALL:
        src, q, recv = inputs(n, m, dist, seed)
        st = fmmkit.build_all(src, q if wq else None, recv, max_level=L)
        out[f"{name}/phi"] = fmmkit.near_field_potentials(st)
    for name in ("u3_L3", "s5_L5"):
        n, m, L, dist, seed = next((c[1], c[2], c[3], c[4], c[5]) for c in SMALL if c[0] == name)
        src, q, recv = inputs(n, m, dist, seed)
        out[f"{name}/direct"] = fmmkit.direct_sum(src, q, recv)
    src, q, recv = clustered()
    out["clustered/in.src"], out["clustered/in.q"], out["clustered/in.recv"] = src, q, recv
    for L in (0, 2):
        st = fmmkit.build_all(src, q, recv, max_level=L)
        out[f"clustered/L{L}/phi"] = fmmkit.near_field_potentials(st)
    out["clustered/direct"] = fmmkit.direct_sum(src, q, recv)
    np.savez_compressed(os.path.join(HERE, "nearfield.npz"), **out)

    hashes = {}
    for name, n, m, L, dist, seed, wq in LARGE:
        src, q, recv = inputs(n, m, dist, seed)
        st = fmmkit.build_all(src, q if wq else None, recv, max_level=L)
        hashes[name] = sha(fmmkit.near_field_potentials(st))
        print(name, "done", flush=True)
    with open(os.path.join(HERE, "nearfield_hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
