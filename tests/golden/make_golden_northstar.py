"""sha256 of every output array of the UNMODIFIED reference's build_all at the
north-star configurations (BASELINE.json configs c2, c3 and one c4 rebuild
step), on exactly the inputs bench.py builds from:

    c2  generate(2^24, 2^24, "uniform", 1), max_level 7
    c3  generate(2^24, 2^24, "sphere", 1),  max_level 9
    c4  workloads.c4_step_inputs(2^23, 4, 1), max_level 7 (one perturbation
        with default_rng(123), clamp-edge coordinates == 1.0 injected)

    python tests/golden/make_golden_northstar.py [c2 c3 c4]

Writes tests/golden/hashes_northstar.json (committed) with the reference's
wall time per build (context only; bench.py times the reference on the GPU
box).  Takes ~35 + 22 + 30 s of reference build plus input generation.
"""

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("FMMB_REFERENCE_SRC", os.path.join(ROOT, "oracle", "_ref")))

import fmmkit  # noqa: E402  (the reference)

from tests.golden_io import northstar_inputs  # noqa: E402

sys.path.insert(0, HERE)
from make_golden import flatten, sha  # noqa: E402

OUT = os.path.join(HERE, "hashes_northstar.json")


def main(names):
    assert fmmkit.backend_name() == "compiled", fmmkit.backend_name()
    out = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            out = json.load(f)
    for name in names:
        src, q, recv, L = northstar_inputs(name)
        t0 = time.perf_counter()
        st = fmmkit.build_all(src, q, recv, max_level=L)
        dt = time.perf_counter() - t0
        out[name] = {"level": L, "n": int(src.shape[0]), "m": int(recv.shape[0]),
                     "reference_build_s": round(dt, 2),
                     "arrays": {k: sha(v) for k, v in flatten(st).items()}}
        print(name, "done", round(dt, 1), "s", flush=True)
        del st
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c4"])
