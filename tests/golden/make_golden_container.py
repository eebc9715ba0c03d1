"""sha256 of the UNMODIFIED reference's FMMS dumps (dump_structures,
lists.py:203-219) for the small golden cases and c1:

    python tests/golden/make_golden_container.py   # needs oracle/_ref

Writes tests/golden/container_hashes.json (committed)."""

import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, os.environ.get("FMMB_REFERENCE_SRC", os.path.join(ROOT, "oracle", "_ref")))

import fmmkit  # noqa: E402  (the reference)

from make_golden import LARGE, SMALL, inputs  # noqa: E402


def main():
    out = {}
    cases = [c for c in SMALL if c[3] >= 0] + [c for c in LARGE if c[0] == "c1"]
    with tempfile.TemporaryDirectory() as d:
        for name, n, m, L, dist, seed, wq in cases:
            src, q, recv = inputs(n, m, dist, seed)
            st = fmmkit.build_all(src, q if wq else None, recv, max_level=L)
            path = os.path.join(d, name + ".fmms")
            fmmkit.lists.dump_structures(st, path)
            with open(path, "rb") as f:
                raw = f.read()
            out[name] = {"sha256": hashlib.sha256(raw).hexdigest(), "bytes": len(raw)}
    with open(os.path.join(HERE, "container_hashes.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
