"""Algorithmic (compulsory) HBM bytes of the build, SURVEY §8(d).

Each input is read once and each output written once in the reference's
output dtypes (the drop-in contract fixes them): f64 points/charges, i64
permutation/bookmarks/CSR, u64 keys, i16 codes.  Implementation-independent.
"""

from __future__ import annotations

import json
import os

NOMINAL_HBM_GBS = 8000.0  # north-star denominator (B200 nominal)
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when no measured file


def measured_hbm_gbs(root: str | None = None) -> tuple[float, str]:
    """(GB/s, source) from MEASURED_PEAKS.json, else the profiling fallback."""
    root = root or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback"


def _shape0(a) -> int:
    return int(a.shape[0])


def build_counts(st) -> dict:
    """Box / list counts of an FmmStructures (numpy or torch)."""
    L = st.max_level
    return {
        "L": L,
        "n": _shape0(st.sorted_src.points),
        "m": _shape0(st.sorted_recv.points),
        "q": st.sorted_src.charges is not None,
        "ks": _shape0(st.sorted_src.non_empty_index),
        "kr": _shape0(st.sorted_recv.non_empty_index),
        "e2": _shape0(st.neighbor_table.neighbor_list),
        "ks_l": {l: _shape0(v) for l, v in st.directory.src_boxes.items()},
        "kr_l": {l: _shape0(v) for l, v in st.directory.recv_boxes.items()},
        "s_l": {l: _shape0(v) for l, v in st.stencils.ranks.items()},
    }


def build_bytes(c: dict) -> int:
    """B_alg of the whole build (SURVEY §8(d) formula)."""
    n, m, L = c["n"], c["m"], c["L"]
    qb = 8 if c["q"] else 0
    b = 24 * n + qb * n + 24 * m  # inputs
    b += (40 + qb) * n + 16 * c["ks"] + 8  # sorted src (points, charges, perm, boxes; bm, ne)
    b += 40 * m + 16 * c["kr"] + 8  # sorted recv
    b += 8 * (c["kr"] + 1) + 8 * c["e2"]  # E2 CSR
    for l in range(2, L):
        b += 8 * (c["ks_l"][l] + c["kr_l"][l])  # directory
    for l in range(2, L + 1):
        b += 8 * (c["kr_l"][l] + 1) + 10 * c["s_l"][l]  # E4 CSR + codes
    return b


def list_write_bytes(c: dict) -> int:
    """Compulsory bytes of the list write kernel (k_lists_write) itself: every
    E2 and E4 entry written once (i64 rank, i16 code), and per receiver parent
    its key and the first CSR offset of its rows (one per CSR it writes: E4,
    and E2 at the finest level) read once.  The CSR bookmarks are written by
    the count pass (k_lists_cscan), not here."""
    L = c["L"]
    b = 8 * c["e2"]
    for l in range(2, L + 1):
        b += 10 * c["s_l"][l]
    for l in range(max(1, 2 if L >= 2 else L), L + 1):
        parents = c["kr_l"].get(l - 1, 0)
        b += 8 * parents * (1 + (1 if l >= 2 else 0) + (1 if l == L else 0))
    return b
