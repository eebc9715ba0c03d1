"""CPU oracle for the FMM data-structure build — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this
module, and only as the checker.  `build_all` restates the reference
`fmmkit.build_all` (pkg/src/fmmkit/lists.py:133-187) on top of the C
restatement in fmm_oracle.c (liborcl.so, built by `make -C oracle`), and
returns the same field layout as the reference FmmStructures (numpy arrays).

Parity: pinned against tests/golden/ (vectors produced by the unmodified
reference, tests/golden/make_golden.py) and against the reference itself
whenever oracle/_ref (oracle/build_ref.sh) is importable.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liborcl.so")
_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", HERE, "oracle_lib"], check=True)
        lib = C.CDLL(LIB)
        p, i64 = C.c_void_p, C.c_int64
        lib.orc_encode.argtypes = [p, i64, C.c_int, p]
        lib.orc_assign_ranks.argtypes = [p, i64, p, i64, p]
        lib.orc_bookmarks.argtypes = [p, i64, p, p]
        lib.orc_bookmarks.restype = i64
        lib.orc_reorder.argtypes = [p, p, i64, p, i64, p, p, p, p, p, p]
        lib.orc_adjacent_segments.argtypes = [p, i64, p, i64, C.c_int, p, p]
        lib.orc_adjacent_segments.restype = i64
        lib.orc_stencil_segments.argtypes = [p, i64, p, i64, C.c_int, p, p, p]
        lib.orc_stencil_segments.restype = i64
        lib.orc_propagate.argtypes = [p, i64, p]
        lib.orc_near_field.argtypes = [p, p, p, p, p, p, p, i64, i64, p]
        lib.orc_direct.argtypes = [p, p, i64, p, i64, p]
        lib.orc_propagate.restype = i64
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def encode(points: np.ndarray, level: int) -> np.ndarray:
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    out = np.empty(pts.shape[0], dtype=np.uint64)
    load().orc_encode(_ptr(pts), pts.shape[0], level, _ptr(out))
    return out


DENSE_LIMIT = 1 << 27  # dense 8^L histogram like the reference; beyond, stable argsort


def sort_points(points, charges, level: int) -> SimpleNamespace:
    """pseudosort.sort_points (pseudosort.py:138-151) for deterministic mode."""
    lib = load()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    keys = encode(pts, level)
    q = None if charges is None else np.ascontiguousarray(charges, dtype=np.float64)
    nbins = 8**level
    if nbins <= DENSE_LIMIT:
        bins = np.empty(nbins, dtype=np.int64)
        ranks = np.empty(n, dtype=np.int64)
        lib.orc_assign_ranks(_ptr(keys), n, bins.ctypes.data, nbins, _ptr(ranks))
        pts_out = np.empty_like(pts)
        q_out = np.empty(n) if q is not None else None
        perm = np.empty(n, dtype=np.int64)
        boxes = np.empty(n, dtype=np.uint64)
        lib.orc_reorder(_ptr(pts), _ptr(q) if q is not None else None, n, bins.ctypes.data,
                        nbins, _ptr(keys), _ptr(ranks), _ptr(pts_out),
                        _ptr(q_out) if q_out is not None else None, _ptr(perm), _ptr(boxes))
        bm = np.empty(min(nbins, max(n, 0)) + 1, dtype=np.int64)
        ne = np.empty(min(nbins, max(n, 1)), dtype=np.uint64)
        k = lib.orc_bookmarks(bins.ctypes.data, nbins, bm.ctypes.data, ne.ctypes.data)
        bm, ne = bm[: k + 1].copy(), ne[:k].copy()
    else:  # same order as the dense counter: stable by key (_pykernels.py:82)
        perm = np.argsort(keys, kind="stable").astype(np.int64)
        boxes = keys[perm]
        pts_out = pts[perm]
        q_out = q[perm] if q is not None else None
        heads = np.ones(n, dtype=bool)
        heads[1:] = boxes[1:] != boxes[:-1]
        starts = np.flatnonzero(heads)
        ne = boxes[starts] if n else np.empty(0, dtype=np.uint64)
        bm = np.append(starts, n).astype(np.int64) if n else np.zeros(1, dtype=np.int64)
    return SimpleNamespace(level=level, points=pts_out, charges=q_out, permutation=perm,
                           bookmarks=bm, non_empty_index=ne, boxes=boxes)


def build_bookmarks(bins):
    """pseudosort.build_bookmarks (pseudosort.py:68-78) via orc_bookmarks."""
    b = np.ascontiguousarray(bins, dtype=np.int64)
    bm = np.empty(b.size + 1, dtype=np.int64)
    ne = np.empty(max(b.size, 1), dtype=np.uint64)
    k = load().orc_bookmarks(b.ctypes.data, b.size, bm.ctypes.data, ne.ctypes.data)
    return bm[: k + 1].copy(), ne[:k].copy()


def reorder(points, charges, bins, boxes, ranks):
    """pseudosort.reorder (pseudosort.py:105-135) via orc_reorder + orc_bookmarks."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    q = None if charges is None else np.ascontiguousarray(charges, dtype=np.float64)
    b = np.ascontiguousarray(bins, dtype=np.int64)
    bx = np.ascontiguousarray(boxes, dtype=np.uint64)
    rk = np.ascontiguousarray(ranks, dtype=np.int64)
    pts_out = np.empty_like(pts)
    q_out = np.empty(n) if q is not None else None
    perm = np.empty(n, dtype=np.int64)
    bo = np.empty(n, dtype=np.uint64)
    load().orc_reorder(_ptr(pts), _ptr(q) if q is not None else None, n, b.ctypes.data, b.size,
                       _ptr(bx), _ptr(rk), _ptr(pts_out),
                       _ptr(q_out) if q_out is not None else None, _ptr(perm), _ptr(bo))
    bm, ne = build_bookmarks(b)
    return SimpleNamespace(points=pts_out, charges=q_out, permutation=perm, bookmarks=bm,
                           non_empty_index=ne, boxes=bo)


def adjacent_segments(recv, src, level):
    lib = load()
    r = np.ascontiguousarray(recv, dtype=np.uint64)
    s = np.ascontiguousarray(src, dtype=np.uint64)
    bm = np.empty(r.size + 1, dtype=np.int64)
    tot = lib.orc_adjacent_segments(_ptr(r), r.size, _ptr(s), s.size, level, bm.ctypes.data, None)
    lst = np.empty(tot, dtype=np.int64)
    lib.orc_adjacent_segments(_ptr(r), r.size, _ptr(s), s.size, level, bm.ctypes.data, _ptr(lst))
    return bm, lst


def stencil_segments(recv, src, level):
    lib = load()
    r = np.ascontiguousarray(recv, dtype=np.uint64)
    s = np.ascontiguousarray(src, dtype=np.uint64)
    bm = np.empty(r.size + 1, dtype=np.int64)
    tot = lib.orc_stencil_segments(_ptr(r), r.size, _ptr(s), s.size, level, bm.ctypes.data,
                                   None, None)
    rk = np.empty(tot, dtype=np.int64)
    cd = np.empty(tot, dtype=np.int16)
    lib.orc_stencil_segments(_ptr(r), r.size, _ptr(s), s.size, level, bm.ctypes.data, _ptr(rk),
                             _ptr(cd))
    return bm, rk, cd


def propagate(boxes):
    b = np.ascontiguousarray(boxes, dtype=np.uint64)
    out = np.empty(b.size, dtype=np.uint64)
    k = load().orc_propagate(_ptr(b), b.size, _ptr(out))
    return out[:k].copy()


def build_all(src, charges, recv, level: int) -> SimpleNamespace:
    """lists.build_all (lists.py:133-187) in deterministic mode."""
    ssrc = sort_points(src, charges, level)
    srecv = sort_points(recv, None, level)
    nb, nl = adjacent_segments(srecv.non_empty_index, ssrc.non_empty_index, level)
    dsrc = {level: ssrc.non_empty_index}
    drecv = {level: srecv.non_empty_index}
    for l in range(level - 1, 1, -1):
        dsrc[l] = propagate(dsrc[l + 1])
        drecv[l] = propagate(drecv[l + 1])
    bm, rk, cd = {}, {}, {}
    for l in range(2, level + 1):
        bm[l], rk[l], cd[l] = stencil_segments(drecv[l], dsrc[l], l)
    return SimpleNamespace(
        max_level=level, sorted_src=ssrc, sorted_recv=srecv,
        neighbor_table=SimpleNamespace(neighbor_bookmark=nb, neighbor_list=nl),
        directory=SimpleNamespace(max_level=level, src_boxes=dsrc, recv_boxes=drecv),
        stencils=SimpleNamespace(bookmark=bm, ranks=rk, codes=cd),
    )


def near_field(src_points, charges, src_bookmark, nbr_bookmark, nbr_list, recv_points,
               recv_bookmark) -> np.ndarray:
    """_ckernels.pyx:290-323 restated (orc_near_field)."""
    sp = np.ascontiguousarray(src_points, dtype=np.float64).reshape(-1, 3)
    rp = np.ascontiguousarray(recv_points, dtype=np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(charges, dtype=np.float64)
    sbm, nbm, nl, rbm = (np.ascontiguousarray(a, dtype=np.int64)
                         for a in (src_bookmark, nbr_bookmark, nbr_list, recv_bookmark))
    phi = np.empty(rp.shape[0], dtype=np.float64)
    load().orc_near_field(_ptr(sp), _ptr(q), _ptr(sbm), _ptr(nbm), _ptr(nl), _ptr(rp),
                          _ptr(rbm), max(0, rbm.shape[0] - 1), rp.shape[0], _ptr(phi))
    return phi


def direct(src_points, charges, recv_points) -> np.ndarray:
    """_ckernels.pyx:326-350 restated (orc_direct)."""
    sp = np.ascontiguousarray(src_points, dtype=np.float64).reshape(-1, 3)
    rp = np.ascontiguousarray(recv_points, dtype=np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(charges, dtype=np.float64)
    phi = np.empty(rp.shape[0], dtype=np.float64)
    load().orc_direct(_ptr(sp), _ptr(q), sp.shape[0], _ptr(rp), rp.shape[0], _ptr(phi))
    return phi
