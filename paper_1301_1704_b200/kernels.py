"""Drop-in for the reference kernel plugin `fmmkit.backend.kernels`.

Same module surface as pkg/src/fmmkit/_ckernels.pyx and _pykernels.py
(IS_COMPILED, spread_bits, compact_bits, interleave_coords,
deinterleave_indices, encode_points, assign_box_ranks,
assign_box_ranks_atomic, adjacent_segments, stencil_segments, near_field,
direct_potentials), every function computed by libfmmb200 on the GPU.
numpy in -> numpy out (the reference contract); CUDA tensors in -> CUDA
tensors out.  Bind it into the reference with `install()` (the reference's
own swap mechanism is plain assignment, cli.py:263-266).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _host, _lib
from .errors import DomainError

IS_COMPILED = True  # backend.backend_name() reports "compiled" (backend.py:30-32)


def _dev_u64(a, dev):
    return _host.to_device(a, dev, torch.uint64, (-1,))


def _out(t: torch.Tensor, device_out: bool):
    return t if device_out else t.cpu().numpy()


def _call(fn_name: str, dev, *args):
    lib = _lib.load()
    h = _lib.handle(dev)
    st = getattr(lib, fn_name)(h, *args, _lib.stream_of(dev))
    _lib.check(st, h)


def _ptr(t: torch.Tensor):
    return t.data_ptr() if t.numel() else None


# ----------------------------------------------------------- bit dilation
def _shape(a) -> tuple:
    """Elementwise plugin functions keep the input's shape (numpy semantics
    of _pykernels.py:22-57, e.g. (B, 27) candidate grids in partition.py)."""
    return tuple(a.shape) if hasattr(a, "shape") else tuple(np.shape(a))


def _unary_u64(fn_name: str, v):
    dev = _host.pick_device(v)
    dout = _host.is_device_input(v)
    shp = _shape(v)
    x = _dev_u64(v, dev)
    o = torch.empty_like(x)
    _call(fn_name, dev, _ptr(x), x.numel(), _ptr(o))
    return _out(o.reshape(shp), dout)


def spread_bits(v):
    """Insert two zero bits between each of the low 21 bits (_pykernels.py:22-30)."""
    return _unary_u64("fmmb_spread_bits", v)


def compact_bits(v):
    """Inverse of spread_bits on bits 3k (_pykernels.py:33-40)."""
    return _unary_u64("fmmb_compact_bits", v)


def interleave_coords(ix, iy, iz):
    """Morton index from box coordinates (_pykernels.py:43-48)."""
    dev = _host.pick_device(ix, iy, iz)
    dout = _host.is_device_input(ix, iy, iz)
    shp = np.broadcast_shapes(_shape(ix), _shape(iy), _shape(iz))
    xs = [_dev_u64(np.broadcast_to(a, shp) if not isinstance(a, torch.Tensor) else
                   a.expand(shp), dev) for a in (ix, iy, iz)]
    n = xs[0].numel()
    o = torch.empty(n, dtype=torch.uint64, device=dev)
    _call("fmmb_interleave_coords", dev, *[_ptr(t) for t in xs], n, _ptr(o))
    return _out(o.reshape(shp), dout)


def deinterleave_indices(idx):
    """(ix, iy, iz) from Morton indices (_pykernels.py:51-57)."""
    dev = _host.pick_device(idx)
    dout = _host.is_device_input(idx)
    shp = _shape(idx)
    k = _dev_u64(idx, dev)
    outs = [torch.empty_like(k) for _ in range(3)]
    _call("fmmb_deinterleave_indices", dev, _ptr(k), k.numel(), *[_ptr(t) for t in outs])
    return tuple(_out(t.reshape(shp), dout) for t in outs)


# --------------------------------------------------------------- encoding
def encode_points_device(x: torch.Tensor, y: torch.Tensor, z: torch.Tensor, level: int):
    """Morton keys of (possibly strided) f64 CUDA columns."""
    dev = _lib.device_of(x.device)
    n = x.numel()
    cols = []
    for c in (x, y, z):
        if c.dtype != torch.float64 or c.dim() != 1:
            c = c.reshape(-1).to(torch.float64)
        cols.append(c)
    o = torch.empty(n, dtype=torch.uint64, device=dev)
    args = []
    for c in cols:
        args += [_ptr(c), c.stride(0) if c.numel() else 1]
    _call("fmmb_encode_points", dev, *args, n, level, _ptr(o))
    return o


def encode_points(x, y, z, level: int):
    """Morton index of the level-`level` box containing each point
    (_ckernels.pyx:85-104): truncating f64 quantisation, upper clamp."""
    dev = _host.pick_device(x, y, z)
    dout = _host.is_device_input(x, y, z)
    shp = _shape(x)
    cols = [_host.to_device(c, dev, torch.float64, (-1,)) for c in (x, y, z)]
    if not (cols[0].numel() == cols[1].numel() == cols[2].numel()):
        raise DomainError("encode_points: coordinate arrays differ in length")
    return _out(encode_points_device(*cols, level).reshape(shp), dout)


# ---------------------------------------------------------- rank assignment
def assign_box_ranks_device(boxes: torch.Tensor, nbins: int):
    dev = _lib.device_of(boxes.device)
    n = boxes.numel()
    bins = torch.empty(nbins, dtype=torch.int64, device=dev)
    ranks = torch.empty(n, dtype=torch.int64, device=dev)
    _call("fmmb_assign_box_ranks", dev, _ptr(boxes), n, nbins, _ptr(bins), _ptr(ranks))
    return bins, ranks


def assign_box_ranks(boxes, nbins: int):
    """Dense occupancy histogram plus each point's arrival rank within its box
    (_ckernels.pyx:107-119)."""
    dev = _host.pick_device(boxes)
    dout = _host.is_device_input(boxes)
    b = _dev_u64(boxes, dev)
    bins, ranks = assign_box_ranks_device(b, int(nbins))
    return _out(bins, dout), _out(ranks, dout)


def assign_box_ranks_atomic(boxes, nbins: int, threads: int = 1):
    """The reference's shared-counter variant (_ckernels.pyx:122-137) allows
    any within-box order; the deterministic order is a legal one
    (_pykernels.py:90-95 makes the same choice)."""
    return assign_box_ranks(boxes, nbins)


# ---------------------------------------------------------- list builders
def _segments(fn_name: str, recv_boxes, src_boxes, level: int, stencil: bool):
    dev = _host.pick_device(recv_boxes, src_boxes)
    dout = _host.is_device_input(recv_boxes, src_boxes)
    r = _dev_u64(recv_boxes, dev)
    s = _dev_u64(src_boxes, dev)
    nr, ns = r.numel(), s.numel()
    bm = torch.empty(nr + 1, dtype=torch.int64, device=dev)
    alloc = _lib.Allocator(dev)
    lst = C.c_void_p()
    codes = C.c_void_p()
    total = C.c_int64()
    lib = _lib.load()
    h = _lib.handle(dev)
    if stencil:
        st = lib.fmmb_stencil_segments(h, _ptr(r), nr, _ptr(s), ns, level, _ptr(bm), alloc.fn,
                                       None, C.byref(lst), C.byref(codes), C.byref(total),
                                       _lib.stream_of(dev))
    else:
        st = lib.fmmb_adjacent_segments(h, _ptr(r), nr, _ptr(s), ns, level, _ptr(bm), alloc.fn,
                                        None, C.byref(lst), C.byref(total), _lib.stream_of(dev))
    if alloc.error is not None:
        raise alloc.error
    _lib.check(st, h)
    e = int(total.value)
    flat = _lib.view(alloc, lst.value, e, "i8")
    if not stencil:
        return _out(bm, dout), _out(flat, dout)
    cd = _lib.view(alloc, codes.value, e, "i2")
    return _out(bm, dout), _out(flat, dout), _out(cd, dout)


def adjacent_segments(recv_boxes, src_boxes, level: int):
    """Per receiver box, the ranks into src_boxes of its in-grid 3x3x3 window
    members present in src_boxes, ascending (_ckernels.pyx:172-202)."""
    return _segments("fmmb_adjacent_segments", recv_boxes, src_boxes, level, False)


def stencil_segments(recv_boxes, src_boxes, level: int):
    """Translation-stencil segments (bookmark, ranks, i16 offset codes)
    (_ckernels.pyx:205-287)."""
    return _segments("fmmb_stencil_segments", recv_boxes, src_boxes, level, True)


# ------------------------------------------------------ directory helpers
def propagate_to_parents(boxes):
    """Ascending unique parents (lists.py:103-105)."""
    dev = _host.pick_device(boxes)
    dout = _host.is_device_input(boxes)
    b = _dev_u64(boxes, dev)
    out = torch.empty(max(b.numel(), 1), dtype=torch.uint64, device=dev)
    cnt = C.c_int64(0)
    _call("fmmb_propagate_to_parents", dev, _ptr(b), b.numel(), _ptr(out), C.byref(cnt))
    return _out(out[: int(cnt.value)], dout)


def exclusive_scan(values):
    """(exclusive prefix sums, total) of non-negative integers (scan.py:25-73)."""
    dev = _host.pick_device(values)
    dout = _host.is_device_input(values)
    v = _host.to_device(values, dev, torch.int64, (-1,))
    if v.numel() == 0:
        raise DomainError("scan input must be a non-empty 1-d array")
    out = torch.empty_like(v)
    tot = C.c_int64(0)
    _call("fmmb_exclusive_scan_i64", dev, _ptr(v), v.numel(), _ptr(out), C.byref(tot))
    return _out(out, dout), int(tot.value)


def build_bookmarks(bins):
    """(bookmarks, non-empty box indices) from a dense histogram
    (pseudosort.py:68-78): fmmb_build_bookmarks (flag scan + compaction on
    the device)."""
    dev = _host.pick_device(bins)
    dout = _host.is_device_input(bins)
    b = _host.to_device(bins, dev, torch.int64, (-1,))
    lib = _lib.load()
    h = _lib.handle(dev)
    alloc = _lib.Allocator(dev)
    bm_p, ne_p, k = C.c_void_p(), C.c_void_p(), C.c_int64(0)
    st = lib.fmmb_build_bookmarks(h, _ptr(b), b.numel(), alloc.fn, None, C.byref(bm_p),
                                  C.byref(ne_p), C.byref(k), _lib.stream_of(dev))
    if alloc.error is not None:
        raise alloc.error
    _lib.check(st, h)
    kk = int(k.value)
    bm = _lib.view(alloc, bm_p.value, kk + 1, "i8")
    ne = _lib.view(alloc, ne_p.value, kk, "u8")
    return _out(bm, dout), _out(ne, dout)


def reorder(points, charges, bins, boxes, ranks, max_level: int):
    """Box-grouped copy from a (bins, boxes, ranks) sort index
    (pseudosort.py:105-135): fmmb_reorder (permutation scatter, gather of
    points / charges / boxes, bookmarks) on the device."""
    from .pseudosort import _point_set_from_c

    dev = _host.pick_device(points, charges, bins, boxes, ranks)
    dout = _host.is_device_input(points, charges, bins, boxes, ranks)
    pts = _host.points_to_device(points, dev)
    n = pts.shape[0]
    bx = _dev_u64(boxes, dev)
    rk = _host.to_device(ranks, dev, torch.int64, (-1,))
    if bx.numel() != n or rk.numel() != n:
        raise DomainError("points and sort index lengths disagree")
    bn = _host.to_device(bins, dev, torch.int64, (-1,))
    if bn.numel() == 0:
        if n:
            raise DomainError("box index outside [0, nbins)")
        bn = torch.zeros(1, dtype=torch.int64, device=dev)  # same (empty) outputs
    q = None
    if charges is not None:
        q = _host.to_device(charges, dev, torch.float64, (-1,))
        if q.numel() < n:
            raise DomainError("charges shorter than points")
    lib = _lib.load()
    h = _lib.handle(dev)
    alloc = _lib.Allocator(dev)
    out = _lib.PointSetC()
    st = lib.fmmb_reorder(h, _ptr(pts), _ptr(q) if q is not None else None, n, _ptr(bn),
                          bn.numel(), _ptr(bx), _ptr(rk), int(max_level), alloc.fn, None,
                          C.byref(out), _lib.stream_of(dev))
    if alloc.error is not None:
        raise alloc.error
    _lib.check(st, h)
    res = _point_set_from_c(out, alloc, max_level, q is not None)
    return res if dout else res.to_numpy()


# ------------------------------------------------- evaluation (not the path)
def _f64_col(c, dev):
    """1-D f64 CUDA view (strided columns of an (N,3) tensor are kept as is)."""
    if isinstance(c, torch.Tensor) and c.is_cuda and c.dtype == torch.float64 and c.dim() == 1:
        return c
    return _host.to_device(c, dev, torch.float64, (-1,))


def _strided(c):
    return [_ptr(c), c.stride(0) if c.numel() else 1]


def near_field_device(sx, sy, sz, sq, src_bookmark, nbr_bookmark, nbr_list, rx, ry, rz,
                      recv_bookmark) -> torch.Tensor:
    """near_field on CUDA tensors (columns may be strided views); phi f64[M]."""
    dev = _lib.device_of(sx.device)
    cols_s = [_f64_col(c, dev) for c in (sx, sy, sz)]
    cols_r = [_f64_col(c, dev) for c in (rx, ry, rz)]
    q = _host.to_device(sq, dev, torch.float64, (-1,)) if sq is not None else None
    sbm, nbm, nl, rbm = (_host.to_device(a, dev, torch.int64, (-1,))
                         for a in (src_bookmark, nbr_bookmark, nbr_list, recv_bookmark))
    ns, nr = cols_s[0].numel(), cols_r[0].numel()
    if cols_s[1].numel() != ns or cols_s[2].numel() != ns or (q is not None and q.numel() != ns):
        raise DomainError("near_field: source arrays differ in length")
    if cols_r[1].numel() != nr or cols_r[2].numel() != nr:
        raise DomainError("near_field: receiver arrays differ in length")
    if nbm.numel() != rbm.numel():
        raise DomainError("near_field: neighbour and receiver bookmarks differ in length")
    phi = torch.empty(nr, dtype=torch.float64, device=dev)
    kr = max(0, rbm.numel() - 1)
    _call("fmmb_near_field", dev, *_strided(cols_s[0]), *_strided(cols_s[1]),
          *_strided(cols_s[2]), _ptr(q) if q is not None else None, ns, _ptr(sbm),
          max(0, sbm.numel() - 1), _ptr(nbm), _ptr(nl), nl.numel(), *_strided(cols_r[0]),
          *_strided(cols_r[1]), *_strided(cols_r[2]), nr, _ptr(rbm), kr, _ptr(phi))
    return phi


def near_field(sx, sy, sz, sq, src_bookmark, nbr_bookmark, nbr_list, rx, ry, rz,
               recv_bookmark):
    """Near-field direct sums over each receiver box's neighbour segments
    (_ckernels.pyx:290-323): bit-identical to the compiled backend."""
    args = (sx, sy, sz, sq, src_bookmark, nbr_bookmark, nbr_list, rx, ry, rz, recv_bookmark)
    dout = _host.is_device_input(*args)
    dev = _host.pick_device(*args)
    kinds = (torch.float64,) * 4 + (torch.int64,) * 3 + (torch.float64,) * 3 + (torch.int64,)
    cols = [a if (isinstance(a, torch.Tensor) and a.is_cuda) or a is None
            else _host.to_device(a, dev, k, (-1,)) for a, k in zip(args, kinds)]
    return _out(near_field_device(*cols), dout)


def direct_potentials_device(sx, sy, sz, sq, rx, ry, rz) -> torch.Tensor:
    dev = _lib.device_of(sx.device)
    cols_s = [_f64_col(c, dev) for c in (sx, sy, sz)]
    cols_r = [_f64_col(c, dev) for c in (rx, ry, rz)]
    q = _host.to_device(sq, dev, torch.float64, (-1,))
    ns, nr = cols_s[0].numel(), cols_r[0].numel()
    if cols_s[1].numel() != ns or cols_s[2].numel() != ns or q.numel() != ns:
        raise DomainError("direct_potentials: source arrays differ in length")
    if cols_r[1].numel() != nr or cols_r[2].numel() != nr:
        raise DomainError("direct_potentials: receiver arrays differ in length")
    phi = torch.empty(nr, dtype=torch.float64, device=dev)
    _call("fmmb_direct_potentials", dev, *_strided(cols_s[0]), *_strided(cols_s[1]),
          *_strided(cols_s[2]), _ptr(q), ns, *_strided(cols_r[0]), *_strided(cols_r[1]),
          *_strided(cols_r[2]), nr, _ptr(phi))
    return phi


def direct_potentials(sx, sy, sz, sq, rx, ry, rz, chunk: int = 1024, threads: int = 1):
    """Brute-force sums, sequential over sources per receiver
    (_ckernels.pyx:326-350).  `chunk` / `threads` do not change the result
    (the reference's receiver blocking / OpenMP width) and are ignored."""
    args = (sx, sy, sz, sq, rx, ry, rz)
    dout = _host.is_device_input(*args)
    dev = _host.pick_device(*args)
    cols = [a if (isinstance(a, torch.Tensor) and a.is_cuda)
            else _host.to_device(a, dev, torch.float64, (-1,)) for a in args]
    return _out(direct_potentials_device(*cols), dout)


def install(fmmkit_module=None):
    """Bind this module as the reference's kernel plugin
    (`fmmkit.backend.kernels = kernels`, the swap of cli.py:263-266)."""
    import sys

    if fmmkit_module is None:
        import fmmkit as fmmkit_module  # noqa: F811 - the caller's reference
    fmmkit_module.backend.kernels = sys.modules[__name__]
    return sys.modules[__name__]
