"""Fixed-grid pseudo-sort API (reference: pkg/src/fmmkit/pseudosort.py).

Same names, arguments, errors and output layout as the reference; the work
runs in libfmmb200 (K1 encode, K2 stable LSD radix sort, K3/K4 gather +
bookmarks) instead of the reference's dense 8^L histogram.  Within-box order
is the input order in every mode, which is the reference's deterministic
contract and a legal order for its "atomic" mode (pseudosort.py:59-64).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _host, _lib
from .errors import CapacityError, DomainError

MAX_LEVEL = _lib.MAX_LEVEL
DEFAULT_HISTOGRAM_BUDGET = 2 << 30  # bytes (pseudosort.py:19)
MODES = ("deterministic", "atomic")


def choose_max_level(n_points: int, cluster_size: int) -> int:
    """Smallest level whose average box occupancy is at most cluster_size
    (pseudosort.py:22-29)."""
    if cluster_size < 1:
        raise DomainError("cluster size must be positive")
    level = 0
    while level < MAX_LEVEL and -(-n_points // (8**level)) > cluster_size:
        level += 1
    return level


def check_level(max_level: int) -> None:
    """pseudosort.py:53-54: level outside [0, MAX_LEVEL] is a CapacityError."""
    if max_level < 0 or max_level > MAX_LEVEL:
        raise CapacityError(f"max_level {max_level} outside [0, {MAX_LEVEL}]")


def check_budget(level: int, budget_bytes: int) -> None:
    """pseudosort.py:32-38.  The device build needs no dense histogram; the
    check is kept so the accepted (level, budget) pairs and the error are the
    reference's."""
    need = (8**level) * 8
    if need > budget_bytes:
        raise CapacityError(
            f"dense histogram for level {level} needs {need} bytes, "
            f"exceeding the configured budget of {budget_bytes}"
        )


def check_mode(mode: str) -> None:
    if mode not in MODES:
        raise DomainError(f"unknown pseudo-sort mode {mode!r}")


@dataclass
class SortedPointSet:
    """Box-grouped points with bookmarks into the grouped array
    (pseudosort.py:81-102).  Arrays are numpy (host inputs) or CUDA tensors."""

    level: int
    points: object  # (N, 3), grouped by box, boxes ascending
    charges: object  # (N,) strengths, same order, or None
    permutation: object  # sorted position -> original position
    bookmarks: object  # (K+1,)
    non_empty_index: object  # (K,) ascending Morton indices
    boxes: object = field(repr=False, default=None)  # (N,) per sorted point

    @property
    def num_points(self) -> int:
        return int(self.points.shape[0])

    @property
    def num_boxes(self) -> int:
        return int(self.non_empty_index.shape[0])

    def box_slice(self, ordinal: int) -> slice:
        return slice(int(self.bookmarks[ordinal]), int(self.bookmarks[ordinal + 1]))

    def _fields(self):
        return ("points", "charges", "permutation", "bookmarks", "non_empty_index", "boxes")

    def to_numpy(self, batch: _host.HostBatch | None = None) -> "SortedPointSet":
        own = batch is None
        batch = batch or _host.HostBatch()
        hosts = {}
        for f in self._fields():
            v = getattr(self, f)
            hosts[f] = batch.add(v) if isinstance(v, torch.Tensor) else v
        out = SortedPointSet(level=self.level, **{f: None for f in self._fields()})
        if own:
            batch.finish()
            for f, h in hosts.items():
                setattr(out, f, h.numpy() if isinstance(h, torch.Tensor) else h)
            return out
        out._pending = hosts  # resolved by the caller after batch.finish()
        return out

    def _resolve(self) -> None:
        for f, h in self.__dict__.pop("_pending").items():
            setattr(self, f, h.numpy() if isinstance(h, torch.Tensor) else h)


def _point_set_from_c(ps: "_lib.PointSetC", alloc: _lib.Allocator, level: int,
                      with_charges: bool) -> SortedPointSet:
    n, k = int(ps.n), int(ps.k)
    return SortedPointSet(
        level=level,
        points=_lib.view(alloc, ps.points, 3 * n, "f8", (n, 3)),
        charges=_lib.view(alloc, ps.charges, n, "f8") if with_charges else None,
        permutation=_lib.view(alloc, ps.permutation, n, "i8"),
        bookmarks=_lib.view(alloc, ps.bookmarks, k + 1, "i8"),
        non_empty_index=_lib.view(alloc, ps.non_empty, k, "u8"),
        boxes=_lib.view(alloc, ps.boxes, n, "u8"),
    )


def sort_points_device(points: torch.Tensor, charges: torch.Tensor | None, max_level: int
                       ) -> SortedPointSet:
    """The device path of sort_points: (N,3) f64 CUDA tensor in, CUDA out."""
    dev = _lib.device_of(points.device)
    lib = _lib.load()
    h = _lib.handle(dev)
    n = int(points.shape[0])
    if charges is not None and int(charges.numel()) != n:
        raise DomainError("charges and points lengths disagree")
    alloc = _lib.Allocator(dev)
    out = _lib.PointSetC()
    st = lib.fmmb_sort_points(
        h, points.data_ptr() if n else None,
        charges.data_ptr() if (charges is not None and n) else None, n, max_level,
        alloc.fn, None, C.byref(out), _lib.stream_of(dev))
    if alloc.error is not None:
        raise alloc.error
    _lib.check(st, h)
    return _point_set_from_c(out, alloc, max_level, charges is not None)


def sort_points(
    points,
    charges,
    max_level: int,
    mode: str = "deterministic",
    workers: int = 1,
    histogram_budget_bytes: int = DEFAULT_HISTOGRAM_BUDGET,
) -> SortedPointSet:
    """Group points by their level-`max_level` Morton box (pseudosort.py:138-151).

    `workers` only affects the reference's atomic mode; the device sort is
    deterministic (input order within each box) in both modes."""
    check_level(max_level)
    check_budget(max_level, histogram_budget_bytes)
    check_mode(mode)
    dev = _host.pick_device(points, charges)
    device_out = _host.is_device_input(points, charges)
    pts = _host.points_to_device(points, dev)
    q = None if charges is None else _host.to_device(charges, dev, torch.float64, (-1,))
    res = sort_points_device(pts, q, max_level)
    return res if device_out else res.to_numpy()


# --------------------------------------------------------------------------
# Unfused reference steps (histogram_and_sort_index, build_bookmarks,
# reorder): device implementations of the same contracts.


def histogram_and_sort_index(
    points,
    max_level: int,
    mode: str = "deterministic",
    workers: int = 1,
    histogram_budget_bytes: int = DEFAULT_HISTOGRAM_BUDGET,
):
    """(bins dense over 8^L, boxes[i], ranks[i]) (pseudosort.py:41-65)."""
    from . import kernels

    check_level(max_level)
    check_budget(max_level, histogram_budget_bytes)
    dev = _host.pick_device(points)
    device_out = _host.is_device_input(points)
    pts = _host.points_to_device(points, dev)
    boxes = kernels.encode_points_device(pts[:, 0], pts[:, 1], pts[:, 2], max_level)
    check_mode(mode)
    bins, ranks = kernels.assign_box_ranks_device(boxes, 8**max_level)
    if device_out:
        return bins, boxes, ranks
    return bins.cpu().numpy(), boxes.cpu().numpy(), ranks.cpu().numpy()


def build_bookmarks(bins):
    """Compact a dense histogram to (bookmarks, non-empty indices) (pseudosort.py:68-78)."""
    from . import kernels

    return kernels.build_bookmarks(bins)


def reorder(points, charges, bins, boxes, ranks, max_level: int) -> SortedPointSet:
    """Copy points into box-grouped order using a (bins, boxes, ranks) sort
    index (pseudosort.py:105-135)."""
    from . import kernels

    return kernels.reorder(points, charges, bins, boxes, ranks, max_level)
