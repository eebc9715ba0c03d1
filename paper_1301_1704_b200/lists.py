"""Interaction lists and the single-call build (reference:
pkg/src/fmmkit/lists.py).

`build_all` is the drop-in for `fmmkit.build_all` (lists.py:133-187): same
arguments, errors and `FmmStructures` layout.  It runs the fused device
pipeline of libfmmb200 (one C-ABI call, `fmmb_build_all`): sources and
receivers are sorted together, the level directory comes from an occupancy
bitmap pyramid, and the E2 neighbour table and every level's E4 stencil are
produced by one enumeration kernel.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _host, _lib
from .errors import DomainError
from .pseudosort import (
    DEFAULT_HISTOGRAM_BUDGET,
    SortedPointSet,
    _point_set_from_c,
    check_budget,
    check_level,
    check_mode,
    choose_max_level,
    sort_points,
)


@dataclass
class NeighborTable:
    """Per non-empty receiver box, the non-empty source boxes adjacent to it
    (lists.py:21-30): ranks into the source non-empty index, ascending."""

    neighbor_bookmark: object
    neighbor_list: object


@dataclass
class LevelDirectory:
    """Per-level non-empty source/receiver box indices (lists.py:33-42)."""

    max_level: int
    src_boxes: dict
    recv_boxes: dict

    def src_rank(self, level: int, boxes):
        arr = self.src_boxes[level]
        if isinstance(arr, torch.Tensor):
            arr = arr.cpu().numpy()
        return np.searchsorted(arr, np.asarray(boxes, dtype=np.uint64))


@dataclass
class TranslationStencils:
    """Per level: each non-empty receiver box's stencil sources (lists.py:45-55)."""

    bookmark: dict
    ranks: dict
    codes: dict


class BuildSeconds(dict):
    """`build_seconds` with the reference's phase keys (lists.py:174-178),
    measured with CUDA events on the build stream and resolved on first read.

    The device build fuses phases: both point sets are sorted by one pass set
    (reported under sort_sources; sort_receivers is 0.0) and the E2 table and
    all E4 stencils come from the same count/write kernels (reported under
    stencils; neighbor_table is 0.0).  Extra keys split `stencils` into
    lists_count, size_readback (the build's one host sync) and lists_write."""

    def __init__(self, events):
        super().__init__()
        self._events = events

    def _resolve(self):
        ev = self.__dict__.get("_events")
        if ev is None:
            return
        self._events = None
        ev[-1].synchronize()
        s = [ev[i].elapsed_time(ev[i + 1]) * 1e-3 for i in range(len(ev) - 1)]
        super().update(
            sort_sources=s[0], sort_receivers=0.0, neighbor_table=0.0,
            level_directory=s[1], stencils=s[2] + s[3] + s[4],
            lists_count=s[2], size_readback=s[3], lists_write=s[4],
        )

    def __getitem__(self, k):
        self._resolve()
        return super().__getitem__(k)

    def __iter__(self):
        self._resolve()
        return super().__iter__()

    def __len__(self):
        self._resolve()
        return super().__len__()

    def items(self):
        self._resolve()
        return super().items()

    def keys(self):
        self._resolve()
        return super().keys()

    def values(self):
        self._resolve()
        return super().values()

    def get(self, k, d=None):
        self._resolve()
        return super().get(k, d)

    def __repr__(self):
        self._resolve()
        return super().__repr__()


@dataclass
class FmmStructures:
    max_level: int
    sorted_src: SortedPointSet
    sorted_recv: SortedPointSet
    neighbor_table: NeighborTable
    directory: LevelDirectory
    stencils: TranslationStencils
    build_seconds: dict = field(default_factory=dict)
    n_launches: int = 0
    sort_path: str = ""  # "bucket" | "onesweep": strategy the sort phase completed on

    def to_numpy(self) -> "FmmStructures":
        """Host copy in the reference's numpy layout (one sync)."""
        batch = _host.HostBatch()
        src = self.sorted_src.to_numpy(batch)
        recv = self.sorted_recv.to_numpy(batch)

        def conv(v):
            return batch.add(v) if isinstance(v, torch.Tensor) else v

        nb = conv(self.neighbor_table.neighbor_bookmark)
        nl = conv(self.neighbor_table.neighbor_list)
        dsrc = {l: conv(v) for l, v in self.directory.src_boxes.items()}
        drecv = {l: conv(v) for l, v in self.directory.recv_boxes.items()}
        sb = {l: conv(v) for l, v in self.stencils.bookmark.items()}
        sr = {l: conv(v) for l, v in self.stencils.ranks.items()}
        sc = {l: conv(v) for l, v in self.stencils.codes.items()}
        batch.finish()
        src._resolve()
        recv._resolve()

        def npy(v):
            return v.numpy() if isinstance(v, torch.Tensor) else v

        # the finest directory level aliases non_empty_index, as in the reference
        L = self.max_level
        dsrc_np = {l: (src.non_empty_index if l == L else npy(v)) for l, v in dsrc.items()}
        drecv_np = {l: (recv.non_empty_index if l == L else npy(v)) for l, v in drecv.items()}
        return FmmStructures(
            max_level=L,
            sorted_src=src,
            sorted_recv=recv,
            neighbor_table=NeighborTable(npy(nb), npy(nl)),
            directory=LevelDirectory(L, dsrc_np, drecv_np),
            stencils=TranslationStencils({l: npy(v) for l, v in sb.items()},
                                         {l: npy(v) for l, v in sr.items()},
                                         {l: npy(v) for l, v in sc.items()}),
            build_seconds=self.build_seconds,
            n_launches=self.n_launches,
            sort_path=self.sort_path,
        )


def _structures_from_c(sc: "_lib.StructuresC", alloc: _lib.Allocator, with_charges: bool,
                       events) -> FmmStructures:
    L = int(sc.max_level)
    src = _point_set_from_c(sc.src, alloc, L, with_charges)
    recv = _point_set_from_c(sc.recv, alloc, L, False)
    kr = int(sc.recv.k)
    table = NeighborTable(
        neighbor_bookmark=_lib.view(alloc, sc.neighbor_bookmark, kr + 1, "i8"),
        neighbor_list=_lib.view(alloc, sc.neighbor_list, int(sc.n_neighbor), "i8"),
    )
    dsrc = {L: src.non_empty_index}
    drecv = {L: recv.non_empty_index}
    for l in range(L - 1, 1, -1):
        dsrc[l] = _lib.view(alloc, sc.dir_src[l], int(sc.n_dir_src[l]), "u8")
        drecv[l] = _lib.view(alloc, sc.dir_recv[l], int(sc.n_dir_recv[l]), "u8")
    bm, rk, cd = {}, {}, {}
    for l in range(2, L + 1):
        nrl = int(drecv[l].shape[0])
        bm[l] = _lib.view(alloc, sc.st_bookmark[l], nrl + 1, "i8")
        rk[l] = _lib.view(alloc, sc.st_ranks[l], int(sc.n_st[l]), "i8")
        cd[l] = _lib.view(alloc, sc.st_codes[l], int(sc.n_st[l]), "i2")
    return FmmStructures(
        max_level=L,
        sorted_src=src,
        sorted_recv=recv,
        neighbor_table=table,
        directory=LevelDirectory(L, dsrc, drecv),
        stencils=TranslationStencils(bm, rk, cd),
        build_seconds=BuildSeconds(events) if events else {},
        n_launches=int(sc.n_launches),
    )


def build_all_device(src: torch.Tensor, charges: torch.Tensor | None, recv: torch.Tensor,
                     max_level: int, timing: bool = True) -> FmmStructures:
    """Device-resident build: (N,3)/(M,3) f64 CUDA tensors in, CUDA tensors out."""
    dev = _lib.device_of(src.device)
    lib = _lib.load()
    h = _lib.handle(dev)
    n, m = int(src.shape[0]), int(recv.shape[0])
    if charges is not None and int(charges.numel()) != n:
        raise DomainError("charges and source points lengths disagree")
    alloc = _lib.Allocator(dev)
    out = _lib.StructuresC()
    secs = None
    ev_arr = None
    if timing:  # reused event sets (EventRing), resolved lazily
        secs = BuildSeconds(None)
        events, ev_arr = _lib.event_ring(dev).take(secs)
        secs._events = events
    st = lib.fmmb_build_all(
        h, src.data_ptr() if n else None,
        charges.data_ptr() if (charges is not None and n) else None, n,
        recv.data_ptr() if m else None, m, max_level, alloc.fn, None, C.byref(out),
        ev_arr, _lib.stream_of(dev))
    if alloc.error is not None:
        raise alloc.error
    _lib.check(st, h)
    res = _structures_from_c(out, alloc, charges is not None, None)
    if secs is not None:
        res.build_seconds = secs
    res.sort_path = _lib.SORT_PATHS.get(int(lib.fmmb_last_sort_path(h)), "")
    return res


def build_all(
    src_points,
    src_charges,
    recv_points,
    max_level: int | None = None,
    cluster_size: int | None = None,
    mode: str = "deterministic",
    workers: int = 1,
    histogram_budget_bytes: int | None = None,
) -> FmmStructures:
    """Pseudo-sort both point sets and construct every interaction list
    (lists.py:133-187).  Either max_level or cluster_size must be given; an
    explicit max_level wins.  numpy/CPU inputs return numpy outputs; CUDA
    tensor inputs return CUDA tensors (no host round trip)."""
    if max_level is None:
        if cluster_size is None:
            raise DomainError("either max_level or cluster_size is required")
        n_src = src_points.shape[0] if hasattr(src_points, "shape") else len(src_points)
        max_level = choose_max_level(int(n_src), cluster_size)
    check_level(max_level)
    check_budget(max_level, DEFAULT_HISTOGRAM_BUDGET if histogram_budget_bytes is None
                 else histogram_budget_bytes)
    check_mode(mode)
    dev = _host.pick_device(src_points, src_charges, recv_points)
    device_out = _host.is_device_input(src_points, src_charges, recv_points)
    src = _host.points_to_device(src_points, dev)
    q = None if src_charges is None else _host.to_device(src_charges, dev, torch.float64, (-1,))
    recv = _host.points_to_device(recv_points, dev)
    if not _bitmap_path_ok(max_level, src.shape[0] + recv.shape[0]):
        res = _build_all_sparse(src, q, recv, max_level)
    else:
        res = build_all_device(src, q, recv, max_level)
    return res if device_out else res.to_numpy()


def _bitmap_path_ok(level: int, n_total: int) -> bool:
    if level > 12:
        return False
    return (8**level) / 8 <= max(64 * 1024 * 1024, 32 * n_total)


def _build_all_sparse(src, q, recv, max_level) -> FmmStructures:
    """Deep levels with few points (occupancy bitmaps would dwarf the data):
    same outputs from the sorted-search list kernels, level by level.  Phase
    times are CUDA-event intervals on the build stream."""
    from .pseudosort import sort_points_device

    dev = src.device
    stream = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record(stream)
    ssrc = sort_points_device(src, q, max_level)
    ev[1].record(stream)
    srecv = sort_points_device(recv, None, max_level)
    ev[2].record(stream)
    table = build_neighbor_table(ssrc.non_empty_index, srecv.non_empty_index, max_level)
    ev[3].record(stream)
    directory = build_level_directory(ssrc.non_empty_index, srecv.non_empty_index, max_level)
    ev[4].record(stream)
    stencils = build_translation_stencils(directory)
    ev[5].record(stream)
    ev[5].synchronize()
    t = [ev[i].elapsed_time(ev[i + 1]) * 1e-3 for i in range(5)]
    return FmmStructures(
        max_level=max_level, sorted_src=ssrc, sorted_recv=srecv, neighbor_table=table,
        directory=directory, stencils=stencils,
        build_seconds={"sort_sources": t[0], "sort_receivers": t[1],
                       "neighbor_table": t[2], "level_directory": t[3], "stencils": t[4]},
    )


# --------------------------------------------------------------------------
# Unfused sub-builders (lists.py:69-130) on the device plugin kernels.


def build_neighbor_table(src_non_empty, recv_non_empty, level: int) -> NeighborTable:
    from . import kernels

    bm, flat = kernels.adjacent_segments(recv_non_empty, src_non_empty, level)
    return NeighborTable(neighbor_bookmark=bm, neighbor_list=flat)


def gather_adjacent_sources(table: NeighborTable, sorted_src: SortedPointSet, ordinal: int):
    """Concatenated source slices for one receiver box (lists.py:80-100)."""
    nb = table.neighbor_bookmark
    if not 0 <= ordinal < nb.shape[0] - 1:
        raise DomainError(f"receiver ordinal {ordinal} out of range")
    seg = table.neighbor_list[int(nb[ordinal]): int(nb[ordinal + 1])]
    on_dev = isinstance(sorted_src.points, torch.Tensor)
    if seg.shape[0] == 0:
        if on_dev:
            d = sorted_src.points.device
            return (torch.empty((0, 3), dtype=torch.float64, device=d),
                    torch.empty(0, dtype=torch.float64, device=d))
        return np.empty((0, 3), dtype=np.float64), np.empty(0, dtype=np.float64)
    bmk = sorted_src.bookmarks
    if on_dev:
        segs = seg.tolist()
        idx = torch.cat([torch.arange(int(bmk[v]), int(bmk[v + 1]), device=bmk.device)
                         for v in segs])
        q = sorted_src.charges[idx] if sorted_src.charges is not None else \
            torch.ones(idx.shape[0], dtype=torch.float64, device=idx.device)
        return sorted_src.points[idx], q
    idx = np.concatenate([np.arange(bmk[v], bmk[v + 1]) for v in seg])
    q = sorted_src.charges[idx] if sorted_src.charges is not None else np.ones(idx.shape[0])
    return sorted_src.points[idx], q


def propagate_to_parents(boxes):
    """Ascending unique parents of an ascending box index array (lists.py:103-105)."""
    from . import kernels

    return kernels.propagate_to_parents(boxes)


def build_level_directory(src_boxes_finest, recv_boxes_finest, max_level: int) -> LevelDirectory:
    """lists.py:108-116."""
    src = {max_level: src_boxes_finest}
    recv = {max_level: recv_boxes_finest}
    if not isinstance(src_boxes_finest, torch.Tensor):
        src[max_level] = np.asarray(src_boxes_finest, dtype=np.uint64)
    if not isinstance(recv_boxes_finest, torch.Tensor):
        recv[max_level] = np.asarray(recv_boxes_finest, dtype=np.uint64)
    for level in range(max_level - 1, 1, -1):
        src[level] = propagate_to_parents(src[level + 1])
        recv[level] = propagate_to_parents(recv[level + 1])
    return LevelDirectory(max_level=max_level, src_boxes=src, recv_boxes=recv)


def build_translation_stencils(directory: LevelDirectory) -> TranslationStencils:
    """lists.py:119-130."""
    from . import kernels

    bookmark, ranks, codes = {}, {}, {}
    for level in range(2, directory.max_level + 1):
        bm, rk, cd = kernels.stencil_segments(
            directory.recv_boxes[level], directory.src_boxes[level], level)
        bookmark[level] = bm
        ranks[level] = rk
        codes[level] = cd
    return TranslationStencils(bookmark=bookmark, ranks=ranks, codes=codes)


# ------------------------------------------------------- FMMS dump / load
def _point_set_arrays(ps: SortedPointSet, prefix: str) -> dict:
    """lists.py:190-200 (same names and order)."""
    arrays = {
        f"{prefix}_points": ps.points,
        f"{prefix}_permutation": ps.permutation,
        f"{prefix}_bookmarks": ps.bookmarks,
        f"{prefix}_non_empty": ps.non_empty_index,
        f"{prefix}_boxes": ps.boxes,
    }
    if ps.charges is not None:
        arrays[f"{prefix}_charges"] = ps.charges
    return arrays


def dump_structures(structures: FmmStructures, path) -> None:
    """Write the CORE / LVLS / STNC container of lists.py:203-219, byte-
    identical to the reference; device-resident structures are streamed out
    of HBM in chunks (container.write_container)."""
    from . import container

    L = structures.max_level
    core = container.Section(tag="CORE", meta={"max_level": L})
    core.arrays.update(_point_set_arrays(structures.sorted_src, "src"))
    core.arrays.update(_point_set_arrays(structures.sorted_recv, "recv"))
    core.arrays["neighbor_bookmark"] = structures.neighbor_table.neighbor_bookmark
    core.arrays["neighbor_list"] = structures.neighbor_table.neighbor_list
    lvls = container.Section(tag="LVLS", meta={"max_level": L})
    for level in range(2, L + 1):
        lvls.arrays[f"src_{level}"] = structures.directory.src_boxes[level]
        lvls.arrays[f"recv_{level}"] = structures.directory.recv_boxes[level]
    stnc = container.Section(tag="STNC")
    for level in range(2, L + 1):
        stnc.arrays[f"bookmark_{level}"] = structures.stencils.bookmark[level]
        stnc.arrays[f"ranks_{level}"] = structures.stencils.ranks[level]
        stnc.arrays[f"codes_{level}"] = structures.stencils.codes[level]
    container.write_container(path, L, [core, lvls, stnc])


def load_structures(path, device=None) -> FmmStructures:
    """lists.py:234-257; with `device` the arrays are uploaded to it."""
    from . import container

    max_level, sections = container.read_container(path, device=device)
    by_tag = {s.tag: s for s in sections}
    core, lvls, stnc = by_tag["CORE"], by_tag["LVLS"], by_tag["STNC"]
    L = max_level
    directory = LevelDirectory(
        max_level=L,
        src_boxes={l: lvls.arrays[f"src_{l}"] for l in range(2, L + 1)},
        recv_boxes={l: lvls.arrays[f"recv_{l}"] for l in range(2, L + 1)},
    )
    stencils = TranslationStencils(
        bookmark={l: stnc.arrays[f"bookmark_{l}"] for l in range(2, L + 1)},
        ranks={l: stnc.arrays[f"ranks_{l}"] for l in range(2, L + 1)},
        codes={l: stnc.arrays[f"codes_{l}"] for l in range(2, L + 1)},
    )

    def ps(prefix):
        a = core.arrays
        return SortedPointSet(level=L, points=a[f"{prefix}_points"],
                              charges=a.get(f"{prefix}_charges"),
                              permutation=a[f"{prefix}_permutation"],
                              bookmarks=a[f"{prefix}_bookmarks"],
                              non_empty_index=a[f"{prefix}_non_empty"], boxes=a[f"{prefix}_boxes"])

    return FmmStructures(
        max_level=L, sorted_src=ps("src"), sorted_recv=ps("recv"),
        neighbor_table=NeighborTable(neighbor_bookmark=core.arrays["neighbor_bookmark"],
                                     neighbor_list=core.arrays["neighbor_list"]),
        directory=directory, stencils=stencils)
