"""ctypes binding of libfmmb200.so (C ABI: include/fmmb200.h).

The shared library is built in-tree (``paper_1301_1704_b200/libfmmb200.so``)
by ``__graft_entry__.build()`` / ``make -C paper_1301_1704_b200/csrc``.  There
is no fallback: if the library or a GPU is missing, every compute entry point
raises :class:`NativeError`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

from .errors import CapacityError, DomainError, NativeError

MAX_LEVEL = 20
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FMMB_LIB") or os.path.join(_HERE, "libfmmb200.so")  # FMMB_LIB: A/B builds

OK, ERR_DOMAIN, ERR_CAPACITY, ERR_CUDA, ERR_ALLOC, ERR_ARG = range(6)

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_uint64)
_p = C.c_void_p
_i64 = C.c_int64


class PointSetC(C.Structure):
    _fields_ = [
        ("points", _p), ("charges", _p), ("permutation", _p), ("bookmarks", _p),
        ("non_empty", _p), ("boxes", _p), ("n", _i64), ("k", _i64),
    ]


_L = MAX_LEVEL + 1


class StructuresC(C.Structure):
    _fields_ = [
        ("max_level", C.c_int32), ("_pad", C.c_int32),
        ("src", PointSetC), ("recv", PointSetC),
        ("neighbor_bookmark", _p), ("neighbor_list", _p), ("n_neighbor", _i64),
        ("dir_src", _p * _L), ("dir_recv", _p * _L),
        ("n_dir_src", _i64 * _L), ("n_dir_recv", _i64 * _L),
        ("st_bookmark", _p * _L), ("st_ranks", _p * _L), ("st_codes", _p * _L),
        ("n_st", _i64 * _L),
        ("n_launches", _i64),
    ]


# (name, restype, argtypes) for every symbol in include/fmmb200.h
SIGNATURES = [
    ("fmmb_abi_version", C.c_int, []),
    ("fmmb_create", C.c_int, [C.c_int, C.POINTER(_p)]),
    ("fmmb_destroy", C.c_int, [_p]),
    ("fmmb_last_error", C.c_char_p, [_p]),
    ("fmmb_last_launch_count", _i64, [_p]),
    ("fmmb_set_sort_path", C.c_int, [_p, C.c_int]),
    ("fmmb_last_sort_path", C.c_int, [_p]),
    ("fmmb_set_overlap", C.c_int, [_p, C.c_int]),
    ("fmmb_trace", C.c_int, [_p, C.POINTER(C.c_float), C.POINTER(C.c_char_p), C.c_int]),
    ("fmmb_spread_bits", C.c_int, [_p, _p, _i64, _p, _p]),
    ("fmmb_compact_bits", C.c_int, [_p, _p, _i64, _p, _p]),
    ("fmmb_interleave_coords", C.c_int, [_p, _p, _p, _p, _i64, _p, _p]),
    ("fmmb_deinterleave_indices", C.c_int, [_p, _p, _i64, _p, _p, _p, _p]),
    ("fmmb_encode_points", C.c_int, [_p, _p, _i64, _p, _i64, _p, _i64, _i64, C.c_int, _p, _p]),
    ("fmmb_assign_box_ranks", C.c_int, [_p, _p, _i64, _i64, _p, _p, _p]),
    ("fmmb_adjacent_segments", C.c_int,
     [_p, _p, _i64, _p, _i64, C.c_int, _p, ALLOC_FN, _p, C.POINTER(_p), C.POINTER(_i64), _p]),
    ("fmmb_stencil_segments", C.c_int,
     [_p, _p, _i64, _p, _i64, C.c_int, _p, ALLOC_FN, _p, C.POINTER(_p), C.POINTER(_p),
      C.POINTER(_i64), _p]),
    ("fmmb_propagate_to_parents", C.c_int, [_p, _p, _i64, _p, C.POINTER(_i64), _p]),
    ("fmmb_exclusive_scan_i64", C.c_int, [_p, _p, _i64, _p, C.POINTER(_i64), _p]),
    ("fmmb_build_bookmarks", C.c_int,
     [_p, _p, _i64, ALLOC_FN, _p, C.POINTER(_p), C.POINTER(_p), C.POINTER(_i64), _p]),
    ("fmmb_reorder", C.c_int,
     [_p, _p, _p, _i64, _p, _i64, _p, _p, C.c_int, ALLOC_FN, _p, C.POINTER(PointSetC), _p]),
    ("fmmb_perturb", C.c_int, [_p, _p, _i64, C.c_uint64, C.c_uint64, C.c_double, _p]),
    ("fmmb_build_all", C.c_int,
     [_p, _p, _p, _i64, _p, _i64, C.c_int, ALLOC_FN, _p, C.POINTER(StructuresC), _p, _p]),
    ("fmmb_sort_points", C.c_int,
     [_p, _p, _p, _i64, C.c_int, ALLOC_FN, _p, C.POINTER(PointSetC), _p]),
    ("fmmb_part_histogram", C.c_int, [_p, _p, _i64, _p, _i64, C.c_int, C.c_int, _p, _p]),
    ("fmmb_part_pack", C.c_int,
     [_p, _p, _p, _i64, _p, _i64, C.c_int, C.c_int, _p, C.c_int, _i64, _i64, _p, _p, _p, _p,
      _p, C.POINTER(_i64), _p]),
    ("fmmb_part_counts", C.c_int,
     [_p, _p, _i64, _p, _i64, C.c_int, C.c_int, _p, C.c_int, C.POINTER(_i64), _p]),
    ("fmmb_part_pack_peer", C.c_int,
     [_p, _p, _p, _i64, _p, _i64, C.c_int, C.c_int, _p, C.c_int, _i64, _i64,
      C.POINTER(_p), C.POINTER(_p), C.POINTER(_p), C.POINTER(_p), C.POINTER(_p),
      C.POINTER(_i64), C.POINTER(_i64), _p]),
    ("fmmb_dist_sort", C.c_int,
     [_p, _p, _p, _i64, _p, _p, _i64, _p, C.c_int, ALLOC_FN, _p, C.POINTER(PointSetC),
      C.POINTER(PointSetC), _p, _p]),
    ("fmmb_dist_join", C.c_int, [_p, _p]),
    ("fmmb_dist_lists", C.c_int,
     [_p, _p, C.c_int, C.c_uint64, C.c_uint64, ALLOC_FN, _p, C.POINTER(StructuresC), _p]),
    ("fmmb_near_field", C.c_int,
     [_p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _p, _i64, _p, _i64, _p, _i64,
      _p, _i64, _i64, _p, _i64, _p, _p]),
    ("fmmb_classify_boxes", C.c_int,
     [_p, _p, _i64, C.c_int, _p, _i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _p, _p]),
    ("fmmb_partition_level", C.c_int,
     [_p, _p, _p, _i64, C.c_int, C.c_int, _i64, C.c_int, _p, _p, _p]),
    ("fmmb_direct_potentials", C.c_int,
     [_p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _p, _p]),
]

_lib = None
_lib_lock = threading.Lock()
_handles: dict[int, int] = {}


def load(path: str = LIB_PATH):
    """Load the CUDA library (raises NativeError if it is missing)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(path):
                raise NativeError(
                    f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = C.CDLL(path)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return [name for name, _, _ in SIGNATURES]


def device_of(device=None) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise NativeError("no CUDA device: the B200 build has no CPU fallback")
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise NativeError(f"device {dev} is not a CUDA device")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def handle(dev: torch.device) -> int:
    """The device's library handle (one per device, created once; every C
    entry point locks it for the duration of the call, so threads may share it)."""
    lib = load()
    idx = dev.index
    h = _handles.get(idx)
    if h is None:
        with _lib_lock:
            h = _handles.get(idx)
            if h is None:
                out = C.c_void_p()
                st = lib.fmmb_create(idx, C.byref(out))
                if st != OK:
                    raise NativeError(f"fmmb_create(device={idx}) failed with status {st}")
                h = out.value
                _handles[idx] = h
    return h


SORT_PATHS = {1: "bucket", 2: "onesweep"}
_SORT_PATH_IDS = {"auto": 0, "bucket": 1, "onesweep": 2, "bucket_hist": 3}


def set_sort_path(path: str, device=None) -> None:
    """Select the sort-phase strategy of the fused build on a device:
    "auto" (bucket sort, Onesweep rerun on overflow), "bucket", "onesweep" or
    "bucket_hist" (bucket sort without speculative regions: histogram pass
    first).  All strategies produce bit-identical outputs."""
    if path not in _SORT_PATH_IDS:
        raise ValueError(f"unknown sort path {path!r}")
    dev = device_of(device)
    h = handle(dev)
    st = load().fmmb_set_sort_path(h, _SORT_PATH_IDS[path])
    check(st, h)


def set_overlap(on: bool, device=None) -> None:
    """Run the bucket path's local + heads passes on a side stream overlapping
    the directory and lists (default) or serially on the caller's stream."""
    dev = device_of(device)
    h = handle(dev)
    check(load().fmmb_set_overlap(h, 1 if on else 0), h)


def stream_of(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def check(st: int, h: int) -> None:
    if st == OK:
        return
    msg = load().fmmb_last_error(h).decode(errors="replace")
    if st == ERR_DOMAIN:
        raise DomainError(msg)
    if st == ERR_CAPACITY:
        raise CapacityError(msg)
    raise NativeError(f"libfmmb200 status {st}: {msg}")


class Allocator:
    """Allocator callback backed by the PyTorch caching allocator.

    Every block handed to the library is a uint8 CUDA tensor kept in
    ``self.blocks`` (so the outputs' lifetime is torch's)."""

    def __init__(self, dev: torch.device):
        self.dev = dev
        blocks: list[torch.Tensor] = []
        spans: list[tuple[int, int]] = []  # (base address, bytes) of each block
        errors: list[BaseException] = []
        self.blocks = blocks
        self.spans = spans
        self._errors = errors

        # the closure must not reference `self` (a cycle would keep every
        # output block alive until the cyclic GC runs)
        def _alloc(_ctx, nbytes):
            try:
                nb = max(int(nbytes), 1)
                t = torch.empty(nb, dtype=torch.uint8, device=dev)
            except BaseException as e:  # noqa: BLE001 - reported after the call
                errors.append(e)
                return None
            blocks.append(t)
            ptr = t.data_ptr()
            spans.append((ptr, nb))
            return ptr

        self.fn = ALLOC_FN(_alloc)

    @property
    def error(self) -> BaseException | None:
        return self._errors[0] if self._errors else None

    def block_of(self, ptr: int) -> tuple[torch.Tensor, int]:
        for b in self.blocks:
            base = b.data_ptr()
            if base <= ptr < base + b.numel() or (ptr == base):
                return b, ptr - base
        raise NativeError(f"pointer {ptr:#x} is not in any allocated block")

    def typed(self, ptr: int, tdt: torch.dtype, size: int) -> tuple[torch.Tensor, int] | None:
        """(whole block viewed as `tdt`, element offset of ptr), cached per
        block and dtype, when the block and the offset are `size`-aligned:
        one slicing op per output view instead of three."""
        cache = self.__dict__.setdefault("_typed", {})
        for i, (base, n) in enumerate(self.spans):
            if base <= ptr < base + n or ptr == base:
                off = ptr - base
                if off % size or n % size:
                    return None
                t = cache.get((i, tdt))
                if t is None:
                    t = self.blocks[i].view(tdt)
                    cache[(i, tdt)] = t
                return t, off // size
        raise NativeError(f"pointer {ptr:#x} is not in any allocated block")


_SIZES = {"f8": 8, "i8": 8, "u8": 8, "i2": 2, "u4": 4, "i4": 4}
_EMPTY: dict = {}
_TORCH_DTYPES = {
    "f8": torch.float64, "i8": torch.int64, "u8": torch.uint64, "i2": torch.int16,
    "u4": torch.uint32, "i4": torch.int32,
}


def view(alloc: Allocator, ptr: int | None, count: int, dtype: str, shape=None) -> torch.Tensor:
    """Typed device view of `count` elements at `ptr` inside an allocated block."""
    tdt = _TORCH_DTYPES[dtype]
    if not ptr or count == 0:
        key = (alloc.dev, tdt, tuple(shape) if shape is not None else (0,))
        t = _EMPTY.get(key)  # zero-size views are shared (nothing to alias)
        if t is None:
            t = torch.empty(key[2], dtype=tdt, device=alloc.dev)
            _EMPTY[key] = t
        return t
    size = _SIZES[dtype]
    tv = alloc.typed(ptr, tdt, size)
    if tv is not None:
        t = tv[0][tv[1]: tv[1] + count]
    else:
        block, off = alloc.block_of(ptr)
        t = block[off: off + count * size].view(tdt)
    if shape is not None:
        t = t.view(*shape)
    return t


def trace(dev) -> list[tuple[str, float]]:
    """(phase, ms since the build's start) of the last build on `dev`
    (FMMB_TRACE=1 in the environment when the handle was created)."""
    lib = load()
    h = handle(dev)
    ms = (C.c_float * 32)()
    names = (C.c_char_p * 32)()
    k = lib.fmmb_trace(h, ms, names, 32)
    return [(names[i].decode(), float(ms[i])) for i in range(k)]


class EventRing:
    """Per-device ring of 6-event sets for the build's phase timing: events
    are created once and reused; a slot's previous owner (a lazily resolved
    BuildSeconds) is resolved before its events are recorded again."""

    SIZE = 64

    def __init__(self):
        self.sets: list = []
        self.owners: list = [None] * self.SIZE
        self.i = 0

    def take(self, owner):
        import weakref

        k = self.i % self.SIZE
        self.i += 1
        if k == len(self.sets):
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            for e in evs:  # torch creates the CUevent lazily, on first record
                e.record()
            self.sets.append((evs, (C.c_void_p * 6)(*[e.cuda_event for e in evs])))
        prev = self.owners[k]() if self.owners[k] is not None else None
        if prev is not None:
            prev._resolve()
        self.owners[k] = weakref.ref(owner)
        return self.sets[k]


_rings: dict[int, EventRing] = {}


def event_ring(dev: torch.device) -> EventRing:
    r = _rings.get(dev.index)
    if r is None:
        r = _rings[dev.index] = EventRing()
    return r
