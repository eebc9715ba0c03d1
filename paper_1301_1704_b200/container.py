"""FMMS structure container: the reference's versioned
little-endian dump format (pkg/src/fmmkit/container.py:1-106, writer of
lists.py:190-257), written straight from device-resident structures.

Layout (byte-identical to the reference writer): magic "FMMS", version u32,
max level u32, section count u32, then sections: 4-byte tag, metadata map
(u32 count, u16-length-prefixed UTF-8 key + i64 value), named arrays (u32
count, u16-length-prefixed name, u8 dtype code, u8 ndim, u64 shape, u64 byte
length, raw little-endian bytes).

B200 path: the headers are laid out on the host while every CUDA array is
copied device->host in chunks into two pinned staging buffers; a writer
thread streams the filled buffer to the file while the next chunk's copy
runs, so a multi-GB dump moves at PCIe / disk speed with one pass over the
data and no full host copy.  `load_structures(path, device=...)` reads the
file and uploads the arrays to the device.
"""

from __future__ import annotations

import struct
import threading
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from .errors import DomainError

MAGIC = b"FMMS"
VERSION = 1

_DTYPES = {  # container.py:23-31
    0: np.dtype("<f8"),
    1: np.dtype("<i8"),
    2: np.dtype("<u8"),
    3: np.dtype("<i2"),
    4: np.dtype("<i4"),
    5: np.dtype("|u1"),
    6: np.dtype("<f4"),
}
_CODES = {v: k for k, v in _DTYPES.items()}
_TORCH_NP = {torch.float64: np.dtype("<f8"), torch.int64: np.dtype("<i8"),
             torch.uint64: np.dtype("<u8"), torch.int16: np.dtype("<i2"),
             torch.int32: np.dtype("<i4"), torch.uint8: np.dtype("|u1"),
             torch.float32: np.dtype("<f4")}
_NP_TORCH = {v: k for k, v in _TORCH_NP.items()}
_CHUNK = 64 << 20  # staging chunk (bytes)


@dataclass
class Section:
    tag: str  # exactly 4 ASCII chars
    meta: dict = field(default_factory=dict)
    arrays: dict = field(default_factory=dict)  # numpy arrays or CUDA tensors


def _str(s: str) -> bytes:
    raw = s.encode("utf-8")
    return struct.pack("<H", len(raw)) + raw


def _array_info(name: str, arr):
    """(dtype, shape, nbytes, source) of a numpy array or CUDA tensor."""
    if isinstance(arr, torch.Tensor):
        if arr.dtype not in _TORCH_NP:
            raise DomainError(f"unsupported dtype {arr.dtype} for array {name!r}")
        t = arr.detach().contiguous()
        return _TORCH_NP[t.dtype], tuple(t.shape), t.numel() * t.element_size(), t
    a = np.ascontiguousarray(arr)
    if a.dtype.byteorder == ">":
        a = a.astype(a.dtype.newbyteorder("<"))
    if a.dtype not in _CODES:
        raise DomainError(f"unsupported dtype {a.dtype} for array {name!r}")
    return a.dtype, a.shape, a.nbytes, a


class _Stream:
    """Chunked writer: host bytes are appended directly; CUDA tensors are
    copied into alternating pinned buffers and written by a worker thread."""

    def __init__(self, fh):
        self.fh = fh
        self.bufs = [None, None]
        self.cur = 0
        self.fill = 0
        self.worker = None
        self.events = [None, None]

    def _buf(self, k):
        if self.bufs[k] is None:
            self.bufs[k] = torch.empty(_CHUNK, dtype=torch.uint8,
                                       pin_memory=torch.cuda.is_available())
        return self.bufs[k]

    def _join(self):
        if self.worker is not None:
            self.worker.join()
            self.worker = None

    def _flush(self):
        if self.fill == 0:
            return
        k, n, ev = self.cur, self.fill, self.events[self.cur]
        self._join()

        def work():
            if ev is not None:
                ev.synchronize()
            self.fh.write(memoryview(self.bufs[k].numpy())[:n])

        self.worker = threading.Thread(target=work)
        self.worker.start()
        self.cur ^= 1
        self.fill = 0
        self.events[self.cur] = None

    def _room(self):
        if self.fill == _CHUNK:
            self._flush()
        return _CHUNK - self.fill

    def host(self, b):
        mv = memoryview(b)
        if mv.nbytes == 0:
            return
        if mv.ndim != 1 or mv.itemsize != 1:
            mv = mv.cast("B")
        if len(mv) >= (1 << 20):  # large host array: straight to the file, in order
            self._flush()
            self._join()
            self.fh.write(mv)
            return
        at = 0
        while at < len(mv):
            n = min(self._room(), len(mv) - at)
            dst = self._buf(self.cur).numpy()
            dst[self.fill:self.fill + n] = np.frombuffer(mv[at:at + n], dtype=np.uint8)
            self.fill += n
            at += n

    def device(self, t: torch.Tensor):
        if t.numel() == 0:
            return
        flat = t.reshape(-1).view(torch.uint8)
        at, tot = 0, flat.numel()
        while at < tot:
            room = self._room()
            n = min(room, tot - at)
            buf = self._buf(self.cur)
            buf[self.fill:self.fill + n].copy_(flat[at:at + n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(t.device))
            self.events[self.cur] = ev
            self.fill += n
            at += n

    def close(self):
        self._flush()
        self._join()


def write_container(path, max_level: int, sections: list) -> None:
    """container.py:53-79; arrays may be CUDA tensors (copied out in chunks)."""
    plan = []
    for sec in sections:
        tag = sec.tag.encode("ascii")
        if len(tag) != 4:
            raise DomainError(f"section tag must be 4 bytes, got {sec.tag!r}")
        arrs = [(name, _array_info(name, a)) for name, a in sec.arrays.items()]
        plan.append((tag, sec.meta, arrs))
    with open(Path(path), "wb") as fh:
        w = _Stream(fh)
        try:
            w.host(MAGIC + struct.pack("<III", VERSION, max_level, len(sections)))
            for tag, meta, arrs in plan:
                hdr = [tag, struct.pack("<I", len(meta))]
                for key, value in meta.items():
                    hdr += [_str(key), struct.pack("<q", int(value))]
                hdr.append(struct.pack("<I", len(arrs)))
                w.host(b"".join(hdr))
                for name, (dt, shape, nbytes, src) in arrs:
                    w.host(_str(name) + struct.pack("<BB", _CODES[dt], len(shape))
                           + struct.pack(f"<{len(shape)}Q", *shape) + struct.pack("<Q", nbytes))
                    if isinstance(src, torch.Tensor) and src.is_cuda:
                        w.device(src)
                    elif isinstance(src, torch.Tensor):
                        w.host(src.reshape(-1).view(torch.uint8).numpy())
                    else:
                        w.host(src.reshape(-1).view(np.uint8))
        finally:
            w.close()


def read_container(path, device=None) -> tuple:
    """container.py:82-106.  With `device`, arrays come back as tensors on it."""
    with open(Path(path), "rb") as fh:
        if fh.read(4) != MAGIC:
            raise DomainError(f"{path}: not a structure container")
        version, max_level, n_sections = struct.unpack("<III", fh.read(12))
        if version != VERSION:
            raise DomainError(f"{path}: unsupported container version {version}")
        sections = []
        for _ in range(n_sections):
            tag = fh.read(4).decode("ascii")
            (n_meta,) = struct.unpack("<I", fh.read(4))
            meta = {}
            for _ in range(n_meta):
                (k,) = struct.unpack("<H", fh.read(2))
                key = fh.read(k).decode("utf-8")
                (meta[key],) = struct.unpack("<q", fh.read(8))
            (n_arrays,) = struct.unpack("<I", fh.read(4))
            arrays = {}
            for _ in range(n_arrays):
                (k,) = struct.unpack("<H", fh.read(2))
                name = fh.read(k).decode("utf-8")
                code, ndim = struct.unpack("<BB", fh.read(2))
                shape = struct.unpack(f"<{ndim}Q", fh.read(8 * ndim))
                (nbytes,) = struct.unpack("<Q", fh.read(8))
                dt = _DTYPES[code]
                if device is None:
                    arr = np.empty(shape, dtype=dt)
                    got = fh.readinto(memoryview(arr.reshape(-1).view(np.uint8)))
                    if got != nbytes or arr.nbytes != nbytes:
                        raise DomainError(f"{path}: truncated structure container")
                    arrays[name] = arr
                else:
                    arrays[name] = _upload(fh, nbytes, dt, shape, device)
            sections.append(Section(tag=tag, meta=meta, arrays=arrays))
        return max_level, sections


_UP_LOCAL = threading.local()


def _upload(fh, nbytes: int, dt, shape, device) -> torch.Tensor:
    """File bytes -> device tensor through two alternating pinned chunks.

    The chunks are per thread and their last-copy events persist across
    calls: a chunk is refilled only after the copy that last read it is done
    (whichever array it belonged to), and the call returns after its own
    copies completed, so no later host write can race an in-flight H2D."""
    out = torch.empty(nbytes, dtype=torch.uint8, device=device)
    up = _UP_LOCAL.__dict__
    if "bufs" not in up:
        up["bufs"] = [torch.empty(_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        up["evs"] = [None, None]
    bufs, evs = up["bufs"], up["evs"]
    at, k = 0, 0
    stream = torch.cuda.current_stream(out.device)
    try:
        while at < nbytes:
            n = min(_CHUNK, nbytes - at)
            if evs[k] is not None:
                evs[k].synchronize()  # the copy that last used this buffer is done
            got = fh.readinto(memoryview(bufs[k].numpy())[:n])
            if got != n:
                raise DomainError("truncated structure container")
            out[at:at + n].copy_(bufs[k][:n], non_blocking=True)
            evs[k] = torch.cuda.Event()
            evs[k].record(stream)
            at += n
            k ^= 1
    finally:
        for e in evs:
            if e is not None:
                e.synchronize()
    return out.view(_NP_TORCH[dt]).reshape(shape)
