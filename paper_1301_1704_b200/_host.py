"""Host-side plumbing shared by the API modules: input staging and the
device->host conversion that keeps the reference's numpy-in / numpy-out
contract (output location follows input location: numpy or CPU inputs give
numpy outputs, CUDA tensors give device-resident torch tensors)."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DomainError


def is_device_input(*arrays) -> bool:
    return any(isinstance(a, torch.Tensor) and a.is_cuda for a in arrays if a is not None)


def pick_device(*arrays) -> torch.device:
    for a in arrays:
        if isinstance(a, torch.Tensor) and a.is_cuda:
            return _lib.device_of(a.device)
    return _lib.device_of(None)


def to_device(a, dev: torch.device, dtype: torch.dtype, shape=None) -> torch.Tensor:
    """Contiguous CUDA tensor of `dtype` (copies only when needed)."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        np_dtype = {torch.float64: np.float64, torch.int64: np.int64,
                    torch.uint64: np.uint64, torch.int16: np.int16}[dtype]
        arr = np.ascontiguousarray(np.asarray(a, dtype=np_dtype))
        t = torch.from_numpy(arr)
    if shape is not None:
        t = t.reshape(shape)
    if t.dtype != dtype:
        t = t.to(dtype)
    if t.device != dev:
        t = t.to(dev, non_blocking=False)
    return t.contiguous()


def points_to_device(points, dev: torch.device) -> torch.Tensor:
    """(N,3) f64 contiguous on `dev`; the reference reshapes with (-1, 3)
    (pseudosort.py:57, morton.py:97)."""
    t = to_device(points, dev, torch.float64)
    if t.numel() % 3:
        raise DomainError(f"points must have 3 coordinates per row, got {tuple(t.shape)}")
    return t.reshape(-1, 3)


class HostBatch:
    """Batches device->host copies into pinned buffers with a single sync."""

    def __init__(self):
        self._items: list[tuple[torch.Tensor, torch.Tensor]] = []

    def add(self, t: torch.Tensor | None):
        if t is None:
            return None
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        if t.numel():
            h.copy_(t, non_blocking=True)
        self._items.append((t, h))
        return h

    def finish(self) -> None:
        if self._items:
            torch.cuda.current_stream(self._items[0][0].device).synchronize()


def to_numpy(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.cpu().numpy() if t.is_cuda else t.numpy()
    return np.asarray(t)
