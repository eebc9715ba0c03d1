"""Prefix-sum and stream-compaction primitives (drop-in for fmmkit.scan,
pkg/src/fmmkit/scan.py:25-81), computed by libfmmb200's device scan
(`fmmb_exclusive_scan_i64`, single-pass decoupled look-back).

The reference scan is blocked over `workers` CPU threads; integer addition is
associative, so its result is the same for every worker count, and so is
this one (`workers` is accepted for signature parity and ignored).
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import CapacityError, DomainError
from .kernels import exclusive_scan as _device_scan

_INT64_GUARD = float(2**62)  # scan.py:16


def exclusive_scan(values, workers: int = 1):
    """(exclusive prefix sum, inclusive total); out[0] = 0 (scan.py:25-73).

    DomainError for an empty / non-1-d / negative input, CapacityError when the
    total would overflow the 64-bit accumulator, as the reference."""
    if isinstance(values, torch.Tensor):
        a = values
        if a.dim() != 1 or a.shape[0] == 0:
            raise DomainError("scan input must be a non-empty 1-d array")
        if bool((a < 0).any()):
            raise DomainError("scan input must be non-negative")
        if float(a.to(torch.float64).sum()) > _INT64_GUARD:
            raise CapacityError("scan total would overflow the 64-bit accumulator")
        return _device_scan(a)
    a = np.asarray(values)
    if a.ndim != 1 or a.shape[0] == 0:
        raise DomainError("scan input must be a non-empty 1-d array")
    if np.any(a < 0):
        raise DomainError("scan input must be non-negative")
    if float(np.sum(a, dtype=np.float64)) > _INT64_GUARD:
        raise CapacityError("scan total would overflow the 64-bit accumulator")
    return _device_scan(a.astype(np.int64, copy=False))


def compact_flags(flags, workers: int = 1):
    """Ranks of flagged entries and their count (scan.py:76-81); flags must
    be binary (DomainError otherwise)."""
    if isinstance(flags, torch.Tensor):
        if not bool(((flags == 0) | (flags == 1)).all()):
            raise DomainError("compact_flags input must be binary")
    else:
        f = np.asarray(flags)
        if not np.all((f == 0) | (f == 1)):
            raise DomainError("compact_flags input must be binary")
    return exclusive_scan(flags, workers=workers)


__all__ = ["exclusive_scan", "compact_flags"]
