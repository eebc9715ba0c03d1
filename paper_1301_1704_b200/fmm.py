"""Consumers of the built structures that stay on the device (SURVEY §8(f)
row 1): the near-field pass of the FMM evaluation and the brute-force
reference sum, with the reference's names and semantics
(pkg/src/fmmkit/fmm.py:21-30 direct_sum, :173-190 near_field_potentials).

Both go through the `kernels` drop-in (libfmmb200 `fmmb_near_field` /
`fmmb_direct_potentials`) and are bit-identical to the compiled backend.
Structures built on the device (`build_all_device`) are consumed in place:
no host round trip between the build and the sums.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels
from .lists import FmmStructures


def direct_sum(src_points, charges, recv_points):
    """phi[j] = sum_i q_i / |y_j - x_i|, skipping exactly coincident pairs
    (fmm.py:21-30)."""
    if isinstance(src_points, torch.Tensor) and src_points.is_cuda:
        s = src_points.reshape(-1, 3).to(torch.float64)
        r = recv_points.reshape(-1, 3).to(torch.float64)
        return kernels.direct_potentials(s[:, 0], s[:, 1], s[:, 2], charges,
                                         r[:, 0], r[:, 1], r[:, 2])
    s = np.ascontiguousarray(src_points, dtype=np.float64).reshape(-1, 3)
    r = np.ascontiguousarray(recv_points, dtype=np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(charges, dtype=np.float64)
    return kernels.direct_potentials(s[:, 0], s[:, 1], s[:, 2], q, r[:, 0], r[:, 1], r[:, 2])


def near_field_potentials(structures: FmmStructures):
    """Direct sums over each receiver box's gathered neighbourhood, per sorted
    receiver (fmm.py:173-190).  Device structures -> CUDA tensor, host
    structures -> numpy."""
    src = structures.sorted_src
    recv = structures.sorted_recv
    nt = structures.neighbor_table
    q = src.charges
    if q is None:
        q = (torch.ones(src.points.shape[0], dtype=torch.float64, device=src.points.device)
             if isinstance(src.points, torch.Tensor) else np.ones(src.points.shape[0]))
    return kernels.near_field(src.points[:, 0], src.points[:, 1], src.points[:, 2], q,
                              src.bookmarks, nt.neighbor_bookmark, nt.neighbor_list,
                              recv.points[:, 0], recv.points[:, 1], recv.points[:, 2],
                              recv.bookmarks)
