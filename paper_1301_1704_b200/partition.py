"""Receiver-load partition plan: drop-in for
`PartitionPlan` and `choose_partition` (pkg/src/fmmkit/partition.py:21-127).
Per candidate level the dense Morton-ordered load, its prefix sum and the
P*g - 1 load cuts run on the device (`fmmb_partition_level`); the level
loop, the balance test and the plan object stay on the host."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _host, _lib
from .errors import DomainError, InfeasiblePartitionError


@dataclass
class PartitionPlan:  # partition.py:21-51
    nodes: int
    units_per_node: int
    partition_level: int
    critical_level: int
    box_proc_id: np.ndarray
    unit_ranges: np.ndarray
    balanced: bool
    load_ratio: float

    @property
    def num_units(self) -> int:
        return self.nodes * self.units_per_node

    def node_of_unit(self, unit: int) -> int:
        return unit // self.units_per_node

    def unit_of_box_index(self, index, level: int):
        if level < self.partition_level:
            raise DomainError("boxes above the partition level have a unit range, not one unit")
        shift = np.uint64(3 * (level - self.partition_level))
        idx = np.asarray(index, dtype=np.uint64) >> shift
        out = self.box_proc_id[idx.astype(np.int64)]
        return out if isinstance(index, np.ndarray) else int(out)

    def node_of_box_index(self, index, level: int):
        unit = self.unit_of_box_index(index, level)
        return (unit // self.units_per_node if isinstance(index, np.ndarray)
                else int(unit) // self.units_per_node)


def choose_partition(recv_boxes, recv_counts, max_level: int, nodes: int, units_per_node: int,
                     tolerance: float = 0.2) -> PartitionPlan:
    """Deepen the partition level until max/mean range load <= 1 + tolerance
    (partition.py:74-127); identical plans to the reference."""
    units = nodes * units_per_node
    if units < 1:
        raise DomainError("need at least one compute unit")
    nbox = int(recv_boxes.shape[0]) if hasattr(recv_boxes, "shape") else len(recv_boxes)
    if units > nbox:
        raise InfeasiblePartitionError(
            f"{units} units exceed the {nbox} non-empty receiver boxes")
    dev = _host.pick_device(recv_boxes, recv_counts)
    boxes = _host.to_device(recv_boxes, dev, torch.uint64, (-1,))
    counts = _host.to_device(recv_counts, dev, torch.int64, (-1,))
    total = int(counts.sum())
    lib = _lib.load()
    h = _lib.handle(dev)
    bounds = torch.empty(units + 1, dtype=torch.int64, device=dev)
    cum = torch.empty(units + 1, dtype=torch.int64, device=dev)
    best = None
    for level in range(2, max(max_level, 2) + 1):
        st = lib.fmmb_partition_level(h, boxes.data_ptr() if boxes.numel() else None,
                                      counts.data_ptr() if counts.numel() else None,
                                      boxes.numel(), int(max_level), level, total, units,
                                      bounds.data_ptr(), cum.data_ptr(), _lib.stream_of(dev))
        _lib.check(st, h)
        b = bounds.cpu().numpy()
        range_loads = np.diff(cum.cpu().numpy())
        mean = total / units
        ratio = float(range_loads.max() / mean) if mean > 0 else 1.0
        box_proc = np.repeat(np.arange(units, dtype=np.int32), np.diff(b).astype(np.int64))
        plan = PartitionPlan(
            nodes=nodes, units_per_node=units_per_node, partition_level=level,
            critical_level=max(level - 1, 2), box_proc_id=box_proc,
            unit_ranges=np.stack([b[:-1], b[1:]], axis=1),
            balanced=ratio <= 1.0 + tolerance, load_ratio=ratio)
        if plan.balanced:
            return plan
        if best is None or plan.load_ratio < best.load_ratio:
            best = plan
    return best


def dump_plan(plan: PartitionPlan, path) -> None:
    """partition.py:229-242 (PLAN section)."""
    from . import container

    sec = container.Section(
        tag="PLAN",
        meta={"nodes": plan.nodes, "units_per_node": plan.units_per_node,
              "partition_level": plan.partition_level, "critical_level": plan.critical_level,
              "balanced": int(plan.balanced),
              "load_ratio_micro": int(round(plan.load_ratio * 1_000_000))},
        arrays={"box_proc_id": plan.box_proc_id, "unit_ranges": plan.unit_ranges})
    container.write_container(path, plan.partition_level, [sec])


def load_plan(path) -> PartitionPlan:
    """partition.py:245-257."""
    from . import container

    _, sections = container.read_container(path)
    sec = next(s for s in sections if s.tag == "PLAN")
    return PartitionPlan(
        nodes=int(sec.meta["nodes"]), units_per_node=int(sec.meta["units_per_node"]),
        partition_level=int(sec.meta["partition_level"]),
        critical_level=int(sec.meta["critical_level"]), box_proc_id=sec.arrays["box_proc_id"],
        unit_ranges=sec.arrays["unit_ranges"], balanced=bool(sec.meta["balanced"]),
        load_ratio=sec.meta["load_ratio_micro"] / 1_000_000)
