"""Per-node classification of the global source boxes on the device
(SURVEY §8(f) row 3): drop-in for pkg/src/fmmkit/boxtype.py (BoxType,
TypedBoxList, classify, dump_typed, load_typed).  Each level is one
`fmmb_classify_boxes` launch (thread per box: the 216-candidate stencil
owner predicate of boxtype.py:63-101 and the type rules of :103-144).
`plan` is the reference's PartitionPlan (or any object with nodes,
units_per_node, partition_level, critical_level, box_proc_id)."""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

import numpy as np
import torch

from . import _host, _lib
from .errors import DomainError


class BoxType(IntEnum):  # boxtype.py:29-34
    DOMESTIC = 0
    EXPORT = 1
    IMPORT = 2
    ROOT = 3
    OTHER = 4


@dataclass
class TypedBoxList:  # boxtype.py:37-55
    node: int
    plan: object
    boxes: dict
    types: dict

    def of_type(self, level: int, box_type: BoxType):
        return self.boxes[level][self.types[level] == box_type]

    def export_boxes(self, level: int):
        return self.of_type(level, BoxType.EXPORT)

    def import_boxes(self, level: int):
        return self.of_type(level, BoxType.IMPORT)

    def root_boxes(self, level: int):
        return self.of_type(level, BoxType.ROOT)


def classify(node: int, global_src_boxes: dict, plan) -> TypedBoxList:
    """Type of every global non-empty source box, per level (boxtype.py:103)."""
    levels = sorted(global_src_boxes)
    arrays = [global_src_boxes[l] for l in levels]
    dout = _host.is_device_input(*arrays)
    dev = _host.pick_device(*arrays)
    bpid_np = np.asarray(plan.box_proc_id)
    bpid = torch.from_numpy(np.ascontiguousarray(bpid_np, dtype=np.int32)).to(dev)
    lib = _lib.load()
    h = _lib.handle(dev)
    types = {}
    for level, arr in zip(levels, arrays):
        if level < 2:
            raise DomainError("octree data start at level 2")
        boxes = _host.to_device(arr, dev, torch.uint64, (-1,))
        out = torch.empty(boxes.numel(), dtype=torch.int8, device=dev)
        st = lib.fmmb_classify_boxes(
            h, boxes.data_ptr() if boxes.numel() else None, boxes.numel(), int(level),
            bpid.data_ptr(), bpid.numel(), int(plan.partition_level), int(plan.critical_level),
            int(plan.nodes), int(plan.units_per_node), int(node),
            out.data_ptr() if out.numel() else None, _lib.stream_of(dev))
        _lib.check(st, h)
        types[level] = out if dout else out.cpu().numpy()
    return TypedBoxList(node=node, plan=plan, boxes=dict(global_src_boxes), types=types)


def dump_typed(typed: TypedBoxList, path) -> None:
    """boxtype.py:147-152 (BTYP section; types as int16)."""
    from . import container

    sec = container.Section(tag="BTYP", meta={"node": typed.node})
    for level in sorted(typed.boxes):
        t = typed.types[level]
        sec.arrays[f"boxes_{level}"] = typed.boxes[level]
        sec.arrays[f"types_{level}"] = (t.to(torch.int16) if isinstance(t, torch.Tensor)
                                        else np.asarray(t).astype(np.int16))
    container.write_container(path, max(typed.boxes), [sec])


def load_typed(path, plan) -> TypedBoxList:
    """boxtype.py:155-166."""
    from . import container

    _, sections = container.read_container(path)
    sec = next(s for s in sections if s.tag == "BTYP")
    boxes, types = {}, {}
    for name, arr in sec.arrays.items():
        kind, level = name.rsplit("_", 1)
        if kind == "boxes":
            boxes[int(level)] = arr
        else:
            types[int(level)] = arr.astype(np.int8)
    return TypedBoxList(node=int(sec.meta["node"]), plan=plan, boxes=boxes, types=types)
