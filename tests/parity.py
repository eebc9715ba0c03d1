"""Field-by-field bit-exact comparison of two FmmStructures-shaped objects
(ours vs the reference's), dtypes included."""

import numpy as np


def _eq(name, a, b, errors):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.dtype != b.dtype:
        errors.append(f"{name}: dtype {a.dtype} != {b.dtype}")
        return
    if a.shape != b.shape:
        errors.append(f"{name}: shape {a.shape} != {b.shape}")
        return
    if not np.array_equal(a, b):
        bad = np.flatnonzero((a != b).reshape(-1)) if a.size else []
        errors.append(f"{name}: {len(bad)} mismatches, first at {bad[:5]}")


def compare_point_sets(name, a, b, errors):
    assert a.level == b.level
    for f in ("points", "permutation", "bookmarks", "non_empty_index", "boxes"):
        _eq(f"{name}.{f}", getattr(a, f), getattr(b, f), errors)
    if (a.charges is None) != (b.charges is None):
        errors.append(f"{name}.charges: None mismatch")
    elif a.charges is not None:
        _eq(f"{name}.charges", a.charges, b.charges, errors)


def compare_structures(ours, ref):
    errors = []
    assert ours.max_level == ref.max_level
    compare_point_sets("sorted_src", ours.sorted_src, ref.sorted_src, errors)
    compare_point_sets("sorted_recv", ours.sorted_recv, ref.sorted_recv, errors)
    _eq("neighbor_bookmark", ours.neighbor_table.neighbor_bookmark,
        ref.neighbor_table.neighbor_bookmark, errors)
    _eq("neighbor_list", ours.neighbor_table.neighbor_list, ref.neighbor_table.neighbor_list,
        errors)
    for side in ("src_boxes", "recv_boxes"):
        da, db = getattr(ours.directory, side), getattr(ref.directory, side)
        if sorted(da) != sorted(db):
            errors.append(f"directory.{side} levels {sorted(da)} != {sorted(db)}")
        for l in db:
            if l in da:
                _eq(f"directory.{side}[{l}]", da[l], db[l], errors)
    for f in ("bookmark", "ranks", "codes"):
        da, db = getattr(ours.stencils, f), getattr(ref.stencils, f)
        if sorted(da) != sorted(db):
            errors.append(f"stencils.{f} levels {sorted(da)} != {sorted(db)}")
        for l in db:
            if l in da:
                _eq(f"stencils.{f}[{l}]", da[l], db[l], errors)
    return errors
