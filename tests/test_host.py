"""Host-side logic of the drop-in API (no GPU needed)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1301_1704_b200 as fb
from paper_1301_1704_b200 import _lib, roofline
from paper_1301_1704_b200.pseudosort import check_budget, check_level, check_mode

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_choose_max_level_table():  # tests/test_pseudosort.py:142-148 of the reference
    assert fb.choose_max_level(1, 1) == 0
    assert fb.choose_max_level(8, 1) == 1
    assert fb.choose_max_level(9, 1) == 2
    assert fb.choose_max_level(2**20, 2**20) == 0
    assert fb.choose_max_level(512, 8) == 2
    assert fb.choose_max_level(513, 8) == 3
    assert fb.choose_max_level(2**23, 16) == 7  # c4
    assert fb.choose_max_level(2**16, 16) == 4  # c1
    with pytest.raises(fb.DomainError):
        fb.choose_max_level(10, 0)


def test_precondition_errors():
    with pytest.raises(fb.CapacityError):
        check_level(21)
    with pytest.raises(fb.CapacityError):
        check_level(-1)
    with pytest.raises(fb.CapacityError, match="budget"):
        check_budget(8, 1024)
    check_budget(9, fb.DEFAULT_HISTOGRAM_BUDGET)
    with pytest.raises(fb.CapacityError):
        check_budget(10, fb.DEFAULT_HISTOGRAM_BUDGET)
    with pytest.raises(fb.DomainError):
        check_mode("bogus")
    with pytest.raises(fb.DomainError):
        fb.build_all(np.random.rand(10, 3), None, np.random.rand(10, 3))
    assert issubclass(fb.DomainError, ValueError)
    assert issubclass(fb.CapacityError, fb.FmmError)


def test_error_classes_subclass_reference_when_loaded(ref):
    """Imported after fmmkit, our error classes are also the reference's."""
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import fmmkit, paper_1301_1704_b200 as fb\n"
        "for n in ('FmmError','CapacityError','DomainError','RoutingError',"
        "'InfeasiblePartitionError'):\n"
        "    assert issubclass(getattr(fb, n), getattr(fmmkit.errors, n)), n\n"
        "print('ok')\n" % (os.path.join(ROOT, "oracle", "_ref"), ROOT))
    out = subprocess.run(["python", "-c", code], capture_output=True, text=True)
    assert out.stdout.strip() == "ok", out.stderr


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "fmmb200.h")).read()
    declared = set(re.findall(r"FMMB_API [^;]*?\b(fmmb_\w+)\(", header))
    lib = _lib.load()
    assert declared == set(_lib.exported_symbols())
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.fmmb_abi_version() == 1


def test_ctypes_layout_matches_c(tmp_path):
    """The ctypes mirror of fmmb_structures / fmmb_point_set has the C layout."""
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "fmmb200.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu\\n\", sizeof(fmmb_point_set),"
        " sizeof(fmmb_structures), offsetof(fmmb_structures, recv),"
        " offsetof(fmmb_structures, st_codes), offsetof(fmmb_structures, n_launches));}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_lib.PointSetC), ctypes.sizeof(_lib.StructuresC),
            _lib.StructuresC.recv.offset, _lib.StructuresC.st_codes.offset,
            _lib.StructuresC.n_launches.offset]
    assert got == want


def test_compute_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(fb.NativeError):
        fb.build_all(np.random.rand(10, 3), None, np.random.rand(10, 3), max_level=2)


def test_algorithmic_bytes_c1():
    """B_alg(c1) = 16,832,192 bytes (counts from the oracle)."""
    from oracle import oracle as orc
    from paper_1301_1704_b200.workloads import generate

    src, q, recv = generate(2**16, 2**16, "uniform", 1)
    st = orc.build_all(src, q, recv, 4)
    assert roofline.build_bytes(roofline.build_counts(st)) == 16_832_192


def test_algorithmic_bytes_c2_from_survey_counts():
    """c2 counts give B_alg = 7,322,505,058 bytes."""
    n = 2**24
    c = {"L": 7, "n": n, "m": n, "q": True, "ks": 2_096_457, "kr": 2_096_431, "e2": 55_705_349,
         "ks_l": {l: 8**l for l in range(2, 7)}, "kr_l": {l: 8**l for l in range(2, 7)},
         "s_l": {}}
    c["kr_l"][7] = 2_096_431
    # full-occupancy closed form below the finest level, measured finest
    s_l = {l: (6 * 2**l - 8) ** 3 - (3 * 2**l - 2) ** 3 for l in range(2, 7)}
    s_l[7] = 382_974_517
    c["s_l"] = s_l
    assert sum(s_l.values()) == 435_312_397
    assert roofline.build_bytes(c) == 7_322_505_058


def _morton(x, y, z):
    k = 0
    for b in range(21):
        k |= ((x >> b) & 1) << (3 * b) | ((y >> b) & 1) << (3 * b + 1) | ((z >> b) & 1) << (3 * b + 2)
    return k


def _window_order_table():
    """Host restatement of lists.cuh WinOrder: 48 cases (3 parities x the
    ranking of K_a * 3 + a), each the 27 window offsets in Morton order."""
    ranks = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    tab = []
    for cs in range(48):
        c = []
        for a in range(3):
            K = ranks[cs >> 3][a] + 1
            c.append((3 << K) - 1 if (cs >> a) & 1 else 3 << K)
        keys = [_morton(c[0] + q % 3 - 1, c[1] + (q // 3) % 3 - 1, c[2] + q // 9 - 1)
                for q in range(27)]
        tab.append(sorted(range(27), key=lambda q: keys[q]))
    return tab


def _window_case(x, y, z, l1):
    par, kk = 0, []
    for a, v in enumerate((x, y, z)):
        odd = v & 1
        w = v + 1 if odd else v
        K = ((w & -w).bit_length() - 1) if (w and w < (1 << l1)) else 64
        par |= odd << a
        kk.append(K * 3 + a)
    rx = (kk[0] > kk[1]) + (kk[0] > kk[2])
    ry = (kk[1] > kk[0]) + (kk[1] > kk[2])
    pi = (0 if ry == 1 else 1) if rx == 0 else (2 if ry == 0 else 3) if rx == 1 else (
        4 if ry == 0 else 5)
    return par | (pi << 3)


def test_window_order_table_matches_sorted_windows():
    """The list writer's table-driven window order (lists.cuh window_case /
    WinOrder) equals sorting the in-grid 3x3x3 window keys, at every level
    and at the grid faces."""
    import random

    tab = _window_order_table()
    rng = random.Random(7)
    for l1 in range(0, 9):
        n = 1 << l1
        pts = {(0, 0, 0), (n - 1, n - 1, n - 1), (0, n - 1, 0)}
        pts |= {tuple(rng.randrange(n) for _ in range(3)) for _ in range(300)}
        for x, y, z in pts:
            members = []
            for q in range(27):
                p = (x + q % 3 - 1, y + (q // 3) % 3 - 1, z + q // 9 - 1)
                if all(0 <= v < n for v in p):
                    members.append((_morton(*p), q))
            want = [q for _, q in sorted(members)]
            inside = {q for _, q in members}
            got = [q for q in tab[_window_case(x, y, z, l1)] if q in inside]
            assert got == want, (l1, x, y, z)
