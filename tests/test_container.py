"""FMMS container: byte-identical to the reference's
writer (pkg/src/fmmkit/container.py, lists.py:203-257) and bit-exact round
trips.  CPU: host arrays; tests/test_gpu_container.py streams device-built
structures."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_1301_1704_b200 import container as C
from paper_1301_1704_b200 import lists as FL
from paper_1301_1704_b200.errors import DomainError
from paper_1301_1704_b200.pseudosort import SortedPointSet
from tests import golden_io as gio

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _structures_from_golden(case):
    out = gio.expected_outputs(case)
    L = int(case["level"])

    def ps(p):
        return SortedPointSet(level=L, points=out[f"{p}.points"], charges=out.get(f"{p}.charges"),
                              permutation=out[f"{p}.permutation"], bookmarks=out[f"{p}.bookmarks"],
                              non_empty_index=out[f"{p}.non_empty_index"], boxes=out[f"{p}.boxes"])

    return FL.FmmStructures(
        max_level=L, sorted_src=ps("src"), sorted_recv=ps("recv"),
        neighbor_table=FL.NeighborTable(out["neighbor_bookmark"], out["neighbor_list"]),
        directory=FL.LevelDirectory(L, {l: out[f"dir_src.{l}"] for l in range(2, L + 1)},
                                    {l: out[f"dir_recv.{l}"] for l in range(2, L + 1)}),
        stencils=FL.TranslationStencils(*({l: out[f"st_{f}.{l}"] for l in range(2, L + 1)}
                                          for f in ("bookmark", "ranks", "codes"))))


@pytest.mark.parametrize("name", sorted(gio.small_cases()))
def test_dump_matches_reference_bytes(tmp_path, name):
    with open(os.path.join(GOLD, "container_hashes.json")) as f:
        want = json.load(f)[name]
    st = _structures_from_golden(gio.small_cases()[name])
    path = tmp_path / "s.fmms"
    FL.dump_structures(st, path)
    raw = path.read_bytes()
    assert len(raw) == want["bytes"]
    assert hashlib.sha256(raw).hexdigest() == want["sha256"]
    back = FL.load_structures(path)
    assert back.max_level == st.max_level
    for a, b in ((back.sorted_src.points, st.sorted_src.points),
                 (back.sorted_recv.permutation, st.sorted_recv.permutation),
                 (back.neighbor_table.neighbor_list, st.neighbor_table.neighbor_list)):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    for l in range(2, st.max_level + 1):
        assert np.array_equal(back.stencils.codes[l], st.stencils.codes[l])
        assert back.stencils.codes[l].dtype == np.int16


def test_round_trip_bit_exact(tmp_path):  # test_container.py:10-30
    rng = np.random.default_rng(0)
    arrays = {"f": rng.normal(size=(10, 3)), "i": rng.integers(-5, 5, size=17),
              "u": rng.integers(0, 100, size=9).astype(np.uint64),
              "s": rng.integers(-3, 3, size=4).astype(np.int16),
              "big": rng.normal(size=(300_000,)), "nan": np.array([np.nan, -0.0, np.inf])}
    C.write_container(tmp_path / "c", 5, [C.Section("TEST", {"alpha": -7, "beta": 12}, arrays),
                                          C.Section("BBBB", {"k": 1})])
    ml, secs = C.read_container(tmp_path / "c")
    assert ml == 5 and [s.tag for s in secs] == ["TEST", "BBBB"]
    assert secs[0].meta == {"alpha": -7, "beta": 12}
    for k, v in arrays.items():
        assert secs[0].arrays[k].dtype == v.dtype and secs[0].arrays[k].tobytes() == v.tobytes()


def test_errors(tmp_path):
    (tmp_path / "bad").write_bytes(b"NOPE" + b"\0" * 32)
    with pytest.raises(DomainError):
        C.read_container(tmp_path / "bad")
    with pytest.raises(DomainError):
        C.write_container(tmp_path / "x", 0, [C.Section(tag="TOOLONG")])
    with pytest.raises(DomainError):
        C.write_container(tmp_path / "y", 0, [C.Section("ABCD", arrays={"c": np.zeros(2, np.complex128)})])
    raw = bytearray(b"FMMS" + (2).to_bytes(4, "little") + b"\0" * 8)
    (tmp_path / "v").write_bytes(bytes(raw))
    with pytest.raises(DomainError):
        C.read_container(tmp_path / "v")


def test_matches_live_reference_writer(tmp_path, ref):
    import fmmkit.container as rc

    rng = np.random.default_rng(3)
    arrays = {"a": rng.normal(size=(7, 3)), "b": rng.integers(0, 9, 5).astype(np.uint64)}
    C.write_container(tmp_path / "ours", 2, [C.Section("ABCD", {"x": 1}, arrays)])
    rc.write_container(tmp_path / "ref", 2, [rc.Section("ABCD", {"x": 1}, arrays)])
    assert (tmp_path / "ours").read_bytes() == (tmp_path / "ref").read_bytes()
