"""Bit-exact parity at the north-star configurations (BASELINE.json configs
c2, c3 and one c4 rebuild step): sha256 of every output array of the device
build against the UNMODIFIED reference's (tests/golden/hashes_northstar.json,
made by tests/golden/make_golden_northstar.py on the same inputs bench.py
builds), for the default sort path (speculative bucket regions at c2/c4,
refined histogram buckets at c3) and for the Onesweep path.

c2 runs the bucket geometry no smaller case reaches (bb = 14 bucket bits,
7 in-bucket key bits, n > 2^23); c4 includes coordinates np.mod maps to
exactly 1.0 (the encoder's clamp edge, _ckernels.pyx:97-102)."""

import json
import os

import pytest

from tests import golden_io as gio

pytestmark = pytest.mark.gpu

HASHES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                      "hashes_northstar.json")


def _hashes():
    with open(HASHES) as f:
        return json.load(f)


@pytest.fixture(params=["auto", "onesweep"])
def path(request, gpu):
    gpu._lib.set_sort_path(request.param)
    yield request.param
    gpu._lib.set_sort_path("auto")


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_northstar_bit_exact(gpu, path, name):
    spec = _hashes()[name]
    src, q, recv, L = gio.northstar_inputs(name)
    assert (L, src.shape[0], recv.shape[0]) == (spec["level"], spec["n"], spec["m"])
    st = gpu.build_all(src, q, recv, max_level=L)
    assert st.sort_path == ("onesweep" if path == "onesweep" else "bucket")
    flat = gio.flatten(st)
    del st
    got = {k: gio.sha(v) for k, v in flat.items()}
    bad = sorted(k for k in spec["arrays"] if got.get(k) != spec["arrays"][k])
    assert set(got) == set(spec["arrays"]), sorted(set(got) ^ set(spec["arrays"]))
    assert not bad, bad
