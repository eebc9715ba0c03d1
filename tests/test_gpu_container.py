"""FMMS dump of DEVICE-built structures (streamed out of HBM through pinned
staging chunks) is byte-identical to the reference's dump of its own CPU
build (tests/golden/container_hashes.json); load(device=...) round trips."""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from tests import golden_io as gio

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _hashes():
    with open(os.path.join(GOLD, "container_hashes.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["u3_L3", "s5_L5", "u_L2", "single", "recv_only", "c1"])
def test_device_dump_bytes(gpu, tmp_path, name):
    want = _hashes()[name]
    if name == "c1":
        src, q, recv, L = gio.large_inputs(gio.hashes()["c1"])
    else:
        src, q, recv, L = gio.case_inputs(gio.small_cases()[name])
    d = torch.device("cuda", 0)
    st = gpu.build_all_device(torch.from_numpy(src).to(d),
                              torch.from_numpy(q).to(d) if q is not None else None,
                              torch.from_numpy(recv).to(d), L)
    path = tmp_path / "d.fmms"
    gpu.dump_structures(st, path)
    raw = path.read_bytes()
    assert len(raw) == want["bytes"]
    assert hashlib.sha256(raw).hexdigest() == want["sha256"]
    back = gpu.load_structures(path, device=d)
    assert back.sorted_src.points.is_cuda
    assert torch.equal(back.sorted_src.points, st.sorted_src.points)
    assert torch.equal(back.neighbor_table.neighbor_list, st.neighbor_table.neighbor_list)
    for l in range(2, L + 1):
        assert torch.equal(back.stencils.ranks[l], st.stencils.ranks[l])
        assert back.stencils.codes[l].dtype == torch.int16
    host = gpu.load_structures(path)
    assert isinstance(host.sorted_recv.points, np.ndarray)


def test_multi_chunk_streaming(gpu, ref, tmp_path):
    """Arrays larger than the 64 MiB staging chunk, mixed device / host
    sources and an odd-sized tail: identical bytes to the reference writer,
    device round trip through the chunked upload."""
    from fmmkit import container as rc

    from paper_1301_1704_b200 import container as C

    g = torch.Generator(device="cuda").manual_seed(3)
    big = torch.randn(20_000_003, dtype=torch.float64, device="cuda", generator=g)  # 160 MB
    codes = torch.randint(-300, 300, (9_000_001,), dtype=torch.int16, device="cuda", generator=g)
    host = np.arange(1_000_003, dtype=np.uint64)
    C.write_container(tmp_path / "ours", 7, [
        C.Section("CORE", {"k": 3}, {"big": big, "host": host}),
        C.Section("STNC", {}, {"codes": codes, "empty": torch.empty(0, dtype=torch.int64,
                                                                  device="cuda")})])
    rc.write_container(tmp_path / "ref", 7, [
        rc.Section("CORE", {"k": 3}, {"big": big.cpu().numpy(), "host": host}),
        rc.Section("STNC", {}, {"codes": codes.cpu().numpy(), "empty": np.empty(0, np.int64)})])
    assert (tmp_path / "ours").read_bytes() == (tmp_path / "ref").read_bytes()
    ml, secs = C.read_container(tmp_path / "ours", device="cuda")
    assert ml == 7 and secs[0].arrays["big"].is_cuda
    assert torch.equal(secs[0].arrays["big"], big)
    assert torch.equal(secs[1].arrays["codes"], codes)
    assert secs[1].arrays["empty"].numel() == 0
