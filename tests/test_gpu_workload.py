"""c4 workload driver: the fused device perturbation (fmmb_perturb)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_perturb_device_is_reproducible_and_distributed(gpu):
    from paper_1301_1704_b200.workloads import perturb_device

    dev = torch.device("cuda", 0)
    base = torch.rand(1_000_001, dtype=torch.float64, device=dev) * 0.5 + 0.25
    a = perturb_device(base.clone(), 123, 7)
    b = perturb_device(base.clone(), 123, 7)
    c = perturb_device(base.clone(), 123, 8)
    assert torch.equal(a, b) and not torch.equal(a, c)
    d = (a - base).cpu().numpy()
    assert abs(d.mean()) < 5e-6 and abs(d.std() - 1e-3) < 2e-5
    # np.mod convention at the unit-cube edges: result in [0, 1], a tiny
    # negative sum lands on exactly 1.0, wrap-around above 1
    edge = torch.tensor([0.0, 1e-300, 0.999999999], dtype=torch.float64, device=dev)
    for step in range(50):
        e = perturb_device(edge.clone(), 5, step).cpu().numpy()
        assert np.all((e >= 0.0) & (e <= 1.0))
    ref = np.mod(base.cpu().numpy() + d, 1.0)
    assert np.allclose(a.cpu().numpy(), ref, rtol=0, atol=1e-15)
