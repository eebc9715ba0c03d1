"""Synthetic inputs of the benchmark configurations (BASELINE.json `configs`).

`generate` reproduces the reference generator byte for byte
(pkg/src/fmmkit/cli.py:68-85): numpy Philox streams spawned from
SeedSequence(seed) — one for sources, one for receivers, one for charges —
uniform points in [0,1)^3 or a sphere shell of radius 0.45 around 0.5.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import FmmError

SPHERE_RADIUS = 0.45  # cli.py:39
SPHERE_CENTER = 0.5  # cli.py:40


def generate(n_sources: int, n_receivers: int, dist: str = "uniform", seed: int = 0):
    """(src (N,3) f64, charges (N,) f64, recv (M,3) f64), as cli.generate."""
    streams = np.random.SeedSequence(seed).spawn(3)
    gen_src, gen_recv, gen_q = (np.random.Generator(np.random.Philox(s)) for s in streams)

    def draw(gen, n):
        if dist == "uniform":
            return gen.random((n, 3))
        if dist == "sphere":
            v = gen.normal(size=(n, 3))
            v /= np.linalg.norm(v, axis=1, keepdims=True)
            return v * SPHERE_RADIUS + SPHERE_CENTER
        raise FmmError(f"unknown distribution {dist!r}")

    src = draw(gen_src, n_sources)
    recv = draw(gen_recv, n_receivers)
    charges = gen_q.normal(size=n_sources)
    return src, charges, recv


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    level: int
    dist: str
    seed: int


# BASELINE.json configs (c5 is the multi-GPU one; c4 perturbs c4 points each step)
WORKLOADS = {
    "c1": Workload("c1", 2**16, 4, "uniform", 1),
    "c2": Workload("c2", 2**24, 7, "uniform", 1),
    "c3": Workload("c3", 2**24, 9, "sphere", 1),
    "c4": Workload("c4", 2**23, 7, "uniform", 4),
    "c5": Workload("c5", 2**30, 8, "uniform", 1),
}


def perturb(points: np.ndarray, rng: np.random.Generator, scale: float = 1e-3) -> np.ndarray:
    """c4 dynamic-rebuild step: x <- mod(x + N(0, scale), 1.0)."""
    return np.mod(points + rng.normal(scale=scale, size=points.shape), 1.0)


# coordinates whose perturbed value np.mod maps to exactly 1.0 (x + noise a
# tiny negative number): the clamp edge of the encoder (_ckernels.pyx:97-102)
C4_EDGE_SLOTS = ((5, 0), (77, 1), (4242, 2), (31337, 0), (31337, 1), (31337, 2))


def c4_step_inputs(n: int = 2**23, seed: int = 4, steps: int = 1):
    """Inputs of the c4 golden rebuild step: generate(n, n, uniform, seed),
    then `steps` perturbations of src and recv drawn from default_rng(123)
    (src first, then recv, as the trajectory driver), with C4_EDGE_SLOTS set
    to np.mod(-1e-18, 1.0) == 1.0 on both sets so the clamp edge is always
    present (a random perturbation reaches it with probability ~1e-9)."""
    src, q, recv = generate(n, n, "uniform", seed)
    rng = np.random.default_rng(123)
    for _ in range(steps):
        src = perturb(src, rng)
        recv = perturb(recv, rng)
    edge = np.mod(np.float64(-1e-18), 1.0)
    for i, j in C4_EDGE_SLOTS:
        if i < n:
            src[i, j] = edge
            recv[i, j] = edge
    return src, q, recv


def perturb_device(points, seed: int, step: int, scale: float = 1e-3):
    """c4 rebuild step on the device, in place: x <- mod(x + N(0, scale), 1.0)
    in one fused libfmmb200 pass (fmmb_perturb: Philox4x32-10 normals keyed
    by (seed, step), np.mod's convention, so a tiny negative sum maps to
    exactly 1.0).  Workload driver only (not part of the build path)."""
    from . import _lib

    if not (points.is_cuda and points.dtype.is_floating_point and points.is_contiguous()):
        raise FmmError("perturb_device needs a contiguous f64 CUDA tensor")
    dev = _lib.device_of(points.device)
    h = _lib.handle(dev)
    st = _lib.load().fmmb_perturb(h, points.data_ptr(), points.numel(), int(seed) & (2**64 - 1),
                                  int(step), float(scale), _lib.stream_of(dev))
    _lib.check(st, h)
    return points
