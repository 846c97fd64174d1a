"""Seeded synthetic particle clouds for the BASELINE.json configurations.

The reference package only ships ``generate_distribution("uniform")`` with
q = 1/n (``/root/reference/pkg/src/fmmkit/geometry.py:273-287``); the
benchmark configurations use their own charge laws and a Plummer sphere, so
the recipes are fixed here once and feed
both the reference/oracle runs and the GPU runs.  Every generator draws from
``numpy.random.default_rng(seed)`` in the documented order, so the bodies
are bit-identical wherever they are regenerated.

All generators return ``(pos, q)`` with ``pos`` of shape (N, 3).  The
``dtype`` of the returned arrays is the configuration's input precision
(float64 for C1, float32 for C2-C5); the solver upcasts to float64 exactly
as the reference's ``ParticleSet`` does (``geometry.py:231-241``).
"""

from __future__ import annotations

import itertools
import math

import numpy as np

__all__ = [
    "config1", "config2", "plummer", "config4", "config5",
    "uniform_unit", "clustered_points", "CONFIGS",
]


def uniform_unit(n: int, seed: int = 0):
    """``generate_distribution("uniform", n, seed)``: [0,1)^3, q = 1/n."""
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3))
    q = np.full(n, 1.0 / n)
    return pos, q


def config1(n: int = 10_000, seed: int = 0):
    """C1: float64 uniform cube, q ~ U[-1,1) mean-subtracted."""
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3))
    q = rng.uniform(-1.0, 1.0, n)
    q -= q.mean()
    return pos, q


def config2(n: int = 1 << 20, seed: int = 0):
    """C2: FP32 uniform cube, q ~ U[0,1) FP32."""
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3)).astype(np.float32)
    q = rng.random(n).astype(np.float32)
    return pos, q


def plummer(n: int = 1 << 22, seed: int = 0, a: float = 1.0, rcut: float = 10.0):
    """C3: Plummer sphere (scale a, truncated at rcut*a), inverse-CDF sampled.

    M(r) = r^3 / (r^2 + 1)^{3/2} is the enclosed-mass fraction in units of a;
    u ~ U[0, M(rcut)) gives r = a (u^{-2/3} - 1)^{-1/2}.  Directions are
    isotropic (cos(theta) ~ U[-1,1), phi ~ U[0, 2 pi)).  FP32 positions,
    equal charges 1/N in FP32.
    """
    rng = np.random.default_rng(seed)
    mcut = rcut ** 3 / (rcut ** 2 + 1.0) ** 1.5
    u = rng.random(n) * mcut
    # libm pow/cos/sin through ``math`` (not numpy's CPU-dispatched SIMD
    # loops) so the cloud is bit-identical on every x86 host of this image
    upow = np.fromiter(map(math.pow, u, itertools.repeat(-2.0 / 3.0)), np.float64, n)
    r = a / np.sqrt(upow - 1.0)
    cth = 2.0 * rng.random(n) - 1.0
    ph = 2.0 * math.pi * rng.random(n)
    sth = np.sqrt(np.maximum(0.0, 1.0 - cth * cth))
    cph = np.fromiter(map(math.cos, ph), np.float64, n)
    sph = np.fromiter(map(math.sin, ph), np.float64, n)
    pos = np.stack([r * sth * cph, r * sth * sph, r * cth], axis=1)
    pos = pos.astype(np.float32)
    q = np.full(n, 1.0 / n, dtype=np.float32)
    return pos, q


def config4(n: int = 1 << 20, seed: int = 0):
    """C4: FP32 uniform cube, q ~ U[-1,1) FP32."""
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3)).astype(np.float32)
    q = rng.uniform(-1.0, 1.0, n).astype(np.float32)
    return pos, q


def config5(n: int = 1 << 24, seed: int = 0):
    """C5: FP32 uniform cube, q ~ U[0,1) FP32 (same law as C2)."""
    return config2(n, seed)


def clustered_points(n: int, seed: int = 0):
    """Blob mixture with very uneven density (the reference's test fixture
    generator, ``/root/reference/pkg/tests/conftest.py:32-40``)."""
    rng = np.random.default_rng(seed)
    centers = rng.random((4, 3))
    scales = np.array([0.002, 0.01, 0.05, 0.2])
    which = rng.integers(0, 4, size=n)
    pts = centers[which] + scales[which, None] * rng.standard_normal((n, 3))
    q = rng.uniform(-1.0, 1.0, size=n)
    return pts, q


# name -> (generator, default N, solver parameters)
CONFIGS = {
    "C1": (config1, 10_000, dict(p=4, theta=0.4, ncrit=64)),
    "C2": (config2, 1 << 20, dict(p=4, theta=0.4, ncrit=64)),
    "C3": (plummer, 1 << 22, dict(p=5, theta=0.5, ncrit=64)),
    "C4": (config4, 1 << 20, dict(p=4, theta=0.4, ncrit=64)),
    "C5": (config5, 1 << 24, dict(p=4, theta=0.4, ncrit=128)),
}
