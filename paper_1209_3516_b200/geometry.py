"""Particles and boxes (the reference's src/geometry.py:168-270 surface).

``ParticleSet`` keeps the reference's structure-of-arrays contract:
positions and charges in, ``phi`` and ``fx/fy/fz`` accumulators out, one
length for all arrays.  Two storage forms are accepted:

* NumPy arrays (the reference's form): ``x, y, z, q`` read as float64
  exactly as in the reference (``geometry.py:231-241``).  A float32 cloud
  is kept as given and upcast lazily on access, so ``build_tree`` ships
  half the bytes to the device and upcasts there (exact either way).
* torch CUDA tensors (float32 or float64): kept on the device as given, so
  a device-resident cloud is solved without host traffic.  The kernels
  upcast to float64 for keys and geometry (bit-exact with the reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

MAX_LEVEL = 21  # src/geometry.py:17

__all__ = ["MAX_LEVEL", "Aabb", "ParticleSet", "compute_bounds", "generate_distribution", "load_particles_csv",
           "save_particles_csv"]


def _is_torch(a) -> bool:
    return isinstance(a, torch.Tensor)


@dataclass(frozen=True)
class Aabb:
    """Axis-aligned box given by its two corners (src/geometry.py:168-197)."""

    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self) -> None:
        object.__setattr__(self, "lo", np.asarray(self.lo, dtype=np.float64).reshape(3).copy())
        object.__setattr__(self, "hi", np.asarray(self.hi, dtype=np.float64).reshape(3).copy())
        if not np.all(self.hi >= self.lo):
            raise ValueError("Aabb hi must be >= lo on every axis")

    @property
    def center(self) -> np.ndarray:
        return 0.5 * (self.lo + self.hi)

    @property
    def extent(self) -> np.ndarray:
        return self.hi - self.lo

    def contains(self, pts: np.ndarray) -> np.ndarray:
        pts = np.atleast_2d(pts)
        return np.all((pts >= self.lo) & (pts <= self.hi), axis=1)


class ParticleSet:
    """Structure-of-arrays bodies (src/geometry.py:213-270)."""

    _raw = None
    _f64 = None

    def __init__(self, x, y, z, q, phi=None, fx=None, fy=None, fz=None):
        if _is_torch(x):
            arrs = [x, y, z, q]
            if not all(_is_torch(a) for a in arrs):
                raise TypeError("mix of torch tensors and other arrays")
            dev = x.device
            arrs = [a.contiguous() for a in arrs]
            if any(a.device != dev for a in arrs):
                raise ValueError("particle tensors live on different devices")
            if any(a.dtype not in (torch.float32, torch.float64) for a in arrs):
                raise TypeError("particle tensors must be float32 or float64")
            if len({a.dtype for a in arrs}) != 1:
                arrs = [a.to(torch.float64) for a in arrs]
            self.x, self.y, self.z, self.q = arrs
            n = self.x.shape[0]
            acc = []
            for a in (phi, fx, fy, fz):
                acc.append(torch.zeros(n, dtype=torch.float64, device=dev) if a is None
                           else torch.as_tensor(a, dtype=torch.float64, device=dev).contiguous())
            self.phi, self.fx, self.fy, self.fz = acc
        else:
            raw = [np.asarray(a) for a in (x, y, z, q)]
            if all(a.dtype == np.float32 for a in raw):
                # float32 host cloud: kept as given (the device upcasts it
                # exactly); the float64 views are materialised on access
                self._raw = [np.ascontiguousarray(a) for a in raw]
                self._f64 = [None] * 4
            else:
                self._raw = None
                self._f64 = [np.ascontiguousarray(a, dtype=np.float64) for a in raw]
            n = (self._raw or self._f64)[0].shape[0]
            self._n = int(n)
            # zero accumulators are materialised on first access (they are
            # written on the device; allocating 4 x 8 B x N zeros up front
            # costs milliseconds per call on large clouds)
            for name, a in zip(("phi", "fx", "fy", "fz"), (phi, fx, fy, fz)):
                if a is not None:
                    object.__setattr__(self, name, np.ascontiguousarray(a, dtype=np.float64))
        # (stored arrays: reading self.x here would upcast a float32 cloud)
        stored = self.host_inputs() if self._f64 is not None else (self.x, self.y, self.z, self.q)
        accs = [self.__dict__[k] for k in ("phi", "fx", "fy", "fz") if k in self.__dict__]
        lengths = {int(a.shape[0]) for a in (*stored, *accs)}
        if lengths != {int(n)}:
            raise ValueError(f"particle arrays disagree on length: {sorted(lengths)}")

    # float64 views of host inputs (the reference's storage form)
    def _get(self, k):
        if self._f64[k] is None:
            self._f64[k] = self._raw[k].astype(np.float64)
        return self._f64[k]

    def _set(self, k, v):
        if self._raw is not None:
            for j in range(4):
                self._get(j)
            self._raw = None
        self._f64[k] = np.ascontiguousarray(v, dtype=np.float64)

    def __getattr__(self, name):  # x, y, z, q of the host form; lazy zero accumulators
        if name in ("phi", "fx", "fy", "fz") and "_n" in self.__dict__:
            a = np.zeros(self.__dict__["_n"])
            object.__setattr__(self, name, a)
            return a
        idx = {"x": 0, "y": 1, "z": 2, "q": 3}.get(name)
        if idx is None or self.__dict__.get("_f64") is None:
            raise AttributeError(name)
        return self._get(idx)

    def __setattr__(self, name, value):
        idx = {"x": 0, "y": 1, "z": 2, "q": 3}.get(name)
        if idx is not None and not isinstance(value, torch.Tensor) and self.__dict__.get("_f64") is not None:
            self._set(idx, value)
        else:
            object.__setattr__(self, name, value)

    def host_inputs(self):
        """(x, y, z, q) host arrays in their stored precision (no copy)."""
        return tuple(self._raw) if self._raw is not None else tuple(self._f64)

    @property
    def n(self) -> int:
        # (a host float32 cloud must not be read through self.x here: that
        # materialises its float64 view, ~1 ms of conversions at 2^20 bodies)
        if "_n" in self.__dict__:
            return self.__dict__["_n"]
        return int(self.x.shape[0])

    @property
    def on_device(self) -> bool:
        return self._raw is None and self._f64 is None

    def positions(self) -> np.ndarray:
        return np.column_stack([_np(self.x), _np(self.y), _np(self.z)])

    def reset_accumulators(self) -> None:
        for a in (self.phi, self.fx, self.fy, self.fz):
            a[:] = 0.0

    def view(self, start: int, stop: int) -> "ParticleSet":
        """Shared-memory slice; writes to accumulators land in the parent."""
        return ParticleSet(*(a[start:stop] for a in (self.x, self.y, self.z, self.q, self.phi, self.fx,
                                                     self.fy, self.fz)))

    def copy(self) -> "ParticleSet":
        return ParticleSet(*(a.clone() if _is_torch(a) else a.copy()
                             for a in (self.x, self.y, self.z, self.q, self.phi, self.fx, self.fy, self.fz)))

    def permuted(self, perm) -> "ParticleSet":
        return ParticleSet(*(a[perm].clone() if _is_torch(a) else a[perm].copy()
                             for a in (self.x, self.y, self.z, self.q, self.phi, self.fx, self.fy, self.fz)))

    def numpy(self) -> "ParticleSet":
        """Host float64 copy (the reference's storage form)."""
        return ParticleSet(*(_np(a) for a in (self.x, self.y, self.z, self.q, self.phi, self.fx, self.fy,
                                              self.fz)))


def _np(a) -> np.ndarray:
    if _is_torch(a):
        return a.detach().to("cpu", torch.float64).numpy()
    return np.asarray(a, dtype=np.float64)


def compute_bounds(ps: ParticleSet) -> Aabb:
    """Tight bounding box of all bodies (src/geometry.py:200-206)."""
    if ps.n == 0:
        raise ValueError("empty particle set")
    if ps.on_device:
        lo = [float(a.min()) for a in (ps.x, ps.y, ps.z)]
        hi = [float(a.max()) for a in (ps.x, ps.y, ps.z)]
        return Aabb(np.array(lo), np.array(hi))
    lo = np.array([ps.x.min(), ps.y.min(), ps.z.min()])
    hi = np.array([ps.x.max(), ps.y.max(), ps.z.max()])
    return Aabb(lo, hi)


def generate_distribution(kind: str, n: int, seed: int = 0) -> ParticleSet:
    """Seeded benchmark cloud (src/geometry.py:273-287): ``uniform`` (alias
    ``cube``) positions in [0, 1)^3 from ``default_rng(seed)``, every charge
    1/n (total charge one)."""
    if n <= 0:
        raise ValueError(f"n must be positive, got {n}")
    if kind not in ("uniform", "cube"):
        raise ValueError(f"unknown distribution kind: {kind!r}")
    pts = np.random.default_rng(seed).random((n, 3))
    return ParticleSet(pts[:, 0], pts[:, 1], pts[:, 2], np.full(n, 1.0 / n))


def save_particles_csv(ps: ParticleSet, path: str) -> None:
    """Bodies as CSV with header ``x,y,z,q``, full float64 round trip
    (src/geometry.py:290-297)."""
    cols = [_np(a) for a in (ps.x, ps.y, ps.z, ps.q)]
    with open(path, "w", newline="") as fh:
        fh.write("x,y,z,q\n")
        for i in range(ps.n):
            fh.write(",".join(repr(float(c[i])) for c in cols) + "\n")


def load_particles_csv(path: str) -> ParticleSet:
    """Bodies from a CSV with header ``x,y,z,q`` (src/geometry.py:298-318);
    ValueError with the line number on malformed input."""
    import csv

    rows = []
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None or [h.strip().lower() for h in header] != ["x", "y", "z", "q"]:
            raise ValueError(f"bad particle CSV header in {path}: expected x,y,z,q")
        for lineno, row in enumerate(reader, start=2):
            if not row:
                continue
            if len(row) != 4:
                raise ValueError(f"bad particle CSV row at line {lineno}: expected 4 fields")
            try:
                rows.append([float(v) for v in row])
            except ValueError as exc:
                raise ValueError(f"bad particle CSV value at line {lineno}: {exc}") from None
    if not rows:
        raise ValueError(f"empty particle set in {path}")
    a = np.asarray(rows, dtype=np.float64)
    return ParticleSet(a[:, 0], a[:, 1], a[:, 2], a[:, 3])
