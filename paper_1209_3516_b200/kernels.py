"""Kernel counters and the device direct-sum checker (src/kernels.py:1-228).

Physics conventions (fixed, as in the reference):

* potential  phi(x_i) = sum_{j != i} q_j / |x_i - x_j|
* force      f(x_i)   = -grad phi = sum_{j != i} q_j (x_i - x_j) / r^3
* an order-p expansion keeps multi-indices with |m| < p
  (p(p+1)(p+2)/6 coefficients, graded-lex order)
* coincident bodies (r = 0) are skipped and counted in ``p2p_skipped``;
  ``p2p_flops == 20 * p2p_pairs`` by construction.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .geometry import ParticleSet

TMAX = 12
P2P_FLOPS_PER_PAIR = 20

__all__ = ["TMAX", "P2P_FLOPS_PER_PAIR", "KernelStats", "ncoef", "direct"]


def ncoef(p: int) -> int:
    """Coefficient count of an order-p expansion: p(p+1)(p+2)/6."""
    return p * (p + 1) * (p + 2) // 6


@dataclass
class KernelStats:
    """Kernel-call counters and per-kernel times in seconds (src/kernels.py:71-119)."""

    p2p_pairs: int = 0
    p2p_skipped: int = 0
    p2p_flops: int = 0
    m2l_calls: int = 0
    m2p_calls: int = 0
    p2m_calls: int = 0
    m2m_calls: int = 0
    l2l_calls: int = 0
    l2p_calls: int = 0
    times: dict = field(default_factory=dict)

    def add_time(self, key: str, seconds: float) -> None:
        self.times[key] = self.times.get(key, 0.0) + seconds

    def merge(self, other: "KernelStats") -> None:
        for k in ("p2p_pairs", "p2p_skipped", "p2p_flops", "m2l_calls", "m2p_calls", "p2m_calls",
                  "m2m_calls", "l2l_calls", "l2p_calls"):
            setattr(self, k, getattr(self, k) + getattr(other, k))
        for k, v in other.times.items():
            self.add_time(k, v)

    def as_dict(self) -> dict:
        return {
            "p2p_pairs": self.p2p_pairs,
            "p2p_skipped": self.p2p_skipped,
            "p2p_flops": self.p2p_flops,
            "m2l_calls": self.m2l_calls,
            "m2p_calls": self.m2p_calls,
            "p2m_calls": self.p2m_calls,
            "m2m_calls": self.m2m_calls,
            "l2l_calls": self.l2l_calls,
            "l2p_calls": self.l2p_calls,
            "times": {k: float(v) for k, v in sorted(self.times.items())},
        }


def direct(ps: ParticleSet, target_indices=None, *, device=None):
    """O(S*N) direct sums on the GPU (src/kernels.py:208-228).

    Returns fresh float64 numpy (phi, fx, fy, fz) for the selected targets
    (all bodies by default); accumulators on ``ps`` are left untouched.
    """
    _lib.require_cuda()
    if ps.n == 0:
        raise ValueError("empty particle set")
    dev = torch.device(device) if device is not None else (
        ps.x.device if ps.on_device else torch.device("cuda", torch.cuda.current_device()))
    xs = [torch.as_tensor(a, device=dev).to(torch.float64).contiguous() for a in (ps.x, ps.y, ps.z, ps.q)]
    if target_indices is None:
        tidx = torch.arange(ps.n, dtype=torch.int64, device=dev)
    else:
        t = np.ascontiguousarray(np.asarray(target_indices, dtype=np.int64)) \
            if not isinstance(target_indices, torch.Tensor) else target_indices
        tidx = torch.as_tensor(t, dtype=torch.int64, device=dev).contiguous()
        if tidx.numel() and (int(tidx.min()) < 0 or int(tidx.max()) >= ps.n):
            raise ValueError("target index out of range")
    out = [torch.empty(tidx.numel(), dtype=torch.float64, device=dev) for _ in range(4)]
    with torch.cuda.device(dev):
        _lib.call("fmm_direct", ps.n, *(_lib.ptr(a) for a in xs), tidx.numel(), _lib.ptr(tidx),
                  *(_lib.ptr(o) for o in out), _lib.stream_handle())
    return tuple(o.cpu().numpy() for o in out)
