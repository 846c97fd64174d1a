"""Dual-tree evaluation on the B200 (src/traversal.py:54-137, :864-932, :1202-1206).

``evaluate_dual_tree`` runs, all on the device:

1. ``upward_pass`` if the tree has no multipoles of order p;
2. the breadth-first dual traversal (csrc/traverse.cu) -> M2L and P2P pair
   lists, bit-exact sets with the reference's ``_collect_units``;
3. CSR by target (radix sort), the P2P run plan (csrc/plan.cu) and the
   reference's pair counters;
4. M2L over the target CSR (csrc/m2l.cu) and P2P over the plan
   (csrc/p2p.cu, FP32 or FP64);
5. ``downward_pass`` (L2L, L2P).

Phase times follow the reference's ``EvalReport`` (build, upward, traversal,
downward; ``total_time`` sums them) and are measured with CUDA events on the
evaluation stream; ``stats.times`` holds the per-kernel-class split
("list", "m2l", "p2p").

``evaluate_treecode`` walks every target leaf against
the tree (csrc/traverse.cu, bit-exact sets with ``_collect_treecode``),
evaluates accepted cells' multipoles at the bodies (M2P, csrc/m2p.cu) and
reuses the P2P plan and kernel for the near field.

``evaluate_list_fmm`` builds the level-wise V/U lists
(csrc/traverse.cu, bit-exact sets with ``_collect_vlist``/``_collect_ulist``)
and reuses the M2L, P2P and downward executors.

Scope: all three strategies (``dualtree`` directed, ``treecode``,
``listfmm``) on one shared tree, and ``dualtree`` / ``treecode`` with a
separate ``source_tree``: the source bodies are appended
after the targets in one set of P2P body arrays, the traversals read the two
trees' cell arrays, M2L/M2P read the source tree's multipoles and the P2P
plan's runs point past the targets.  ``mutual=True``
runs the mutual traversal (``mutual_lists``): the reference's mutual list
sets, partition demotion included, written directed so the same M2L / P2P
executors evaluate them.
``precision`` is a new knob: "fp64" (default, the reference's arithmetic),
"fp32" (FP32 near field; far field stays float64) or "fp32acc" (float32
pair terms summed in float64; ~1e-7 near-field floor for ~5 % more time).
"""

from __future__ import annotations

import ctypes as C
import json
import os
import threading
import weakref
from dataclasses import dataclass, field

import torch

from . import _lib
from .kernels import TMAX, KernelStats, ncoef
from .mac import MacConfig
from .tree import Tree, downward_pass, upward_pass

STRATEGIES = ("treecode", "listfmm", "dualtree")
PRECISIONS = ("fp64", "fp32", "fp32acc")
REPORT_SCHEMA = "fmmkit-report-v1"

__all__ = ["STRATEGIES", "PRECISIONS", "EvalConfig", "EvalReport", "evaluate_dual_tree", "evaluate_list_fmm",
           "evaluate_treecode", "evaluate_on_tree", "interaction_lists", "listfmm_lists", "treecode_lists"]


@dataclass
class EvalConfig:
    """Knobs of one evaluation run (src/traversal.py:61-80) + ``precision``."""

    strategy: str = "dualtree"
    mac: MacConfig = field(default_factory=lambda: MacConfig("fmm", 0.6))
    p: int = 4
    mutual: bool = False
    task_grain: int = 5000
    use_rsqrt: bool = False
    precision: str = "fp64"
    symmetric: bool | None = None  # mutual=True: symmetric executors (None: FMM_B200_SYMMETRIC, default off)

    def __post_init__(self) -> None:
        if self.strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {self.strategy!r}: expected one of {STRATEGIES}")
        if not isinstance(self.mac, MacConfig):
            raise TypeError("mac must be a MacConfig")
        if not 1 <= self.p <= TMAX:
            raise ValueError(f"expansion order {self.p} outside supported range 1..{TMAX}")
        if self.task_grain < 1:
            raise ValueError(f"task_grain must be >= 1, got {self.task_grain}")
        if self.precision not in PRECISIONS:
            raise ValueError(f"unknown precision {self.precision!r}: expected one of {PRECISIONS}")


@dataclass
class EvalReport:
    """Outcome of one evaluation (src/traversal.py:83-137)."""

    strategy: str
    n: int
    n_sources: int
    p: int
    mac_kind: str
    theta: float
    mutual: bool
    threads: int
    task_grain: int
    stats: KernelStats
    build_time: float
    upward_time: float
    traversal_time: float
    downward_time: float
    achieved_error: float | None = None
    trace: list | None = None
    # raw per-stream spans (seconds) of the overlapped evaluation; the phase
    # times above are their critical-path split (``critical_path``)
    spans: dict = field(default_factory=dict)
    near_field: str = "fp64"

    @property
    def total_time(self) -> float:
        return self.build_time + self.upward_time + self.traversal_time + self.downward_time

    def to_dict(self) -> dict:
        counts = {k: v for k, v in self.stats.as_dict().items() if k != "times"}
        return {
            "schema": REPORT_SCHEMA,
            "params": {"strategy": self.strategy, "n": self.n, "n_sources": self.n_sources, "p": self.p,
                       "mac": self.mac_kind, "theta": self.theta, "mutual": self.mutual,
                       "threads": self.threads, "task_grain": self.task_grain},
            "counts": counts,
            "times_ms": {"build": int(round(self.build_time * 1e3)),
                         "upward": int(round(self.upward_time * 1e3)),
                         "traversal": int(round(self.traversal_time * 1e3)),
                         "downward": int(round(self.downward_time * 1e3)),
                         "total": int(round(self.total_time * 1e3))},
            "kernel_times_ms": {k: int(round(v * 1e3)) for k, v in sorted(self.stats.times.items())},
            "achieved_error": self.achieved_error,
            # additive keys (not in the reference's schema)
            "stream_spans_ms": {k: round(v * 1e3, 3) for k, v in sorted(self.spans.items())},
            "near_field_precision": self.near_field,
        }

    def to_json(self, indent: int = 2) -> str:
        return json.dumps(self.to_dict(), indent=indent)


def critical_path(t_near: float, t_up: float, t_far: float, wall: float) -> tuple[float, float, float]:
    """Split one overlapped evaluation's wall time into the reference's
    sequential phases (src/traversal.py:104-106, :875-931), so that
    upward + traversal + downward == wall (times from the evaluation start):

    * traversal: until the near field (lists + P2P) ends, plus any far-field
      interaction (M2L / M2P) still running after it and after the upward
      pass -- the reference's traversal phase runs M2L and P2P;
    * upward: the part of the upward pass that outlasts the near field;
    * downward: the remainder (L2L/L2P tail and the final combine).

    ``t_near``/``t_up``/``t_far`` are the end times of the near field, the
    upward pass and the far-field interactions."""
    up = max(0.0, t_up - t_near)
    trav = t_near + max(0.0, t_far - max(t_near, t_up))
    return up, trav, max(0.0, wall - up - trav)


def _setup_gap(tree: Tree, e0) -> float:
    """Seconds between the end of ``tree``'s build and this evaluation's
    first event, once per build: host set-up the reference bills to its
    upward phase (src/traversal.py:875-879).  The first evaluation after a
    build also replaces the build's host-timed ``build_time`` by its span
    on the device timeline (the evaluation has synchronised by now), so
    build + upward + traversal + downward tiles the device time."""
    ev = tree.__dict__.pop("_ev_built", None)
    ev0 = tree.__dict__.pop("_ev_build_start", None)
    if ev is None:
        return 0.0
    if ev0 is not None:
        tree.build_time = ev0.elapsed_time(ev) * 1e-3
    return ev.elapsed_time(e0) * 1e-3


_TIMED = frozenset(("stats", "build_time", "upward_time", "traversal_time", "downward_time", "spans"))


class DeferredReport(EvalReport):
    """An ``EvalReport`` whose times are read from the evaluation's CUDA
    events on first use.  Each ``Event.elapsed_time`` costs ~7 us of host time
    and the report needs 14 of them, all after the evaluation's final
    synchronisation, when the GPU has nothing left to do: read eagerly they
    are 0.7 % of a C2 step.  The counters are final when the report is
    returned; ``stats.times``, the phase times and ``spans`` are filled by
    ``resolve_times`` when any of them (or ``stats``) is first touched, or by
    the thread's next evaluation while its kernels run (``_EventPool``: the
    events are double-buffered, so they stay intact until then)."""

    def __getattribute__(self, name):
        if name in _TIMED:
            thunk = object.__getattribute__(self, "__dict__").pop("_thunk", None)  # (atomic: one caller runs it)
            if thunk is not None:
                thunk(self)
        return object.__getattribute__(self, name)

    def resolve_times(self) -> None:
        thunk = self.__dict__.pop("_thunk", None)
        if thunk is not None:
            thunk(self)


# ---------------------------------------------------------------------------
# traversal -> CSR lists
# ---------------------------------------------------------------------------
class Lists:
    """Device interaction lists of one traversal (CSR by target cell).

    A traversal run from a capacity hint does not wait for its counters:
    ``settle()`` reads them later (one host synchronisation, at the end of
    the evaluation) and reports whether every list fit its buffer; until
    then ``n_m2l`` / ``n_p2p`` / ``peak_frontier`` are read on demand."""

    _COUNTS = ("n_m2l", "n_p2p", "peak_frontier")

    def __init__(self, **kw):
        self.__dict__.update(kw)

    def __getattr__(self, name):
        if name == "p2p_src" and "p2p_grp" in self.__dict__:
            # the P2P plan reads its rows unsorted; sort them when asked
            grp, rows = self.__dict__["p2p_grp"], self.__dict__["p2p_rows"]
            out = torch.empty_like(grp)
            wsp, wsb = _lib.workspace(rows.numel(), grp.device)
            _lib.call("fmm_sort_rows", rows.numel() - 1, _lib.ptr(rows), _lib.ptr(grp), _lib.ptr(out), wsp, wsb,
                      _lib.stream_handle())
            self.__dict__["p2p_src"] = out
            return out
        if name in Lists._COUNTS and self.__dict__.get("_deferred") is not None:
            if not self.settle():
                raise RuntimeError("interaction lists overflowed their capacity hint; re-evaluate")
            return self.__dict__[name]
        raise AttributeError(name)

    def device_counters(self) -> list:
        """The device tensors ``settle`` and the pair counters read (int64),
        for one batched copy to the host (``EndReadback``)."""
        out = [self.dev_stats.long(), self.dev_runs_needed.long()]
        d = self.__dict__.get("_deferred")
        if d is not None:
            out.append(d[0].long())
        return out

    def settle(self, host=None) -> bool:
        """Read deferred traversal counters; False if a list overflowed (the
        lists are then incomplete and the evaluation must be redone).
        ``host`` holds ``device_counters()`` already copied to the host."""
        d = self.__dict__.get("_deferred")
        if d is None:
            return True
        log, caps, key = d
        hl = host[2].tolist() if host is not None else log.tolist()
        runs_needed = int(host[1][0]) if host is not None else int(self.__dict__["dev_runs_needed"][0])
        n_p2p, n_m2l, fronts = hl[0], hl[1], hl[2:]
        peak = max(fronts)
        self.__dict__.update(n_p2p=n_p2p, n_m2l=n_m2l, peak_frontier=peak, _deferred=None)
        ok = n_p2p <= caps[0] and n_m2l <= caps[1] and peak <= caps[2] and fronts[-1] == 0
        ok = ok and runs_needed == 0  # (runs are sized like pairs)
        if ok:
            _hint[key] = (max(caps[0], int(n_p2p * 1.02) + 4096), max(caps[1], int(n_m2l * 1.02) + 4096),
                          max(caps[2], int(peak * 1.05) + 4096))
        else:
            _hint.pop(key, None)  # the redo takes the synchronising path
        return ok

    def host_pairs(self, which: str):
        """(targets, sources) int64 numpy arrays sorted by (target, source)."""
        if self.__dict__.get("_deferred") is not None and not self.settle():
            raise RuntimeError("interaction lists overflowed their capacity hint; build them again")
        rows = getattr(self, which + "_rows").cpu()
        src = getattr(self, which + "_src")[:int(rows[-1])].cpu().long()
        t = torch.repeat_interleave(torch.arange(rows.numel() - 1), rows[1:] - rows[:-1])
        sym = self.__dict__.get("sym_" + which)
        if sym is not None and sym.n:
            # unordered entries (a, b) stand for (a, b) and (b, a), the
            # reference's trace expansion (src/traversal.py:644-650)
            a, b = sym.pairs()
            t, src = torch.cat([t, a, b]), torch.cat([src, b, a])
            order = torch.argsort(t * (rows.numel() + 1) + src)
            t, src = t[order], src[order]
        return t.numpy(), src.numpy()


_hint = {}


def interaction_lists(tree: Tree, mac: MacConfig, body_range: tuple[int, int] | None = None,
                      m2l_ready: torch.cuda.Event | None = None,
                      side: torch.cuda.Stream | None = None, m2l_owner_only: bool = False,
                      src: Tree | None = None, defer: bool = False,
                      target_mask: torch.Tensor | None = None, sort_far: bool = True) -> Lists:
    """Dual traversal from (root, root) -> target-sorted CSR M2L/P2P lists
    (the sets of src/traversal.py:159-262).

    ``body_range=(lo, hi)`` keeps only pairs whose target cell holds bodies
    in [lo, hi) (a multi-GPU rank's share); the default keeps all.
    ``src`` is a separate source tree (cross-tree lists: sources index its
    cells, the P2P plan points at its bodies appended after the targets).
    With ``defer`` and a capacity hint for this shape the host does not wait
    for the traversal's counters: the caller must check ``Lists.settle`` and
    redo the traversal when a list outgrew its hinted buffer (the evaluators
    do, at their final read-back); the default waits and sizes exactly.  ``target_mask`` (uint8
    per target cell) keeps only the flagged targets' rows (sampled
    evaluations: ``tuner.ErrorProbe``)."""
    blo, bhi = body_range if body_range is not None else (0, tree.n)
    dev = tree.device
    P = _lib.ptr
    st = _lib.stream_handle()
    i32 = torch.int32
    th2 = mac.theta * mac.theta
    cross = src is not None and src is not tree
    sb = src if cross else tree
    tm = _lib.ptr(target_mask)
    key = (tree.ncells, tree.nleaves, mac.kind, th2, blo, bhi, m2l_owner_only, sb.ncells if cross else 0, tm)
    # every step opens one side of a pair: at most depth_A + depth_B + 1 steps
    nsteps = tree.depth + sb.depth + 2
    bcells = _source_cells(tree, src)
    log = torch.empty(nsteps + 3, dtype=torch.int64, device=dev)
    if defer and key in _hint and _sync_free():
        # capacities known from an earlier run of this shape: chain the
        # traversal, both CSRs and the plan on the device, no host wait
        cap_p2p, cap_m2l, cap_next = _hint[key]
        # one allocation for the pair buffers and the four frontiers
        pool = torch.empty(2 * cap_p2p + 2 * cap_m2l + 4 * cap_next, dtype=i32, device=dev)
        p2p_t, p2p_s, m2l_t, m2l_s, *fr = torch.split(pool, [cap_p2p, cap_p2p, cap_m2l, cap_m2l] + [cap_next] * 4)
        _lib.call("fmm_traverse", P(fr[0]), P(fr[1]), P(fr[2]), P(fr[3]), cap_next, nsteps, P(tree.d_children),
                  P(tree.d_leaf), P(tree.d_ctr), P(tree.d_bmax), P(tree.d_rmax), *bcells, P(tree.d_start),
                  P(tree.d_end), blo, bhi, tm, int(m2l_owner_only), mac.code, th2, P(p2p_t), P(p2p_s), cap_p2p,
                  P(m2l_t), P(m2l_s), cap_m2l, P(log), st)
        del fr
        ncells = tree.ncells
        items = max(cap_p2p, cap_m2l, tree.n, ncells + 1)
        wsp, wsb = _lib.workspace(items, dev, stream=torch.cuda.current_stream())
        m2l_src, m2l_rows = _far_csr(m2l_t, m2l_s, cap_m2l, ncells, dev, wsp, wsb, st, side, m2l_ready,
                                     dev_n=log[1:], nsrc=sb.ncells, sort=sort_far)
        p2p_grp, p2p_rows = _csr(p2p_t, p2p_s, cap_p2p, ncells, dev, wsp, wsb, st, dev_n=log, nsrc=sb.ncells,
                                 sort=False)
        del p2p_t, p2p_s, m2l_t, m2l_s
        return Lists(m2l_src=m2l_src, m2l_rows=m2l_rows, p2p_rows=p2p_rows,
                     _deferred=(log, (cap_p2p, cap_m2l, cap_next), key),
                     **_p2p_plan(tree, p2p_grp, p2p_rows, cap_p2p, blo, bhi, wsp, wsb, st, src=src, tmask=target_mask))
    cap_p2p, cap_m2l, cap_next = _hint.get(key, (max(4096, tree.nleaves * 64), max(4096, tree.ncells * 32),
                                                 max(4096, tree.ncells * 8)))
    while True:
        p2p_t = torch.empty(cap_p2p, dtype=i32, device=dev)
        p2p_s = torch.empty(cap_p2p, dtype=i32, device=dev)
        m2l_t = torch.empty(cap_m2l, dtype=i32, device=dev)
        m2l_s = torch.empty(cap_m2l, dtype=i32, device=dev)
        fr = [torch.empty(cap_next, dtype=i32, device=dev) for _ in range(4)]
        _lib.call("fmm_traverse", P(fr[0]), P(fr[1]), P(fr[2]), P(fr[3]), cap_next, nsteps, P(tree.d_children),
                  P(tree.d_leaf), P(tree.d_ctr), P(tree.d_bmax), P(tree.d_rmax), *bcells, P(tree.d_start),
                  P(tree.d_end), blo, bhi, tm, int(m2l_owner_only), mac.code, th2, P(p2p_t), P(p2p_s), cap_p2p, P(m2l_t),
                  P(m2l_s), cap_m2l, P(log), st)
        hl = log.tolist()  # the one synchronisation of the traversal
        done_p2p, done_m2l, fronts = hl[0], hl[1], hl[2:]
        peak = max(fronts)
        if fronts[-1] != 0:
            raise RuntimeError("dual traversal did not terminate within 2*depth+2 steps")
        if done_p2p <= cap_p2p and done_m2l <= cap_m2l and peak <= cap_next:
            break
        cap_p2p = max(cap_p2p, int(done_p2p * 1.05) + 4096)
        cap_m2l = max(cap_m2l, int(done_m2l * 1.05) + 4096)
        cap_next = max(cap_next, int(peak * 1.05) + 4096)
    del fr
    _hint[key] = (int(done_p2p * 1.02) + 4096, int(done_m2l * 1.02) + 4096, int(peak * 1.05) + 4096)
    ncells = tree.ncells
    wsp, wsb = _lib.workspace(max(done_m2l, done_p2p, tree.n, ncells + 1), dev, stream=torch.cuda.current_stream())
    m2l_src, m2l_rows = _far_csr(m2l_t, m2l_s, done_m2l, ncells, dev, wsp, wsb, st, side, m2l_ready,
                                 nsrc=sb.ncells, sort=sort_far)
    p2p_grp, p2p_rows = _csr(p2p_t, p2p_s, done_p2p, ncells, dev, wsp, wsb, st, nsrc=sb.ncells, sort=False)
    del p2p_t, p2p_s, m2l_t, m2l_s
    return Lists(n_m2l=done_m2l, n_p2p=done_p2p, m2l_src=m2l_src, m2l_rows=m2l_rows,
                 p2p_rows=p2p_rows, peak_frontier=peak,
                 **_p2p_plan(tree, p2p_grp, p2p_rows, done_p2p, blo, bhi, wsp, wsb, st, src=src, tmask=target_mask))


def _source_cells(tree: Tree, src: Tree | None) -> tuple:
    """The source tree's cell arrays for the traversal ABI (NULLs: the
    target tree is its own source)."""
    if src is None or src is tree:
        return (None,) * 5
    P = _lib.ptr
    return P(src.d_children), P(src.d_leaf), P(src.d_ctr), P(src.d_bmax), P(src.d_rmax)


def partition_owner(tree: Tree, grain: int) -> torch.Tensor:
    """Device owner map of the mutual traversal's target partition
    (src/traversal.py:621-640): the partition root holding each cell, -1
    above the partition."""
    if grain < 1:
        raise ValueError(f"task_grain must be >= 1, got {grain}")
    cache = tree.__dict__.setdefault("_owner_cache", {})
    if grain not in cache:
        owner = torch.empty(tree.ncells, dtype=torch.int32, device=tree.device)
        P = _lib.ptr
        _lib.call("fmm_partition_owner", tree.ncells, P(tree.d_parent), P(tree.d_leaf), P(tree.d_start),
                  P(tree.d_end), int(grain), P(owner), _lib.stream_handle())
        cache.clear()
        cache[grain] = owner
    return cache[grain]


def mutual_lists(tree: Tree, mac: MacConfig, task_grain: int, body_range: tuple[int, int] | None = None,
                 m2l_ready: torch.cuda.Event | None = None, side: torch.cuda.Stream | None = None,
                 defer: bool = False, sort_far: bool = True, symmetric: bool = False,
                 symmetric_m2l: bool = False) -> Lists:
    """Mutual dual traversal (src/traversal.py:159-262 with mutual units,
    :704-791 driver) -> DIRECTED target-sorted CSR M2L/P2P lists: each
    mutual entry (a, b) contributes (a, b) and (b, a), the reference's trace
    expansion, so the lists equal the reference's trace sets and feed the
    directed executors.  The sets depend on ``task_grain`` through the
    partition: a mutual pair straddling two partition roots is demoted to
    two directed pairs.

    ``symmetric=True`` keeps the mutual P2P entries of two distinct leaves
    UNORDERED (``Lists.sym_p2p``) for the symmetric near field
    (``run_p2p_sym``, the reference's _p2p_mutual); the directed lists then
    hold the demoted pairs and the self pairs.  ``symmetric_m2l=True`` keeps
    the mutual M2L entries unordered too (``Lists.sym_m2l``, ``run_m2l_sym``,
    the reference's _m2l_mutual).  ``n_p2p`` / ``n_m2l`` and ``host_pairs``
    still describe the directed-expanded sets."""
    if symmetric:
        return _mutual_lists_sym(tree, mac, task_grain, body_range, m2l_ready, side, sort_far, symmetric_m2l)
    blo, bhi = body_range if body_range is not None else (0, tree.n)
    dev, P, st, i32 = tree.device, _lib.ptr, _lib.stream_handle(), torch.int32
    th2 = mac.theta * mac.theta
    owner = partition_owner(tree, task_grain)
    key = ("mutual", tree.ncells, tree.nleaves, mac.kind, th2, blo, bhi, task_grain)
    cap_p2p, cap_m2l, cap_next = _hint.get(key, (max(4096, tree.nleaves * 64), max(4096, tree.ncells * 32),
                                                 max(4096, tree.ncells * 16)))
    nsteps = 2 * tree.depth + 2
    log = torch.empty(nsteps + 3, dtype=torch.int64, device=dev)
    if defer and key in _hint and _sync_free():
        # capacities known from an earlier run of this shape: the traversal,
        # both CSRs and the plan chain on the device (as interaction_lists)
        pool = torch.empty(2 * cap_p2p + 2 * cap_m2l + 4 * cap_next, dtype=i32, device=dev)
        p2p_t, p2p_s, m2l_t, m2l_s, *fr = torch.split(pool, [cap_p2p, cap_p2p, cap_m2l, cap_m2l] + [cap_next] * 4)
        _lib.call("fmm_traverse_mutual", P(fr[0]), P(fr[1]), P(fr[2]), P(fr[3]), cap_next, nsteps,
                  P(tree.d_children), P(tree.d_leaf), P(tree.d_ctr), P(tree.d_bmax), P(tree.d_rmax), P(owner),
                  P(tree.d_start), P(tree.d_end), blo, bhi, mac.code, th2, P(p2p_t), P(p2p_s), cap_p2p, P(m2l_t),
                  P(m2l_s), cap_m2l, P(log), st)
        del fr
        ncells = tree.ncells
        wsp, wsb = _lib.workspace(max(cap_p2p, cap_m2l, tree.n, ncells + 1), dev,
                                  stream=torch.cuda.current_stream())
        m2l_src, m2l_rows = _far_csr(m2l_t, m2l_s, cap_m2l, ncells, dev, wsp, wsb, st, side, m2l_ready,
                                     dev_n=log[1:], sort=sort_far)
        p2p_grp, p2p_rows = _csr(p2p_t, p2p_s, cap_p2p, ncells, dev, wsp, wsb, st, dev_n=log, sort=False)
        del p2p_t, p2p_s, m2l_t, m2l_s
        return Lists(m2l_src=m2l_src, m2l_rows=m2l_rows, p2p_rows=p2p_rows,
                     _deferred=(log, (cap_p2p, cap_m2l, cap_next), key),
                     **_p2p_plan(tree, p2p_grp, p2p_rows, cap_p2p, blo, bhi, wsp, wsb, st))
    while True:
        p2p_t = torch.empty(cap_p2p, dtype=i32, device=dev)
        p2p_s = torch.empty(cap_p2p, dtype=i32, device=dev)
        m2l_t = torch.empty(cap_m2l, dtype=i32, device=dev)
        m2l_s = torch.empty(cap_m2l, dtype=i32, device=dev)
        fr = [torch.empty(cap_next, dtype=i32, device=dev) for _ in range(4)]
        _lib.call("fmm_traverse_mutual", P(fr[0]), P(fr[1]), P(fr[2]), P(fr[3]), cap_next, nsteps,
                  P(tree.d_children), P(tree.d_leaf), P(tree.d_ctr), P(tree.d_bmax), P(tree.d_rmax), P(owner),
                  P(tree.d_start), P(tree.d_end), blo, bhi, mac.code, th2, P(p2p_t), P(p2p_s), cap_p2p, P(m2l_t),
                  P(m2l_s), cap_m2l, P(log), st)
        hl = log.tolist()  # the one synchronisation of the traversal
        done_p2p, done_m2l, fronts = hl[0], hl[1], hl[2:]
        peak = max(fronts)
        if done_p2p <= cap_p2p and done_m2l <= cap_m2l and peak <= cap_next:
            if fronts[-1] != 0:
                raise RuntimeError("mutual traversal did not terminate within 2*depth+2 steps")
            break
        cap_p2p = max(cap_p2p, int(done_p2p * 1.05) + 4096)
        cap_m2l = max(cap_m2l, int(done_m2l * 1.05) + 4096)
        cap_next = max(cap_next, int(peak * 1.05) + 4096)
    del fr
    _hint[key] = (int(done_p2p * 1.02) + 4096, int(done_m2l * 1.02) + 4096, int(peak * 1.05) + 4096)
    ncells = tree.ncells
    wsp, wsb = _lib.workspace(max(done_m2l, done_p2p, tree.n, ncells + 1), dev, stream=torch.cuda.current_stream())
    m2l_src, m2l_rows = _far_csr(m2l_t, m2l_s, done_m2l, ncells, dev, wsp, wsb, st, side, m2l_ready,
                                 sort=sort_far)
    p2p_grp, p2p_rows = _csr(p2p_t, p2p_s, done_p2p, ncells, dev, wsp, wsb, st, sort=False)
    del p2p_t, p2p_s, m2l_t, m2l_s
    return Lists(n_m2l=done_m2l, n_p2p=done_p2p, m2l_src=m2l_src, m2l_rows=m2l_rows,
                 p2p_rows=p2p_rows, peak_frontier=peak,
                 **_p2p_plan(tree, p2p_grp, p2p_rows, done_p2p, blo, bhi, wsp, wsb, st))


def _mutual_lists_sym(tree: Tree, mac: MacConfig, task_grain: int, body_range, m2l_ready, side, sort_far,
                      sym_m2l: bool = False) -> Lists:
    """``mutual_lists(symmetric=True)``: one traversal writing the directed
    lists and the unordered mutual P2P (and, ``sym_m2l``, M2L) pairs; the
    counts are read once (the reaction buffers are sized from them)."""
    blo, bhi = body_range if body_range is not None else (0, tree.n)
    dev, P, st, i32 = tree.device, _lib.ptr, _lib.stream_handle(), torch.int32
    th2 = mac.theta * mac.theta
    owner = partition_owner(tree, task_grain)
    key = ("mutual-sym", tree.ncells, tree.nleaves, mac.kind, th2, blo, bhi, task_grain, sym_m2l)
    cap_p2p, cap_m2l, cap_next, cap_sym, cap_sm = _hint.get(
        key, (max(4096, tree.nleaves * 64), max(4096, tree.ncells * 32), max(4096, tree.ncells * 16),
              max(4096, tree.nleaves * 16), max(4096, tree.ncells * 16) if sym_m2l else 0))
    nsteps = 2 * tree.depth + 2
    log = torch.empty(nsteps + 3 + 2, dtype=torch.int64, device=dev)  # [traversal log | symmetric counts]
    while True:
        pool = torch.empty(2 * cap_p2p + 2 * cap_m2l + 4 * cap_next + 2 * cap_sym + 2 * cap_sm, dtype=i32, device=dev)
        p2p_t, p2p_s, m2l_t, m2l_s, sym_a, sym_b, sm_a, sm_b, *fr = torch.split(
            pool, [cap_p2p, cap_p2p, cap_m2l, cap_m2l, cap_sym, cap_sym, cap_sm, cap_sm] + [cap_next] * 4)
        _lib.call("fmm_traverse_mutual_sym", P(fr[0]), P(fr[1]), P(fr[2]), P(fr[3]), cap_next, nsteps,
                  P(tree.d_children), P(tree.d_leaf), P(tree.d_ctr), P(tree.d_bmax), P(tree.d_rmax), P(owner),
                  P(tree.d_start), P(tree.d_end), blo, bhi, mac.code, th2, P(p2p_t), P(p2p_s), cap_p2p, P(m2l_t),
                  P(m2l_s), cap_m2l, P(log), P(sym_a), P(sym_b), cap_sym, P(sm_a) if sym_m2l else None,
                  P(sm_b) if sym_m2l else None, cap_sm, P(log[nsteps + 3:]), st)
        hl = log.tolist()  # the one synchronisation of the traversal
        done_p2p, done_m2l, fronts, n_sym, n_sm = hl[0], hl[1], hl[2:nsteps + 3], hl[nsteps + 3], hl[nsteps + 4]
        peak = max(fronts)
        if (done_p2p <= cap_p2p and done_m2l <= cap_m2l and peak <= cap_next and n_sym <= cap_sym
                and n_sm <= cap_sm):
            if fronts[-1] != 0:
                raise RuntimeError("mutual traversal did not terminate within 2*depth+2 steps")
            break
        cap_p2p = max(cap_p2p, int(done_p2p * 1.05) + 4096)
        cap_m2l = max(cap_m2l, int(done_m2l * 1.05) + 4096)
        cap_next = max(cap_next, int(peak * 1.05) + 4096)
        cap_sym = max(cap_sym, int(n_sym * 1.05) + 4096)
        cap_sm = max(cap_sm, int(n_sm * 1.05) + 4096) if sym_m2l else 0
    del fr
    _hint[key] = (int(done_p2p * 1.02) + 4096, int(done_m2l * 1.02) + 4096, int(peak * 1.05) + 4096,
                  int(n_sym * 1.02) + 4096, int(n_sm * 1.02) + 4096 if sym_m2l else 0)
    ncells = tree.ncells
    wsp, wsb = _lib.workspace(max(done_m2l, done_p2p, n_sym, n_sm, tree.n, ncells + 1), dev,
                              stream=torch.cuda.current_stream())
    # (the unordered M2L pairs first: the far-field event is recorded after the directed CSR)
    sym_far = _sym_pairs(tree, sm_a, sm_b, n_sm, wsp, wsb, st, slots=False) if sym_m2l else None
    m2l_src, m2l_rows = _far_csr(m2l_t, m2l_s, done_m2l, ncells, dev, wsp, wsb, st, side, m2l_ready, sort=sort_far)
    p2p_grp, p2p_rows = _csr(p2p_t, p2p_s, done_p2p, ncells, dev, wsp, wsb, st, sort=False)
    plan = _p2p_plan(tree, p2p_grp, p2p_rows, done_p2p, blo, bhi, wsp, wsb, st)
    sym = _sym_pairs(tree, sym_a, sym_b, n_sym, wsp, wsb, st, slots=True)
    if n_sym:
        # the reference counts both directions of a symmetric body pair
        # (src/_taylor.py:439, pairs += 2): added to the plan's pair counter
        size = (tree.d_end - tree.d_start).long()
        plan["dev_stats"][0] += 2 * (size[sym_a[:n_sym].long()] * size[sym_b[:n_sym].long()]).sum()
    del p2p_t, p2p_s, m2l_t, m2l_s, sym_a, sym_b, sm_a, sm_b, pool
    # (m2l_calls counts both directions of a mutual pair, src/traversal.py:500-517)
    return Lists(n_m2l=done_m2l + 2 * n_sm, n_p2p=done_p2p + 2 * n_sym, m2l_src=m2l_src, m2l_rows=m2l_rows,
                 p2p_rows=p2p_rows, peak_frontier=peak, sym_p2p=sym, sym_m2l=sym_far, **plan)


def _sync_free() -> bool:
    """Hinted traversals skip the host wait (FMM_B200_SYNC_FREE=0 disables)."""
    return os.environ.get("FMM_B200_SYNC_FREE", "1") != "0"


def _csr(t, s, n, ncells, dev, wsp, wsb, stream, dev_n=None, nsrc=0, sort=True):
    """(sources, row offsets) of pairs (t, s) sorted by target then source
    (counting CSR: per-target counts, scatter, per-row sort).  ``n`` is the
    pair count, or with ``dev_n`` (a device counter) the buffer capacity, the
    count then read on the device (no host wait).  Sources are ids below
    ``nsrc`` (0: ``ncells``).  ``sort=False`` leaves each row's sources in
    arrival order (the P2P plan sorts its rows itself)."""
    src = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    rows = torch.empty(ncells + 1, dtype=torch.int64, device=dev)
    if dev_n is None:
        dev_n = torch.full((1,), n, dtype=torch.int64, device=dev)
    _lib.call("fmm_pairs_to_rows", _lib.ptr(t), _lib.ptr(s), _lib.ptr(dev_n), n, ncells, nsrc, int(sort),
              _lib.ptr(src), _lib.ptr(rows), wsp, wsb, stream)
    return src, rows


_sync_ring = threading.local()


def _sync_event(dev) -> torch.cuda.Event:
    """A cross-stream ordering event from a per-thread, per-device ring of
    64: a stream wait captures the event's state when it is issued, so
    re-recording it later is safe, and no CUDA event is created per call."""
    ring = _sync_ring.__dict__.setdefault(torch.device(dev).index or 0, [[], 0])
    evs, i = ring
    if len(evs) < 64:
        with torch.cuda.device(dev):
            evs.append(torch.cuda.Event())
        return evs[-1]
    ring[1] = (i + 1) % 64
    return evs[i]


def _far_csr(t, s, n, ncells, dev, wsp, wsb, st, side, ready, dev_n=None, nsrc=0, sort=True):
    """CSR of a far-field list (M2L or M2P).  Only the far field reads it, so
    with a ``side`` stream it is sorted there, off the P2P critical path,
    with its own scratch buffer; ``ready`` is recorded once it is final."""
    if side is None:
        out = _csr(t, s, n, ncells, dev, wsp, wsb, st, dev_n, nsrc, sort=sort)
        if ready is not None:
            ready.record()
        return out
    if dev_n is None:  # the count, written on this stream before the side stream waits
        dev_n = torch.full((1,), n, dtype=torch.int64, device=dev)
    traversed = _sync_event(dev)
    traversed.record()
    side.wait_event(traversed)
    swp, swb = _lib.workspace(max(n, ncells + 1, 1), dev, slot=1, stream=side)
    out = _csr(t, s, n, ncells, dev, swp, swb, side.cuda_stream, dev_n, nsrc, sort=sort)
    for a in (t, s, *out) + ((dev_n,) if dev_n is not None else ()):
        a.record_stream(side)
    if ready is not None:
        ready.record(side)
    return out


class SymPairs:
    """Unordered mutual pairs (a < b) of one kind for the symmetric
    executors: CSR by first member (``rows_a``/``src_a``, rows ascending),
    CSR by second member (``rows_b``/``src_b``) and, for P2P, the reaction
    slot offsets (``slot_off[k]`` = bodies of the second leaves before pair
    k)."""

    def __init__(self, n, rows_a, src_a, rows_b, src_b, slot_off=None):
        self.n, self.rows_a, self.src_a, self.rows_b, self.src_b = n, rows_a, src_a, rows_b, src_b
        self.slot_off = slot_off
        self.chunks = None

    def pairs(self):
        """(first, second) int64 host tensors in CSR order."""
        rows = self.rows_a.cpu()
        a = torch.repeat_interleave(torch.arange(rows.numel() - 1), rows[1:] - rows[:-1])
        return a, self.src_a[:self.n].cpu().long()


def symmetric_default() -> bool:
    """``EvalConfig.symmetric=None``: FMM_B200_SYMMETRIC=1 turns the symmetric
    executors on for mutual evaluations (default: directed executors)."""
    return os.environ.get("FMM_B200_SYMMETRIC", "0") == "1"


def _sym_pairs(tree: Tree, a, b, n: int, wsp, wsb, st, slots: bool) -> SymPairs:
    dev, ncells = tree.device, tree.ncells
    src_a, rows_a = _csr(a, b, n, ncells, dev, wsp, wsb, st, sort=True)
    src_b, rows_b = _csr(b, a, n, ncells, dev, wsp, wsb, st, sort=True)
    slot_off = None
    if slots:
        size = (tree.d_end - tree.d_start).long()
        slot_off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        if n:
            torch.cumsum(size[src_a[:n].long()], 0, out=slot_off[1:])
    return SymPairs(n, rows_a, src_a, rows_b, src_b, slot_off)


def _p2p_plan(tree: Tree, p2p_grp, p2p_rows, n_p2p: int, blo: int, bhi: int, wsp, wsb, st,
              src: Tree | None = None, tmask: torch.Tensor | None = None) -> dict:
    """P2P run plan + the reference's pair counters (no host round trip:
    runs <= pairs, and the row count stays on the device).  With a separate
    source tree the runs address its bodies at offset ``tree.n`` of the
    concatenated body arrays (``CrossBodies``)."""
    dev, P, i32, ncells = tree.device, _lib.ptr, torch.int32, tree.ncells
    leaf_rows = torch.empty(ncells, dtype=i32, device=dev)
    run_off = torch.empty(2 * ncells, dtype=torch.int64, device=dev)  # (first, end) run per row
    stats3 = torch.empty(3, dtype=torch.int64, device=dev)  # pairs, skipped, runs capacity needed (0: fit)
    dev_nrows = torch.empty(1, dtype=i32, device=dev)
    cap_runs = max(n_p2p, 1)
    runs = torch.empty((cap_runs, 4), dtype=i32, device=dev)  # row-local: runs <= pairs per row
    cross = src is not None and src is not tree
    sleaf, sstart, send = (P(src.d_leaf), P(src.d_start), P(src.d_end)) if cross else (None, None, None)
    _lib.call("fmm_p2p_plan", ncells, P(tree.d_leaf), P(tree.d_start), P(tree.d_end), blo, bhi, P(tmask), P(p2p_rows),
              P(p2p_grp), P(tree.d_x), P(tree.d_y), P(tree.d_z), P(tree.d_keys), sleaf,
              src.ncells if cross else 0, sstart, send, tree.n if cross else 0, P(leaf_rows), P(run_off), P(runs), cap_runs,
              None, None, P(dev_nrows), P(stats3), wsp, wsb, st)
    return dict(p2p_grp=p2p_grp, leaf_rows=leaf_rows, nrows=tree.nleaves, dev_nrows=dev_nrows, run_off=run_off,
                runs=runs, dev_stats=stats3[:2], dev_runs_needed=stats3[2:])


# Orders from which M2L runs offset-grouped on the FP64 tensor pipe
# (fmm_m2l_grouped: one D per (level_t, level_s, lattice offset), 8 targets
# per CTA, mma.m8n8k4.f64); it needs lattice centres (cubic, geometric) and
# one tree.  FMM_B200_M2L_GROUPED_MIN_P=99 keeps the per-pair kernels.
M2L_GROUPED_MIN_P = int(os.environ.get("FMM_B200_M2L_GROUPED_MIN_P", "8"))
M2L_GROUPED_MAX_P = 10


def m2l_grouped(tree: Tree, p: int, src: Tree | None = None) -> bool:
    """Whether ``run_m2l`` takes the offset-grouped tensor-pipe kernel."""
    cross = src is not None and src is not tree
    return (not cross and tree.shape == "cubic" and tree.center_mode == "geometric"
            and M2L_GROUPED_MIN_P <= p <= M2L_GROUPED_MAX_P)


def run_m2l(tree: Tree, lists: Lists, p: int, src: Tree | None = None) -> None:
    """M2L over the target CSR into ``tree``'s locals; the multipoles and
    centres are ``src``'s when it is a separate source tree
    (src/traversal.py:500-517 with ``MA``/``ctrB`` of the source)."""
    P = _lib.ptr
    cross = src is not None and src is not tree
    if m2l_grouped(tree, p, src):
        cap = lists.m2l_src.numel()
        need = C.c_size_t(0)
        _lib.call("fmm_m2l_grouped_bytes", p, tree.ncells, cap, C.byref(need))
        ws = torch.empty(int(need.value), dtype=torch.uint8, device=tree.device)  # on the current (M2L) stream
        _lib.call("fmm_m2l_grouped", p, tree.ncells, P(lists.m2l_rows), P(lists.m2l_src), cap, P(tree.d_level),
                  P(tree.d_key), P(tree.d_ctr), P(tree.d_root), P(tree._M), P(tree._L), P(ws), ws.numel(),
                  _lib.stream_handle())
        return
    _lib.call("fmm_m2l_csr", p, tree.ncells, P(lists.m2l_rows), P(lists.m2l_src), P(tree.d_ctr),
              P(src.d_ctr) if cross else None, P(src._M if cross else tree._M), P(tree._L), _lib.stream_handle())


# orders the symmetric M2L kernel covers (include/fmm_b200.h FMM_M2L_SYM_MAX_P)
M2L_SYM_MAX_P = 7


def m2l_symmetric(tree: Tree, p: int) -> bool:
    """Whether a symmetric mutual evaluation keeps its M2L pairs unordered:
    orders the register kernel covers, below the offset-grouped tensor
    kernel's range (that one shares a D over a whole lattice group)."""
    return p <= M2L_SYM_MAX_P and not m2l_grouped(tree, p)


def run_m2l_sym(tree: Tree, lists: Lists, p: int) -> None:
    """The symmetric M2L over ``lists.sym_m2l`` (after ``run_m2l`` on the
    same stream): every unordered cell pair gets one derivative tensor,
    contracted into both cells' locals (src/_taylor.py:191-217),
    deterministically (``fmm_m2l_sym``)."""
    sym = lists.__dict__.get("sym_m2l")
    if sym is None or sym.n == 0:
        return
    P, dev, item = _lib.ptr, tree.device, ncoef(p) * 8
    nch = max(1, -(-sym.n * item // SYM_BUFFER_BYTES))
    if nch == 1:
        cuts, bases = [0, tree.ncells], [0, sym.n]
    else:  # first-member ranges whose slots fit the buffer (one read)
        want = torch.arange(1, nch, device=dev, dtype=torch.int64) * (sym.n // nch)
        mid = torch.searchsorted(sym.rows_a, want, right=True).clamp_(1, tree.ncells) - 1
        cuts = sorted(set([0, tree.ncells] + mid.tolist()))
        bases = sym.rows_a[torch.tensor(cuts, device=dev)].tolist()
    cap = max(b1 - b0 for b0, b1 in zip(bases[:-1], bases[1:]))
    react = torch.empty(max(cap, 1) * ncoef(p), dtype=torch.float64, device=dev)
    for (a0, a1), base in zip(zip(cuts[:-1], cuts[1:]), bases[:-1]):
        _lib.call("fmm_m2l_sym", p, tree.ncells, a0, a1, P(sym.rows_a), P(sym.src_a), P(sym.rows_b), P(sym.src_b),
                  base, P(tree.d_ctr), P(tree._M), P(react), P(tree._L), _lib.stream_handle())
    for t in (react, sym.rows_a, sym.src_a, sym.rows_b, sym.src_b):
        t.record_stream(torch.cuda.current_stream())


class CrossBodies:
    """P2P body arrays of a cross-tree evaluation: the target tree's bodies
    followed by the source tree's, so one plan's runs address both
    (``_p2p_plan`` shifts source runs by ``tree.n``).  Results land in the
    target tree's accumulators."""

    def __init__(self, tree: Tree, src: Tree):
        cat = lambda a, b: torch.cat((a, b))  # noqa: E731
        self.d_x, self.d_y, self.d_z, self.d_q = (cat(getattr(tree, k), getattr(src, k))
                                                  for k in ("d_x", "d_y", "d_z", "d_q"))
        self.d_b32 = cat(tree.d_b32, src.d_b32)
        self.d_b32lo = cat(tree.d_b32lo, src.d_b32lo)
        self.fp32_exact = tree.fp32_exact and src.fp32_exact


# precision="fp32" keeps the near field in float32 only while float32
# rounding stays well under the expansion's truncation error.  The FP32
# near-field floor is ~3-6e-7 relative (mixed-sign charges, tens of
# thousands of sources per target; profiles/r01_c4_sweep.json), while the
# reference's own error scales as ~1.6e-3 * theta^p (potential, C4 grid).
# Below theta^p = FP32_GUARD_THETA_P the truncation error would drop under
# the float32 floor (the C4 corner p=10/theta<=0.4, p=8/theta=0.3), so the
# near field is evaluated in float64 there and the result stays within 2x
# the reference's error, the north-star bar for FP32 mode.
FP32_GUARD_THETA_P = 5e-4
# ... but float32 TERMS are accurate enough there: summed in float64
# ("fp32acc", FMM_PREC_FP32_ACC64) the near field's floor is ~1.1e-7
# (C4 corner, tools/nearfield_sweep.py: p=8/theta=0.3 force 3.56e-7 and
# potential 2.33e-7 against the reference's 3.38e-7 / 2.09e-7, at 32.7 ms
# a step instead of FP64's 75.5), which stays within 2x the reference's
# error while that error exceeds ~6e-8, i.e. theta^p >= FP32ACC_THETA_P.
# Below it (p=10, theta=0.3: reference 2.0e-8) the near field is float64.
FP32ACC_THETA_P = 5e-5
# listfmm ignores theta: its V-list pairs same-level cells at least one cell
# apart, an opening ratio of (2 * sqrt(3)/2 * s) / (2 s) = sqrt(3)/2
LISTFMM_THETA_EQ = 3 ** 0.5 / 2


def near_field_precision(cfg: "EvalConfig") -> str:
    """Arithmetic of the near field for ``cfg``: "fp64" / "fp32acc" for those
    precisions;
    for precision="fp32", "fp32" unless theta^p < FP32_GUARD_THETA_P, then
    "fp32acc" down to FP32ACC_THETA_P and "fp64" below (see above;
    FMM_B200_FP32_STRICT=1 disables the promotion).
    FMM_B200_NEAR_FIELD=fp32|fp32acc|fp64 forces one (measurements)."""
    force = os.environ.get("FMM_B200_NEAR_FIELD")
    if force:
        if force not in NEAR_FIELDS:
            raise ValueError(f"FMM_B200_NEAR_FIELD={force!r}: one of {NEAR_FIELDS}")
        return force
    if cfg.precision in ("fp64", "fp32acc"):
        return cfg.precision
    if os.environ.get("FMM_B200_FP32_STRICT", "0") == "1":
        return "fp32"
    theta = LISTFMM_THETA_EQ if cfg.strategy == "listfmm" else cfg.mac.theta
    tp = theta ** cfg.p
    return "fp32" if tp >= FP32_GUARD_THETA_P else ("fp32acc" if tp >= FP32ACC_THETA_P else "fp64")


def _near_field(cfg: "EvalConfig", *trees) -> str:
    """``near_field_precision`` for these body sets: "fp32acc" has no
    anchored form, so inputs float32 cannot hold take "fp64"."""
    nf = near_field_precision(cfg)
    if nf == "fp32acc" and not all(t.fp32_exact for t in trees):
        nf = "fp64"
    return nf


# near-field arithmetics: float32 pairs and sums; float32 pairs (refined
# 1/sqrt) with float64 sums (FMM_PREC_FP32_ACC64); float64
NEAR_FIELDS = ("fp32", "fp32acc", "fp64")


def _packed_f64(b) -> torch.Tensor:
    """The double4 (x, y, z, q) body copy the streamed FP64 P2P reads,
    packed once per body set (32 B per body)."""
    t = b.__dict__.get("d_b64")
    if t is None:
        t = torch.empty((b.d_x.numel(), 4), dtype=torch.float64, device=b.d_x.device)
        P = _lib.ptr
        _lib.call("fmm_pack_bodies_f64", b.d_x.numel(), P(b.d_x), P(b.d_y), P(b.d_z), P(b.d_q), P(t),
                  _lib.stream_handle())
        b.__dict__["d_b64"] = t
    return t


def run_p2p(tree: Tree, lists: Lists, precision: str, use_rsqrt: bool = False, safe: bool = False,
            flag=None, bodies: CrossBodies | None = None) -> None:
    """P2P over the plan into ``tree``'s accumulators; ``bodies`` holds the
    concatenated body arrays of a cross-tree plan (the target leaf then
    sweeps only the source runs).  ``precision`` is the near-field
    arithmetic (``near_field_precision``)."""
    P = _lib.ptr
    b = tree if bodies is None else bodies
    if precision == "fp32acc" and (safe or use_rsqrt or not b.fp32_exact):
        # no guarded / anchored / reference-rsqrt variant of the float64-summed
        # kernel: those cases take the float64 near field
        precision = "fp64"
    if precision == "fp32":
        # float32 cannot hold these float64 inputs: anchor offsets per row
        prec = _lib.PREC_FP32 if b.fp32_exact else _lib.PREC_FP32_ANCHORED
        packed, packed_lo = b.d_b32, b.d_b32lo
    elif precision == "fp32acc":
        prec, packed, packed_lo = _lib.PREC_FP32_ACC64, b.d_b32, None
    else:
        prec = _lib.PREC_FP64
        # use_rsqrt (the reference's float32 1/sqrt) keeps the SoA kernel
        packed, packed_lo = (None if use_rsqrt else _packed_f64(b)), None
    _lib.call("fmm_p2p", prec, int(safe), int(use_rsqrt), int(bodies is not None), lists.nrows,
              P(lists.dev_nrows), P(lists.leaf_rows), P(tree.d_start), P(tree.d_end), P(lists.run_off),
              P(lists.runs), P(b.d_x), P(b.d_y), P(b.d_z), P(b.d_q), P(packed), P(packed_lo), P(tree.d_phi),
              P(tree.d_fx), P(tree.d_fy), P(tree.d_fz), P(flag), _lib.stream_handle())


# reaction buffer bound of the symmetric near field (bytes; larger lists
# are swept in chunks of first leaves)
SYM_BUFFER_BYTES = int(float(os.environ.get("FMM_B200_SYM_BUFFER_MB", "4096")) * (1 << 20))


def run_p2p_sym(tree: Tree, lists: Lists, precision: str) -> None:
    """The symmetric near field over ``lists.sym_p2p`` (after ``run_p2p``,
    which STORES the directed near field): every unordered leaf pair is
    evaluated once and added to both leaves (src/_taylor.py:410-449),
    deterministically (``fmm_p2p_sym``).  ``precision`` "fp32" needs
    float32-exact inputs; "fp32acc" and inexact inputs take float64."""
    sym = lists.__dict__.get("sym_p2p")
    if sym is None or sym.n == 0:
        return
    P, dev = _lib.ptr, tree.device
    if precision == "fp32" and tree.fp32_exact:
        prec, packed, item = _lib.PREC_FP32, tree.d_b32, 16
    else:
        prec, packed, item = _lib.PREC_FP64, _packed_f64(tree), 32
    chunks = sym.chunks
    if chunks is None or chunks[0] != item or chunks[3] != SYM_BUFFER_BYTES:
        # first-leaf ranges whose reaction slots fit the buffer (one read)
        row_slot = sym.slot_off[sym.rows_a]  # slots before each first leaf's row
        total = int(row_slot[-1])
        nch = max(1, -(-total * item // SYM_BUFFER_BYTES))
        if nch == 1:
            cuts, bases = [0, tree.ncells], [0, total]
        else:
            want = torch.arange(1, nch, device=dev, dtype=torch.int64) * (total // nch)
            mid = torch.searchsorted(row_slot, want, right=True).clamp_(1, tree.ncells) - 1
            cuts = sorted(set([0, tree.ncells] + mid.tolist()))
            bases = row_slot[torch.tensor(cuts, device=dev)].tolist()
        chunks = sym.chunks = (item, cuts, bases, SYM_BUFFER_BYTES)
    _, cuts, bases, _ = chunks
    cap = max(b1 - b0 for b0, b1 in zip(bases[:-1], bases[1:]))
    react = torch.empty(max(cap, 1) * item, dtype=torch.uint8, device=dev)
    for (a0, a1), base in zip(zip(cuts[:-1], cuts[1:]), bases[:-1]):
        _lib.call("fmm_p2p_sym", prec, tree.ncells, a0, a1, P(sym.rows_a), P(sym.src_a), P(sym.rows_b),
                  P(sym.src_b), P(sym.slot_off), base, P(tree.d_start), P(tree.d_end), P(packed), P(react),
                  P(tree.d_phi), P(tree.d_fx), P(tree.d_fy), P(tree.d_fz), _lib.stream_handle())
    react.record_stream(torch.cuda.current_stream())


def count_coincident(tree: Tree, lists: Lists, bodies: CrossBodies) -> torch.Tensor:
    """Device count of the cross-tree P2P pairs at distance 0.0 (float64),
    which the reference skips and counts as ``p2p_skipped``
    (src/traversal.py:552-597)."""
    P = _lib.ptr
    n = torch.zeros(1, dtype=torch.int64, device=tree.device)
    _lib.call("fmm_p2p_coincident", lists.nrows, P(lists.dev_nrows), P(lists.leaf_rows), P(tree.d_start),
              P(tree.d_end), P(lists.run_off), P(lists.runs), P(bodies.d_x), P(bodies.d_y), P(bodies.d_z), P(n),
              _lib.stream_handle())
    return n


def treecode_lists(tree: Tree, mac: MacConfig, body_range: tuple[int, int] | None = None,
                   m2p_ready: torch.cuda.Event | None = None, side: torch.cuda.Stream | None = None,
                   src: Tree | None = None) -> Lists:
    """Treecode walk (src/traversal.py:265-313) of every target leaf against
    the source tree -> target-sorted CSR M2P and P2P lists (bit-exact sets
    with the reference's ``_collect_treecode``) + the P2P run plan.

    ``body_range=(lo, hi)`` keeps the target leaves whose bodies meet
    [lo, hi) (a multi-GPU rank's share); ``src`` is a separate source tree."""
    blo, bhi = body_range if body_range is not None else (0, tree.n)
    dev, P, st, i32 = tree.device, _lib.ptr, _lib.stream_handle(), torch.int32
    th2 = mac.theta * mac.theta
    ncells = tree.ncells
    cross = src is not None and src is not tree
    sb = src if cross else tree
    key = ("treecode", ncells, tree.nleaves, mac.kind, th2, blo, bhi, sb.ncells if cross else 0)
    cap_p2p, cap_m2p, cap_next = _hint.get(key, (max(4096, tree.nleaves * 64), max(4096, tree.nleaves * 256),
                                                 max(4096, ncells * 8)))
    nsteps = sb.depth + 2  # one source level per step
    bcells = _source_cells(tree, src)
    log = torch.empty(nsteps + 3, dtype=torch.int64, device=dev)
    wsp, wsb = _lib.workspace(max(ncells, tree.n), dev)
    while True:
        cap_front = max(cap_next, ncells)
        fr = [torch.empty(cap_front, dtype=i32, device=dev) for _ in range(4)]
        m2p_t = torch.empty(cap_m2p, dtype=i32, device=dev)
        m2p_s = torch.empty(cap_m2p, dtype=i32, device=dev)
        p2p_t = torch.empty(cap_p2p, dtype=i32, device=dev)
        p2p_s = torch.empty(cap_p2p, dtype=i32, device=dev)
        _lib.call("fmm_treecode_traverse", P(fr[0]), P(fr[1]), P(fr[2]), P(fr[3]), cap_front, nsteps, ncells,
                  P(tree.d_children), P(tree.d_leaf), P(tree.d_ctr), P(tree.d_bmax), P(tree.d_rmax), *bcells,
                  P(tree.d_start), P(tree.d_end), blo, bhi, mac.code, th2, P(m2p_t), P(m2p_s), cap_m2p, P(p2p_t),
                  P(p2p_s), cap_p2p, P(log), wsp, wsb, st)
        hl = log.tolist()  # the one synchronisation of the walk
        done_p2p, done_m2p, fronts = hl[0], hl[1], hl[2:]
        peak = max(fronts)
        if fronts[-1] != 0:
            raise RuntimeError("treecode walk did not terminate within depth+2 steps")
        if done_p2p <= cap_p2p and done_m2p <= cap_m2p and peak <= cap_front:
            break
        cap_p2p = max(cap_p2p, int(done_p2p * 1.05) + 4096)
        cap_m2p = max(cap_m2p, int(done_m2p * 1.05) + 4096)
        cap_next = max(cap_next, int(peak * 1.05) + 4096)
    del fr
    _hint[key] = (int(done_p2p * 1.02) + 4096, int(done_m2p * 1.02) + 4096, int(peak * 1.05) + 4096)
    wsp, wsb = _lib.workspace(max(done_m2p, done_p2p, tree.n, ncells + 1), dev)
    m2p_src, m2p_rows = _far_csr(m2p_t, m2p_s, done_m2p, ncells, dev, wsp, wsb, st, side, m2p_ready,
                                 nsrc=sb.ncells)
    p2p_grp, p2p_rows = _csr(p2p_t, p2p_s, done_p2p, ncells, dev, wsp, wsb, st, nsrc=sb.ncells, sort=False)
    del p2p_t, p2p_s, m2p_t, m2p_s
    return Lists(n_m2l=0, n_m2p=done_m2p, n_p2p=done_p2p, m2p_src=m2p_src, m2p_rows=m2p_rows,
                 p2p_rows=p2p_rows, peak_frontier=peak,
                 **_p2p_plan(tree, p2p_grp, p2p_rows, done_p2p, blo, bhi, wsp, wsb, st, src=src))


def listfmm_lists(tree: Tree, body_range: tuple[int, int] | None = None,
                  m2l_ready: torch.cuda.Event | None = None, side: torch.cuda.Stream | None = None,
                  sort_far: bool = True) -> Lists:
    """Level-wise V (M2L) and U (P2P) lists of the cubic tree
    (src/traversal.py:341-497; bit-exact sets with the reference's
    ``_collect_vlist`` / ``_collect_ulist``) -> target-sorted CSR + P2P plan.
    ``body_range`` keeps the targets whose bodies meet [lo, hi)."""
    blo, bhi = body_range if body_range is not None else (0, tree.n)
    dev, P, st, i32 = tree.device, _lib.ptr, _lib.stream_handle(), torch.int32
    ncells = tree.ncells
    key = ("listfmm", ncells, tree.nleaves, blo, bhi)
    cap_p2p, cap_m2l = _hint.get(key, (max(4096, tree.nleaves * 48), max(4096, ncells * 200)))
    off = (C.c_int64 * len(tree.level_off))(*tree.level_off)
    cnt = torch.empty(2, dtype=torch.int64, device=dev)
    wsp, wsb = _lib.workspace(max(ncells, tree.n), dev, stream=torch.cuda.current_stream())
    while True:
        m2l_t = torch.empty(cap_m2l, dtype=i32, device=dev)
        m2l_s = torch.empty(cap_m2l, dtype=i32, device=dev)
        p2p_t = torch.empty(cap_p2p, dtype=i32, device=dev)
        p2p_s = torch.empty(cap_p2p, dtype=i32, device=dev)
        _lib.call("fmm_listfmm_lists", ncells, tree.depth, off, P(tree.d_level), P(tree.d_key), P(tree.d_parent),
                  P(tree.d_children), P(tree.d_leaf), P(tree.d_sub_end), P(tree.d_start), P(tree.d_end),
                  blo, bhi, P(m2l_t), P(m2l_s), cap_m2l, P(p2p_t), P(p2p_s), cap_p2p,
                  P(cnt), wsp, wsb, st)
        done_p2p, done_m2l = cnt.tolist()  # the one synchronisation
        if done_p2p <= cap_p2p and done_m2l <= cap_m2l:
            break
        cap_p2p = max(cap_p2p, int(done_p2p * 1.05) + 4096)
        cap_m2l = max(cap_m2l, int(done_m2l * 1.05) + 4096)
    _hint[key] = (int(done_p2p * 1.02) + 4096, int(done_m2l * 1.02) + 4096)
    wsp, wsb = _lib.workspace(max(done_m2l, done_p2p, tree.n, ncells + 1), dev, stream=torch.cuda.current_stream())
    m2l_src, m2l_rows = _far_csr(m2l_t, m2l_s, done_m2l, ncells, dev, wsp, wsb, st, side, m2l_ready, sort=sort_far)
    p2p_grp, p2p_rows = _csr(p2p_t, p2p_s, done_p2p, ncells, dev, wsp, wsb, st, sort=False)
    del p2p_t, p2p_s, m2l_t, m2l_s
    return Lists(n_m2l=done_m2l, n_p2p=done_p2p, m2l_src=m2l_src, m2l_rows=m2l_rows,
                 p2p_rows=p2p_rows, peak_frontier=0,
                 **_p2p_plan(tree, p2p_grp, p2p_rows, done_p2p, blo, bhi, wsp, wsb, st))


def run_m2p(tree: Tree, lists: Lists, p: int, out, src: Tree | None = None, precision: str = "fp64") -> None:
    """Treecode far field into ``out`` = (phi, fx, fy, fz) (accumulated);
    the accepted cells (centres, multipoles) are ``src``'s when given.
    ``precision="fp32"`` evaluates each (body, cell) term in float32 for
    p <= 6 (float64 running sums); higher orders stay float64."""
    P = _lib.ptr
    sb = tree if src is None else src
    prec = _lib.PREC_FP32 if precision == "fp32" else _lib.PREC_FP64
    _lib.call("fmm_m2p_csr", p, prec, tree.ncells, P(lists.m2p_rows), P(lists.m2p_src), P(tree.d_start),
              P(tree.d_end), P(sb.d_ctr), P(sb._M), P(tree.d_x), P(tree.d_y), P(tree.d_z), *(P(a) for a in out),
              _lib.stream_handle())


_side = {}
last_events = None


def _side_stream(dev, which: int = 0) -> torch.cuda.Stream:
    """Persistent auxiliary streams per device: 0 = far field, 1 = P2P,
    2 = list construction, 3 = the upward pass.  Three priority levels:
    the lists (they gate P2P) highest, the far field and the upward pass
    above P2P -- their short kernels take SM slots as P2P blocks retire
    instead of queueing behind the whole P2P grid, so the far field finishes
    early (its spans are then its kernel times) -- and P2P lowest.  The far
    field sits below the lists so that the M2L row sort does not compete
    with the P2P plan (FMM_B200_FAR_PRIORITY: "mid" (default), "high", or
    "low" = P2P's)."""
    key = (torch.device(dev).index or 0, which)
    if key not in _side:
        least, greatest = torch.cuda.Stream.priority_range()
        mode = os.environ.get("FMM_B200_FAR_PRIORITY", "mid")
        if which == 2:
            prio = greatest
        elif which == 1:
            prio = least
        else:
            prio = {"high": greatest, "low": least}.get(mode, (least + greatest) // 2)
        _side[key] = torch.cuda.Stream(device=dev, priority=prio)
    return _side[key]


def _nchunks(tree: Tree) -> int:
    """Target chunks of one evaluation (FMM_B200_CHUNKS; default 1).

    Chunking bounds the list memory of one pass and lets chunk k + 1's lists
    run beside chunk k's P2P, but measured on B200 it does not pay: the P2P
    grid already saturates the SMs, so list blocks displace P2P blocks
    (C2: 14.20 ms at 1 chunk, 14.32 at 2, 14.86 at 4)."""
    env = os.environ.get("FMM_B200_CHUNKS")
    return max(1, int(env)) if env else 1


def _chunk_cuts(tree: Tree, k: int) -> list[int]:
    """Body cut points 0 = c0 < ... < ck = n on leaf boundaries (the start of
    the leaf holding body i * n / k); duplicates collapse."""
    if k <= 1:
        return [0, tree.n]
    at = torch.tensor([i * tree.n // k for i in range(1, k)], dtype=torch.int64, device=tree.device)
    inner = tree.d_start[tree.d_body_leaf[at].long()].tolist()
    cuts = [0]
    for c in inner:
        if cuts[-1] < c < tree.n:
            cuts.append(int(c))
    return cuts + [tree.n]


class ChunkedLists:
    """The lists of a chunked evaluation, viewed as one (trace, tests)."""

    def __init__(self, parts):
        self.parts = parts
        self.n_m2l = sum(x.n_m2l for x in parts)
        self.n_p2p = sum(x.n_p2p for x in parts)
        self.peak_frontier = max(x.peak_frontier for x in parts)

    def host_pairs(self, which: str):
        import numpy as np
        tt, ss = zip(*(x.host_pairs(which) for x in self.parts))
        return np.concatenate(tt), np.concatenate(ss)


class EndReadback:
    """Every small counter an evaluation needs on the host, copied in ONE
    device-to-host transfer into pinned memory that is enqueued right after
    the last kernel: the evaluation then synchronises once (on its end
    event) instead of once per counter, and the combine kernel no longer
    waits for a host round trip on the FP32 flag."""

    _pinned = threading.local()

    def __init__(self, tensors):
        self.sizes = [t.numel() for t in tensors]
        dev = torch.cat([t.reshape(-1).long() for t in tensors])
        key = (dev.device.index or 0, dev.numel())
        pool = self._pinned.__dict__.setdefault("bufs", {})
        host = pool.get(key)
        if host is None:
            host = pool[key] = torch.empty(dev.numel(), dtype=torch.int64, pin_memory=True)
        host.copy_(dev, non_blocking=True)
        self.host = host

    def parts(self):
        """The tensors' host copies (valid after the end event)."""
        out, o = [], 0
        for n in self.sizes:
            out.append(self.host[o:o + n])
            o += n
        return out


class _EventPool:
    """Timing events of one evaluation, reused across evaluations of the
    calling thread: creating ~10-20 CUDA events per step costs host time
    while the GPU waits for the first launch.  Two sets alternate, so the
    events of the previous evaluation stay intact while this one runs: a
    ``DeferredReport`` reads them late (``defer``), at the latest when its
    set comes up for reuse."""

    _pools = threading.local()

    def __init__(self, dev, deferred: bool = False):
        key = torch.device(dev).index or 0
        st = self._pools.__dict__.setdefault("by_dev", {}).setdefault(
            key, {"sets": ([], []), "gen": 0, "pending": [None, None]})
        self._st, self._k = st, st["gen"] & 1
        st["gen"] += 1
        self._settle(self._k)  # this set's last report reads its events before they are re-recorded
        if not deferred:  # an evaluator that reads its times eagerly: no report stays pending behind it
            self._settle(1 - self._k)
        self.events = st["sets"][self._k]
        self.i = 0

    def _settle(self, k: int) -> None:
        ref = self._st["pending"][k]
        self._st["pending"][k] = None
        rep = ref() if ref is not None else None
        if rep is not None:
            rep.resolve_times()

    def __call__(self) -> torch.cuda.Event:
        if self.i == len(self.events):
            self.events.append(torch.cuda.Event(enable_timing=True))
        self.i += 1
        return self.events[self.i - 1]

    def defer(self, report: "DeferredReport") -> None:
        """``report`` reads this evaluation's events later."""
        self._st["pending"][self._k] = weakref.ref(report)

    def settle_previous(self) -> None:
        """Resolve the previous evaluation's report now (called once this
        evaluation's kernels are queued: the host is about to wait anyway)."""
        self._settle(1 - self._k)


def evaluate_dual_tree(tree: Tree, cfg: EvalConfig, *, source_tree: Tree | None = None, threads: int = 1,
                       trace: bool = False, target_mask: torch.Tensor | None = None) -> EvalReport:
    """Simultaneous traversal of the tree against itself, on the GPU.

    Three streams.  The targets may be cut into Morton chunks on leaf
    boundaries (``_nchunks``, default one chunk); the main stream (a
    high-priority list stream when chunked) builds each chunk's lists
    (traversal, P2P CSR and run plan) and a P2P stream runs the chunk's near
    field as soon as its plan exists.  M2L pairs are
    emitted only by the chunk owning their target's first body, so the
    chunks partition both lists exactly.  A side stream runs the far field:
    the upward pass as soon as the tree exists, each chunk's M2L as soon as
    its M2L list is sorted, then the downward pass, into separate
    accumulators that one combine kernel adds at the end.

    With a separate ``source_tree`` (src/traversal.py:864-932) the upward
    pass runs on the source tree, the traversal pairs target cells with
    source cells, and P2P sweeps the source bodies (``CrossBodies``);
    coincident target/source bodies are skipped and counted as the
    reference does.

    ``target_mask`` (uint8 per cell, additive) evaluates only the flagged
    target cells: results are exact on the bodies of flagged leaves whose
    ancestors are all flagged (``tuner.ErrorProbe.mask``), the counters
    cover the kept rows."""
    src = tree if source_tree is None else source_tree
    cross = src is not tree
    if cfg.mutual and cross:
        raise ValueError("mutual traversal needs target and source to share one tree")
    if target_mask is not None and cfg.mutual:
        raise ValueError("a target mask needs the directed traversal (mutual=False)")
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")
    _same_device(tree, src)
    stats = KernelStats()
    dev = tree.device
    p = cfg.p
    nf = _near_field(cfg, tree, src)
    symmetric = cfg.mutual and not cfg.use_rsqrt and (
        cfg.symmetric if cfg.symmetric is not None else symmetric_default())
    with torch.cuda.device(dev):
        main = torch.cuda.current_stream(dev)
        side = _side_stream(dev)
        pst = _side_stream(dev, 1)
        ust = _side_stream(dev, 3)  # the upward pass: launched after the first lists
        E = _EventPool(dev, deferred=True)
        e0, e_alloc, e_up0, e_up1, e_down0, e_down1, e_l1, e_pend, e_end = (E() for _ in range(9))
        need_up = src._M is None or src.p != p
        nc = ncoef(p)
        # the traversal starts first (it needs no buffers); the far-field and
        # accumulator buffers are allocated on main while it runs, and the
        # other streams wait for them (e_alloc)
        e0.record(main)

        def allocate():
            # the expansions and the flag share one fill: [M (if rebuilt) | L | flag]
            nm = src.ncells * nc if need_up else 0
            nl = tree.ncells * nc
            buf = torch.zeros(nm + nl + 1, dtype=torch.float64, device=dev)
            M = buf[:nm].view(src.ncells, nc) if need_up else src._M
            L = buf[nm:nm + nl].view(tree.ncells, nc)
            flag = buf[-1:].view(torch.int32)[:1]
            far = torch.zeros((4, tree.n), dtype=torch.float64, device=dev)
            bodies = CrossBodies(tree, src) if cross else None
            e_alloc.record(main)
            for st_ in (side, pst, ust):
                st_.wait_event(e_alloc)
            return M, L, flag, far, bodies

        def launch_upward():
            # after the traversal's launches, so its host cost is off the
            # critical path; on its own stream, so it runs beside the lists
            with torch.cuda.stream(ust):
                e_up0.record(ust)
                if need_up:
                    upward_pass(src, p, stats, sync=False, M=M)  # (resets src._L)
                e_up1.record(ust)
            src._M, src.p = M, p
            _attach_locals(tree, p, L)
            side.wait_event(e_up1)

        cuts = _chunk_cuts(tree, 1 if cfg.mutual else _nchunks(tree))
        nch = len(cuts) - 1
        # the lists gate P2P, so they build on a high-priority stream: the
        # far field's M2L blocks then yield SM slots to the CSR and plan
        # kernels (C2: 13.05-13.10 ms against 13.09-13.35 on the main stream;
        # C3 and C5 unchanged).  FMM_B200_LIST_PRIORITY=0 builds them on main.
        lst = _side_stream(dev, 2) if os.environ.get("FMM_B200_LIST_PRIORITY", "1") == "1" else main
        lst.wait_event(e0)
        parts, m2l_ev, p2p_ev = [], [], []
        for k in range(nch):
            rng = (cuts[k], cuts[k + 1]) if nch > 1 else None
            ready = E()
            with torch.cuda.stream(lst):
                # the grouped M2L orders its pairs itself: its rows need no sort
                sort_far = not m2l_grouped(tree, p, src)
                if cfg.mutual:
                    lists = mutual_lists(tree, cfg.mac, cfg.task_grain, m2l_ready=ready, side=side, sort_far=sort_far,
                                         symmetric=symmetric, symmetric_m2l=symmetric and m2l_symmetric(tree, p),
                                         defer=True)
                else:
                    lists = interaction_lists(tree, cfg.mac, body_range=rng, m2l_ready=ready, side=side,
                                              m2l_owner_only=nch > 1, src=src, target_mask=target_mask,
                                              sort_far=sort_far, defer=True)
            parts.append(lists)
            if k == 0:
                M, L, flag, far, bodies = allocate()
                src._M, src.p = (M, p) if need_up else (src._M, src.p)
                _attach_locals(tree, p, L)
                launch_upward()
            with torch.cuda.stream(side):  # M2L rows of this chunk: after upward and its sorted list
                ea, eb = E(), E()
                ea.record(side)
                run_m2l(tree, lists, p, src)
                run_m2l_sym(tree, lists, p)
                eb.record(side)
                m2l_ev.append((ea, eb))
            planned = E()
            planned.record(lst)
            pst.wait_event(planned)
            with torch.cuda.stream(pst):
                ea, eb = E(), E()
                ea.record(pst)
                run_p2p(tree, lists, nf, cfg.use_rsqrt, False, flag, bodies)
                run_p2p_sym(tree, lists, nf)
                eb.record(pst)
                p2p_ev.append((ea, eb))
        e_l1.record(lst)
        main.wait_event(e_l1)
        with torch.cuda.stream(side):
            e_down0.record(side)
            downward_pass(tree, stats, sync=False, out=tuple(far))
            e_down1.record(side)
        e_pend.record(pst)
        main.wait_event(e_pend)
        # cross-tree, float64 near field: float64-coincident pairs
        coinc = [count_coincident(tree, x, bodies) for x in parts] if cross and nf == "fp64" else []
        main.wait_event(e_down1)
        P = _lib.ptr
        combine = lambda: _lib.call("fmm_combine", tree.n, *(P(a) for a in far), P(tree.d_phi),  # noqa: E731
                                    P(tree.d_fx), P(tree.d_fy), P(tree.d_fz), _lib.stream_handle())
        combine()
        rb = EndReadback([flag] + [t for x in parts for t in x.device_counters()] + coinc)
        e_end.record(main)
        E.settle_previous()  # (the previous report's event reads, while this evaluation's kernels run)
        e_end.synchronize()
        host = rb.parts()
        redo = nf in ("fp32", "fp32acc") and int(host[0][0]) != 0
        if redo:
            # two distinct bodies collided in FP32 outside a self run: redo guarded (the
            # near field is rewritten, so the far field is added again)
            for lists in parts:
                run_p2p(tree, lists, nf, cfg.use_rsqrt, True, flag, bodies)
                run_p2p_sym(tree, lists, nf)
            combine()
            if cross:  # (float64-coincident pairs are FP32 collisions too)
                coinc = [count_coincident(tree, x, bodies) for x in parts]
            e_end.record(main)
            e_end.synchronize()
        k = 1
        hparts = []
        for lists in parts:
            n = 3 if lists.__dict__.get("_deferred") is not None else 2
            hparts.append(host[k:k + n])
            k += n
        if not all([x.settle(h) for x, h in zip(parts, hparts)]):
            # a hinted list outgrew its buffer: redo with exact counts
            return evaluate_dual_tree(tree, cfg, source_tree=source_tree, threads=threads, trace=trace,
                                      target_mask=target_mask)
        pairs = skipped = 0
        for h in hparts:
            a, b = h[0].tolist()
            pairs += a
            skipped += b
        for c in (coinc if redo else host[k:]):
            k_ = int(c.item() if isinstance(c, torch.Tensor) and c.is_cuda else c[0])
            pairs -= k_
            skipped += k_
    lists = parts[0] if nch == 1 else ChunkedLists(parts)
    tree.list_cache = lists
    global last_events  # (start, P2P chunk (begin, end) events, end): tools/step_probe.py
    last_events = (e0, p2p_ev, e_end)
    stats.p2p_pairs += int(pairs)
    stats.p2p_skipped += int(skipped)
    stats.p2p_flops += 20 * int(pairs)
    stats.m2l_calls += lists.n_m2l
    tree._results_changed()
    events = None
    if trace:
        events = []
        mt, ms_ = lists.host_pairs("m2l")
        events += [("m2l", int(a), int(b)) for a, b in zip(mt, ms_)]
        pt, ps = lists.host_pairs("p2p")
        events += [("p2p", int(a), int(b)) for a, b in zip(pt, ps)]

    def times(rep):
        # phases overlap (far field on the side streams, near field on the
        # P2P stream): the report splits the wall time along the critical
        # path; the raw stream spans stay in ``spans``
        ms = lambda a, b: a.elapsed_time(b) * 1e-3  # noqa: E731
        d = rep.__dict__
        m2l_s, p2p_s = sum(ms(a, b) for a, b in m2l_ev), sum(ms(a, b) for a, b in p2p_ev)
        t_lists = ms(e0, e_l1)
        st_ = d["stats"]
        st_.add_time("list", t_lists)
        st_.add_time("m2l", m2l_s)
        st_.add_time("p2p", p2p_s)  # kernel time, all chunks
        wall = ms(e0, e_end)
        up, trav, down = critical_path(ms(e0, e_pend), ms(e0, e_up1), max(ms(e0, b) for _, b in m2l_ev), wall)
        up += _setup_gap(tree, e0)
        d.update(build_time=_build_time(tree, src), upward_time=up, traversal_time=trav, downward_time=down,
                 spans={"lists": t_lists, "upward": ms(e_up0, e_up1), "m2l": m2l_s, "p2p": p2p_s,
                        "downward": ms(e_down0, e_down1), "wall": wall})

    rep = DeferredReport(strategy="dualtree", n=tree.n, n_sources=src.n, p=p, mac_kind=cfg.mac.kind,
                         theta=cfg.mac.theta, mutual=cfg.mutual, threads=threads, task_grain=cfg.task_grain,
                         stats=stats, build_time=0.0, upward_time=0.0, traversal_time=0.0, downward_time=0.0,
                         trace=events, near_field=nf)
    rep.__dict__["_thunk"] = times
    E.defer(rep)
    return rep


def evaluate_treecode(tree: Tree, cfg: EvalConfig, *, source_tree: Tree | None = None, threads: int = 1,
                      trace: bool = False) -> EvalReport:
    """Classic one-tree-at-a-time walk; the far field lands directly on the
    bodies (src/traversal.py:1002-1046), on the GPU.

    Same two-stream layout as ``evaluate_dual_tree``: the main stream walks
    the tree and runs P2P; the side stream runs the upward pass and, once
    the M2P list is sorted, M2P into separate accumulators that one combine
    kernel adds at the end.  The walk is target-leaf driven, so
    ``cfg.mutual`` has no effect here (as in the reference).  A separate
    ``source_tree`` (src/traversal.py:1002-1046) is walked from every target
    leaf; its multipoles and bodies are the sources."""
    src = tree if source_tree is None else source_tree
    cross = src is not tree
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")
    _same_device(tree, src)
    stats = KernelStats()
    dev = tree.device
    p = cfg.p
    nf = _near_field(cfg, tree, src)
    with torch.cuda.device(dev):
        main = torch.cuda.current_stream(dev)
        side = _side_stream(dev)
        E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        e0, e_up0, e_up1, e_m0, e_m1, e_l1, e_p0, e_p1, e_end = (E() for _ in range(9))
        need_up = src._M is None or src.p != p
        M = torch.zeros((src.ncells, ncoef(p)), dtype=torch.float64, device=dev) if need_up else src._M
        far = torch.zeros((4, tree.n), dtype=torch.float64, device=dev)
        bodies = CrossBodies(tree, src) if cross else None
        e0.record(main)
        side.wait_event(e0)
        with torch.cuda.stream(side):
            e_up0.record(side)
            if need_up:
                upward_pass(src, p, stats, sync=False, M=M)  # (resets src._L)
            e_up1.record(side)
        src._M, src.p = M, p
        m2p_ready = torch.cuda.Event()
        lists = treecode_lists(tree, cfg.mac, m2p_ready=m2p_ready, side=side, src=src)
        tree.list_cache = lists
        e_l1.record(main)
        side.wait_event(m2p_ready)
        with torch.cuda.stream(side):
            e_m0.record(side)
            run_m2p(tree, lists, p, tuple(far), src, nf)
            e_m1.record(side)
        e_p0.record(main)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        run_p2p(tree, lists, nf, cfg.use_rsqrt, False, flag, bodies)
        e_p1.record(main)
        redo = nf in ("fp32", "fp32acc") and int(flag.item()) != 0
        if redo:
            run_p2p(tree, lists, nf, cfg.use_rsqrt, True, flag, bodies)
            e_p1.record(main)
        coinc = count_coincident(tree, lists, bodies) if cross and (redo or nf == "fp64") else None
        main.wait_event(e_m1)
        P = _lib.ptr
        _lib.call("fmm_combine", tree.n, *(P(a) for a in far), P(tree.d_phi), P(tree.d_fx), P(tree.d_fy),
                  P(tree.d_fz), _lib.stream_handle())
        e_end.record(main)
        e_end.synchronize()
        pairs, skipped = lists.dev_stats.tolist()
        if coinc is not None:
            k = int(coinc.item())
            pairs -= k
            skipped += k
    stats.p2p_pairs += int(pairs)
    stats.p2p_skipped += int(skipped)
    stats.p2p_flops += 20 * int(pairs)
    stats.m2p_calls += lists.n_m2p
    stats.add_time("list", e0.elapsed_time(e_l1) * 1e-3)
    stats.add_time("m2p", e_m0.elapsed_time(e_m1) * 1e-3)
    stats.add_time("p2p", e_p0.elapsed_time(e_p1) * 1e-3)
    tree._results_changed()
    events = None
    if trace:
        events = []
        mt, ms = lists.host_pairs("m2p")
        events += [("m2p", int(a), int(b)) for a, b in zip(mt, ms)]
        pt, ps = lists.host_pairs("p2p")
        events += [("p2p", int(a), int(b)) for a, b in zip(pt, ps)]
    ms = lambda a, b: a.elapsed_time(b) * 1e-3  # noqa: E731
    wall = ms(e0, e_end)
    up, trav, down = critical_path(ms(e0, e_p1), ms(e0, e_up1), ms(e0, e_m1), wall)
    up += _setup_gap(tree, e0)
    trav, down = trav + down, 0.0  # the treecode has no downward phase (src/traversal.py:1002-1046)
    spans = {"lists": ms(e0, e_l1), "upward": ms(e_up0, e_up1), "m2p": ms(e_m0, e_m1), "p2p": ms(e_p0, e_p1),
             "wall": wall}
    return EvalReport(strategy="treecode", n=tree.n, n_sources=src.n, p=p, mac_kind=cfg.mac.kind,
                      theta=cfg.mac.theta, mutual=cfg.mutual, threads=threads, task_grain=cfg.task_grain,
                      stats=stats, build_time=_build_time(tree, src), upward_time=up, traversal_time=trav,
                      downward_time=down, trace=events, spans=spans, near_field=nf)


def evaluate_list_fmm(tree: Tree, cfg: EvalConfig, *, source_tree: Tree | None = None, threads: int = 1,
                      trace: bool = False) -> EvalReport:
    """Level-wise interaction lists, adjacency-based; theta plays no role
    (src/traversal.py:1121-1189), on the GPU.

    Same two-stream layout as ``evaluate_dual_tree``: the main stream builds
    the V/U lists and runs P2P over the U list; the side stream runs the
    upward pass, M2L over the V list and the downward pass into separate
    accumulators that one combine kernel adds at the end."""
    if source_tree is not None and source_tree is not tree:
        raise ValueError("listfmm evaluates one tree onto itself")
    if tree.shape != "cubic":
        raise ValueError("listfmm requires cubic cells; rebuild the tree with shape='cubic'")
    if threads < 1:
        raise ValueError(f"threads must be >= 1, got {threads}")
    stats = KernelStats()
    dev = tree.device
    p = cfg.p
    nf = _near_field(cfg, tree)
    with torch.cuda.device(dev):
        main = torch.cuda.current_stream(dev)
        side = _side_stream(dev)
        E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        e0, e_up0, e_up1, e_m0, e_m1, e_d1, e_l1, e_p0, e_p1, e_end = (E() for _ in range(10))
        need_up = tree._M is None or tree.p != p
        nc = ncoef(p)
        M = torch.zeros((tree.ncells, nc), dtype=torch.float64, device=dev) if need_up else tree._M
        L = torch.zeros((tree.ncells, nc), dtype=torch.float64, device=dev)
        far = torch.zeros((4, tree.n), dtype=torch.float64, device=dev)
        e0.record(main)
        side.wait_event(e0)
        with torch.cuda.stream(side):
            e_up0.record(side)
            if need_up:
                upward_pass(tree, p, stats, sync=False, M=M)  # (resets tree._L)
            e_up1.record(side)
        tree._M, tree.p, tree._L = M, p, L
        m2l_ready = torch.cuda.Event()
        lists = listfmm_lists(tree, m2l_ready=m2l_ready, side=side, sort_far=not m2l_grouped(tree, p))
        tree.list_cache = lists
        e_l1.record(main)
        side.wait_event(m2l_ready)
        with torch.cuda.stream(side):
            e_m0.record(side)
            run_m2l(tree, lists, p)
            e_m1.record(side)
            downward_pass(tree, stats, sync=False, out=tuple(far))
            e_d1.record(side)
        e_p0.record(main)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        run_p2p(tree, lists, nf, cfg.use_rsqrt, False, flag)
        e_p1.record(main)
        if nf in ("fp32", "fp32acc") and int(flag.item()) != 0:
            run_p2p(tree, lists, nf, cfg.use_rsqrt, True, flag)
            e_p1.record(main)
        main.wait_event(e_d1)
        P = _lib.ptr
        _lib.call("fmm_combine", tree.n, *(P(a) for a in far), P(tree.d_phi), P(tree.d_fx), P(tree.d_fy),
                  P(tree.d_fz), _lib.stream_handle())
        e_end.record(main)
        e_end.synchronize()
        pairs, skipped = lists.dev_stats.tolist()
    stats.p2p_pairs += int(pairs)
    stats.p2p_skipped += int(skipped)
    stats.p2p_flops += 20 * int(pairs)
    stats.m2l_calls += lists.n_m2l
    stats.add_time("list", e0.elapsed_time(e_l1) * 1e-3)
    stats.add_time("m2l", e_m0.elapsed_time(e_m1) * 1e-3)
    stats.add_time("p2p", e_p0.elapsed_time(e_p1) * 1e-3)
    tree._results_changed()
    events = None
    if trace:
        events = []
        mt, ms = lists.host_pairs("m2l")
        events += [("m2l", int(a), int(b)) for a, b in zip(mt, ms)]
        pt, ps = lists.host_pairs("p2p")
        events += [("p2p", int(a), int(b)) for a, b in zip(pt, ps)]
    ms = lambda a, b: a.elapsed_time(b) * 1e-3  # noqa: E731
    wall = ms(e0, e_end)
    up, trav, down = critical_path(ms(e0, e_p1), ms(e0, e_up1), ms(e0, e_m1), wall)
    up += _setup_gap(tree, e0)
    spans = {"lists": ms(e0, e_l1), "upward": ms(e_up0, e_up1), "m2l": ms(e_m0, e_m1), "p2p": ms(e_p0, e_p1),
             "downward": ms(e_m1, e_d1), "wall": wall}
    return EvalReport(strategy="listfmm", n=tree.n, n_sources=tree.n, p=p, mac_kind=cfg.mac.kind,
                      theta=cfg.mac.theta, mutual=cfg.mutual, threads=threads, task_grain=cfg.task_grain,
                      stats=stats, build_time=tree.build_time, upward_time=up, traversal_time=trav,
                      downward_time=down, trace=events, spans=spans, near_field=nf)


def _same_device(tree: Tree, src: Tree) -> None:
    if src is not tree and torch.device(src.device) != torch.device(tree.device):
        raise ValueError(f"source tree on {src.device}, target tree on {tree.device}")


def _build_time(tree: Tree, src: Tree) -> float:
    """Both trees' build times (src/traversal.py:922)."""
    return tree.build_time + (src.build_time if src is not tree else 0.0)


def _attach_locals(tree: Tree, p: int, L: torch.Tensor) -> None:
    """Fresh order-p locals on the target tree (src/traversal.py:614-618); its
    multipoles stay valid only if they are of order p."""
    if tree._M is not None and tree.p != p:
        tree._M = None
    tree.p, tree._L = p, L


def evaluate_on_tree(tree: Tree, cfg: EvalConfig, *, source_tree: Tree | None = None, threads: int = 1,
                     trace: bool = False) -> EvalReport:
    """Run ``cfg.strategy`` on the tree; results land in ``tree.bodies``."""
    fn = {"treecode": evaluate_treecode, "listfmm": evaluate_list_fmm, "dualtree": evaluate_dual_tree}
    return fn[cfg.strategy](tree, cfg, source_tree=source_tree, threads=threads, trace=trace)
