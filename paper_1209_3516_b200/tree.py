"""Adaptive octree on the B200 and the vertical passes.

Drop-in for the reference's ``build_tree`` / ``Tree`` / ``upward_pass`` /
``downward_pass`` (src/tree.py:275-488).  All state lives on the device:

* bodies in Morton order as float64 SoA (``x, y, z, q``) plus a float4
  ``(x, y, z, q)`` FP32 copy feeding the FP32 P2P kernel, and the float64
  accumulators ``phi, fx, fy, fz``;
* cells in the reference's pre-order numbering as SoA arrays (int32 ids,
  uint64 keys, float64 geometry), plus ``cells_by_level`` (pre-order ids
  grouped by level) for the level-synchronous passes.

The reference's attribute names (``cell_children``, ``cell_start`` ...,
``bodies``, ``permutation``, ``multipole``, ``local``) are host NumPy views
materialised on first access, with the reference's dtypes (int64 indices,
uint64 keys, float64 geometry, bool leaf flags).

Build (csrc/tree_build.cu): ingest + bounds -> depth-21 Morton keys ->
stable radix sort -> permute -> single-pass carve (cells numbered in
pre-order by one scan) -> geometry (cubic or rect boxes, geometric or
charge-weighted centers).  Bit-exact with src/tree.py:370-454 (keys,
permutation and every cell array; tests/test_gpu_parity.py).
"""

from __future__ import annotations

import ctypes as C
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _lib
from .geometry import MAX_LEVEL, Aabb, ParticleSet
from .kernels import TMAX, KernelStats, ncoef

SHAPES = ("cubic", "rect")
CENTER_MODES = ("geometric", "com")

__all__ = ["Tree", "build_tree", "upward_pass", "downward_pass", "check_invariants"]


# snapshots of host inputs run here, overlapping the GPU work (numpy copies
# release the GIL)
_snap = ThreadPoolExecutor(max_workers=1, thread_name_prefix="fmm-snapshot")


def _u64_np(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


class Tree:
    """Device-resident adaptive octree with the reference's ``Tree`` surface."""

    def __init__(self, **kw):
        self.__dict__.update(kw)
        self._host = {}
        self._bodies_host = None
        self._M = None
        self._L = None
        self.p = None
        self.upward_time = 0.0
        self.list_cache = None  # interaction lists of the last traversal (csr)

    # ---- sizes ---------------------------------------------------------
    @property
    def fp32_exact(self) -> bool:
        """Every float64 input is exactly representable in float32 (read in
        the build's one host transfer; the device flag otherwise)."""
        v = self.__dict__.get("_fp32_exact")
        if v is None:
            v = int(self.d_inexact.item()) == 0
            self._fp32_exact = v
        return v

    @property
    def ncells(self) -> int:
        return int(self._ncells)

    @property
    def nleaves(self) -> int:
        return int(self._nleaves)

    @property
    def depth(self) -> int:
        return len(self.level_off) - 2

    # ---- host views with the reference's names and dtypes ----------------
    def _h(self, name, fn):
        v = self._host.get(name)
        if v is None:
            v = fn()
            self._host[name] = v
        return v

    @property
    def cell_children(self):
        return self._h("children", lambda: self.d_children.cpu().numpy().astype(np.int64))

    @property
    def cell_parent(self):
        return self._h("parent", lambda: self.d_parent.cpu().numpy().astype(np.int64))

    @property
    def cell_level(self):
        return self._h("level", lambda: self.d_level.cpu().numpy().astype(np.int64))

    @property
    def cell_key(self):
        return self._h("key", lambda: _u64_np(self.d_key))

    @property
    def cell_start(self):
        return self._h("start", lambda: self.d_start.cpu().numpy().astype(np.int64))

    @property
    def cell_end(self):
        return self._h("end", lambda: self.d_end.cpu().numpy().astype(np.int64))

    @property
    def cell_sub_end(self):
        return self._h("sub_end", lambda: self.d_sub_end.cpu().numpy().astype(np.int64))

    @property
    def cell_lo(self):
        return self._h("lo", lambda: self.d_lo.cpu().numpy())

    @property
    def cell_hi(self):
        return self._h("hi", lambda: self.d_hi.cpu().numpy())

    @property
    def cell_center(self):
        return self._h("center", lambda: self.d_ctr.cpu().numpy())

    @property
    def cell_bmax(self):
        return self._h("bmax", lambda: self.d_bmax.cpu().numpy())

    @property
    def cell_rmax(self):
        return self._h("rmax", lambda: self.d_rmax.cpu().numpy())

    @property
    def cell_leaf(self):
        return self._h("leaf", lambda: self.d_leaf.cpu().numpy().astype(bool))

    @property
    def permutation(self):
        return self._h("perm", lambda: self.d_perm.cpu().numpy().astype(np.int64))

    @property
    def keys(self):
        """Sorted depth-21 Morton keys of the bodies (uint64)."""
        return self._h("keys", lambda: _u64_np(self.d_keys))

    @property
    def root_box(self) -> Aabb:
        def mk():
            r = self.d_root.cpu().numpy()
            return Aabb(r[0:3], r[0:3] + r[3])
        return self._h("root_box", mk)

    # ---- bodies and results ---------------------------------------------
    @property
    def bodies(self) -> ParticleSet:
        """Host float64 view of the Morton-ordered bodies and accumulators."""
        if self._bodies_host is None:
            self._bodies_host = ParticleSet(*(a.cpu().numpy() for a in (
                self.d_x, self.d_y, self.d_z, self.d_q, self.d_phi, self.d_fx, self.d_fy, self.d_fz)))
        return self._bodies_host

    def device_bodies(self) -> ParticleSet:
        """The same bodies as device tensors (no copy)."""
        return ParticleSet(self.d_x, self.d_y, self.d_z, self.d_q, self.d_phi, self.d_fx, self.d_fy, self.d_fz)

    def _results_changed(self) -> None:
        self._bodies_host = None

    def reset_accumulators(self) -> None:
        for a in (self.d_phi, self.d_fx, self.d_fy, self.d_fz):
            a.zero_()
        self._bodies_host = None
        self._L = None

    def results_in_input_order(self) -> ParticleSet:
        """Copy of the bodies (with accumulators) in the caller's ordering
        (src/tree.py:344-348).  The permutation is undone on the device and
        only the accumulators travel back (through pinned buffers); positions
        and charges come from the caller's own arrays when they were given
        on the host."""
        if self._bodies_host is not None:  # host-side edits win (reference semantics)
            b = self._bodies_host
            inv = np.empty(self.n, dtype=np.int64)
            inv[self.permutation] = np.arange(self.n)
            return b.permuted(inv)
        acc = self.device_results_in_input_order()
        host = []
        for a in acc:
            h = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
            h.copy_(a, non_blocking=True)
            host.append(h)
        if self._input_snapshot is not None:
            # the caller's arrays as of build time (the reference's tree holds
            # its own copy of the bodies), in their stored precision (a
            # float32 cloud stays float32 and is upcast lazily on access);
            # copied on a worker thread while the GPU worked
            src = self._input_snapshot.result()
        else:
            src = None
        torch.cuda.current_stream(self.device).synchronize()
        if src is None:
            perm = self.d_perm.long()
            src = []
            for a in (self.d_x, self.d_y, self.d_z, self.d_q):
                o = torch.empty_like(a)
                o[perm] = a
                src.append(o.cpu().numpy())
        return ParticleSet(*src, *(h.numpy() for h in host))

    def device_results_in_input_order(self):
        """(phi, fx, fy, fz) on the device, in the caller's ordering."""
        out = [torch.empty_like(self.d_phi) for _ in range(4)]
        with torch.cuda.device(self.device):
            P = _lib.ptr
            _lib.call("fmm_unpermute", P(self.d_perm), self.n, P(self.d_phi), P(self.d_fx), P(self.d_fy),
                      P(self.d_fz), *(P(o) for o in out), _lib.stream_handle())
        return tuple(out)

    # ---- expansions --------------------------------------------------------
    @property
    def multipole(self):
        return None if self._M is None else self._M.cpu().numpy()

    @multipole.setter
    def multipole(self, v):
        self._M = None if v is None else torch.as_tensor(np.asarray(v, np.float64), device=self.device)

    @property
    def local(self):
        return None if self._L is None else self._L.cpu().numpy()

    @local.setter
    def local(self, v):
        self._L = None if v is None else torch.as_tensor(np.asarray(v, np.float64), device=self.device)

    # ---- misc ---------------------------------------------------------------
    def leaves(self) -> np.ndarray:
        return np.flatnonzero(self.cell_leaf)

    def body_count(self, index: int) -> int:
        return int(self.cell_end[index] - self.cell_start[index])

    def stats(self) -> dict:
        leaf = self.cell_leaf
        leaf_sizes = (self.cell_end - self.cell_start)[leaf]
        per_level = np.bincount(self.cell_level, minlength=self.depth + 1)
        return {
            "n": self.n, "ncells": self.ncells, "nleaves": self.nleaves, "depth": self.depth,
            "ncrit": self.ncrit, "shape": self.shape, "center_mode": self.center_mode,
            "cells_per_level": per_level.tolist(),
            "leaf_occupancy": {"min": int(leaf_sizes.min()), "max": int(leaf_sizes.max()),
                               "mean": float(leaf_sizes.mean())},
        }

    def level_off_c(self):
        arr = (C.c_int32 * len(self.level_off))(*self.level_off)
        return arr


def _to_device(a: np.ndarray, dev):
    """Host array -> device.  Pageable memory goes through a pinned staging
    buffer (torch's caching host allocator reuses it across calls); an array
    that already lives in page-locked memory (e.g. the NumPy view of a
    ``pin_memory=True`` tensor) is copied from where it is -- the build
    synchronises with its stream before it returns, so the caller may reuse
    the array afterwards."""
    h = torch.from_numpy(np.ascontiguousarray(a))
    if h.is_pinned():
        return h.to(dev, non_blocking=True)
    pinned = torch.empty(h.shape, dtype=h.dtype, pin_memory=True)
    pinned.copy_(h)
    return pinned.to(dev, non_blocking=True)


def build_tree(ps: ParticleSet, ncrit: int = 30, shape: str = "cubic", center_mode: str = "geometric",
               allow_oversized_leaves: bool = False, *, device=None) -> Tree:
    """Build the adaptive octree for ``ps`` on the GPU (src/tree.py:370-454).

    Same validation and errors as the reference, all four geometry modes
    (``shape`` "cubic"/"rect", ``center_mode`` "geometric"/"com",
    src/tree.py:80-160) bit-exact.
    """
    t0 = time.perf_counter()
    if shape not in SHAPES:
        raise ValueError(f"unknown cell shape {shape!r}: expected one of {SHAPES}")
    if center_mode not in CENTER_MODES:
        raise ValueError(f"unknown center mode {center_mode!r}: expected one of {CENTER_MODES}")
    if ncrit < 1:
        raise ValueError(f"ncrit must be >= 1, got {ncrit}")
    if ps.n == 0:
        raise ValueError("empty particle set")
    _lib.require_cuda()
    if device is None:
        dev = ps.x.device if ps.on_device else torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device(device)
    n = ps.n
    with torch.cuda.device(dev):
        ev_start = _build_event(dev)  # the build's span on the device timeline
        ev_start.record()
        st = _lib.stream_handle()
        f64, i32 = torch.float64, torch.int32
        if ps.on_device:
            src = tuple(a.to(dev) for a in (ps.x, ps.y, ps.z, ps.q))
        else:
            src = tuple(_to_device(a, dev) for a in ps.host_inputs())
        # the tree's own copy of the caller's arrays (the reference's tree
        # holds one): taken on a worker thread while the GPU builds (after
        # the staging copies above, which want the memory bandwidth)
        snapshot = None if ps.on_device else _snap.submit(lambda a=ps.host_inputs(): [np.array(v) for v in a])
        dcode = _lib.DTYPE_F64 if src[0].dtype == torch.float64 else _lib.DTYPE_F32
        x64 = torch.empty(n, dtype=f64, device=dev)
        y64, z64, q64 = torch.empty_like(x64), torch.empty_like(x64), torch.empty_like(x64)
        root = torch.empty(8, dtype=f64, device=dev)
        wsp, wsb = _lib.workspace(n, dev)
        P = _lib.ptr
        _lib.call("fmm_ingest_bounds", *(P(a) for a in src), dcode, n, P(x64), P(y64), P(z64), P(q64),
                  P(root), wsp, wsb, st)
        keys = torch.empty(n, dtype=torch.int64, device=dev)
        iota = torch.empty(n, dtype=i32, device=dev)
        _lib.call("fmm_morton_keys", P(x64), P(y64), P(z64), n, P(root), P(keys), P(iota), st)
        skeys = torch.empty_like(keys)
        perm = torch.empty_like(iota)
        _lib.call("fmm_sort_pairs_u64", P(keys), P(iota), P(skeys), P(perm), n, 63, wsp, wsb, st)
        xs, ys, zs, qs = (torch.empty_like(x64) for _ in range(4))
        b32 = torch.empty((n, 4), dtype=torch.float32, device=dev)
        b32lo = torch.empty((n, 4), dtype=torch.float32, device=dev)
        inexact = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("fmm_permute_bodies", P(perm), P(x64), P(y64), P(z64), P(q64), n, P(xs), P(ys), P(zs),
                  P(qs), P(b32), P(b32lo), P(inexact), st)
        del x64, y64, z64, q64, keys, iota
        tree = _carve_tree(dev, st, wsp, wsb, n, ncrit, shape, center_mode, allow_oversized_leaves, skeys, perm, root,
                           (xs, ys, zs, qs, b32, b32lo), inexact)
    tree._input_snapshot = snapshot
    tree.build_time = time.perf_counter() - t0
    with torch.cuda.device(dev):  # the evaluation bills the host gap after the build to its first phase
        tree._ev_built = _build_event(dev)
        tree._ev_built.record()
    tree._ev_build_start = ev_start
    return tree


_cell_hint = {}  # (n, ncrit, allow, device) -> largest cell count built

_build_ring = threading.local()


def _build_event(dev) -> torch.cuda.Event:
    """A timing event for a build's start/end marks, from a per-thread ring
    of 128 (creating CUDA events costs host time while the GPU waits; a mark
    is read by the tree's first evaluation, long before the ring wraps)."""
    ring = _build_ring.__dict__.setdefault("ev", {}).setdefault(torch.device(dev).index or 0, [[], 0])
    evs, i = ring
    if len(evs) < 128:
        with torch.cuda.device(dev):
            evs.append(torch.cuda.Event(enable_timing=True))
        ring[1] = len(evs) % 128
        return evs[-1]
    ring[1] = (i + 1) % 128
    return evs[i]


def _cell_arrays(cap: int, dev) -> dict:
    """Every per-cell array of a tree, ``cap`` rows each."""
    i32, f64 = torch.int32, torch.float64
    e = lambda *shape, dtype=i32: torch.empty(shape, dtype=dtype, device=dev)  # noqa: E731
    return dict(children=e(cap, 8), parent=e(cap), level=e(cap, dtype=torch.int8), key=e(cap, dtype=torch.int64),
                start=e(cap), end=e(cap), sub_end=e(cap), leaf=e(cap, dtype=torch.uint8), by_level=e(cap),
                lo=e(cap, 3, dtype=f64), hi=e(cap, 3, dtype=f64), ctr=e(cap, 3, dtype=f64), bmax=e(cap, dtype=f64),
                rmax=e(cap, dtype=f64))


def _carve_tree(dev, st, wsp, wsb, n: int, ncrit: int, shape: str, center_mode: str, allow_oversized_leaves: bool,
                skeys, perm, root, bodies, inexact) -> Tree:
    """Cells from the sorted keys (single-pass carve: per-body leaf level,
    cells numbered in pre-order by one scan, csrc/tree_build.cu; one host
    synchronisation) and their geometry, around Morton-ordered ``bodies`` =
    (xs, ys, zs, qs, b32, b32lo).  Shared by ``build_tree`` and the sharded
    multi-GPU build (``sharded.build_tree_sharded``)."""
    P = _lib.ptr
    f64, i32 = torch.float64, torch.int32
    xs, ys, zs, qs, b32, b32lo = bodies
    cbase = torch.empty(n, dtype=i32, device=dev)
    leaf_level = torch.empty(n, dtype=torch.int8, device=dev)
    body_leaf = torch.empty(n, dtype=i32, device=dev)
    # the cell arrays are allocated BEFORE the carve's one synchronisation
    # when an earlier build of this size left a capacity (the host would
    # otherwise allocate them while the GPU idles after the sync), and
    # sliced to the exact count after it
    hint_key = (n, int(ncrit), bool(allow_oversized_leaves), dev)
    cap = _cell_hint.get(hint_key, 0)
    pre = _cell_arrays(cap, dev) if cap else None
    hist = (C.c_int32 * 23)()
    nc_host = C.c_int32(0)
    inexact_host = C.c_int32(0)  # read with the counts: no separate sync later
    _lib.call("fmm_carve_count", P(skeys), n, int(ncrit), int(bool(allow_oversized_leaves)), P(cbase),
              P(leaf_level), hist, C.byref(nc_host), P(inexact), C.byref(inexact_host), wsp, wsb, st)
    ncells = int(nc_host.value)
    nleaves = int(hist[22])
    depth = max(L for L in range(22) if hist[L] > 0)
    off = [0]
    for L in range(22):
        off.append(off[-1] + int(hist[L]))
    level_off = off[:depth + 2]
    off23 = (C.c_int32 * 23)(*off[:23])
    if pre is None or ncells > cap:
        pre = _cell_arrays(ncells, dev)
    _cell_hint[hint_key] = max(cap, ncells)
    cc = {k: v[:ncells] for k, v in pre.items()}
    cells_by_level = cc.pop("by_level")
    _lib.call("fmm_carve_emit", P(skeys), n, P(cbase), P(leaf_level), ncells, off23, P(cc["children"]),
              P(cc["parent"]), P(cc["level"]), P(cc["key"]), P(cc["start"]), P(cc["end"]), P(cc["sub_end"]),
              P(cc["leaf"]), P(cells_by_level), P(body_leaf), wsp, wsb, st)
    del cbase, leaf_level
    lo, hi, ctr, bmax, rmax = (cc.pop(k) for k in ("lo", "hi", "ctr", "bmax", "rmax"))
    _lib.call("fmm_cell_geometry", ncells, P(cc["level"]), P(cc["key"]), P(cc["start"]), P(cc["end"]),
              P(xs), P(ys), P(zs), P(qs), int(shape == "rect"), int(center_mode == "com"), P(root), P(lo),
              P(hi), P(ctr), P(bmax), P(rmax), wsp, wsb, st)
    zeros = torch.zeros((4, n), dtype=f64, device=dev).unbind(0)  # one fill
    tree = Tree(
        device=dev, n=n, ncrit=ncrit, shape=shape, center_mode=center_mode,
        allow_oversized_leaves=bool(allow_oversized_leaves), _ncells=ncells, _nleaves=nleaves,
        level_off=level_off, d_root=root, d_keys=skeys, d_perm=perm,
        d_x=xs, d_y=ys, d_z=zs, d_q=qs, d_b32=b32, d_b32lo=b32lo, d_inexact=inexact,
        d_phi=zeros[0], d_fx=zeros[1], d_fy=zeros[2], d_fz=zeros[3],
        d_children=cc["children"], d_parent=cc["parent"], d_level=cc["level"], d_key=cc["key"],
        d_start=cc["start"], d_end=cc["end"], d_sub_end=cc["sub_end"], d_leaf=cc["leaf"],
        d_body_leaf=body_leaf, d_cells_by_level=cells_by_level,
        d_lo=lo, d_hi=hi, d_ctr=ctr, d_bmax=bmax, d_rmax=rmax,
    )
    tree._fp32_exact = int(inexact_host.value) == 0
    return tree


def upward_pass(tree: Tree, p: int, stats: KernelStats | None = None, *, sync: bool = True,
                M: torch.Tensor | None = None) -> None:
    """P2M at the leaves, M2M up to the root; attaches ``tree.multipole``
    (src/tree.py:457-472).  ``M`` (zeroed, [ncells, ncoef(p)]) may be
    preallocated by a caller that runs the pass on a side stream."""
    if not 1 <= p <= TMAX:
        raise ValueError(f"expansion order {p} outside supported range 1..{TMAX}")
    t0 = time.perf_counter()
    dev = tree.device
    with torch.cuda.device(dev):
        if M is None:
            M = torch.zeros((tree.ncells, ncoef(p)), dtype=torch.float64, device=dev)
        P = _lib.ptr
        _lib.call("fmm_upward", p, tree.ncells, P(tree.d_children), P(tree.d_start), P(tree.d_end),
                  P(tree.d_leaf), P(tree.d_ctr), P(tree.d_x), P(tree.d_y), P(tree.d_z), P(tree.d_q),
                  P(tree.d_cells_by_level), tree.level_off_c(), len(tree.level_off) - 1, P(M),
                  _lib.stream_handle())
        if sync:
            torch.cuda.current_stream(dev).synchronize()
    tree._M = M
    tree.p = p
    tree._L = None
    tree.upward_time = time.perf_counter() - t0
    if stats is not None:
        stats.p2m_calls += tree.nleaves
        stats.m2m_calls += tree.ncells - 1


def downward_pass(tree: Tree, stats: KernelStats | None = None, *, sync: bool = True,
                  body_range: tuple[int, int] | None = None, out=None) -> None:
    """L2L down the tree, L2P into the leaf bodies (src/tree.py:475-488).

    Requires local expansions populated by a traversal (``tree.local``).
    ``body_range=(lo, hi)`` restricts L2P to those bodies (multi-GPU);
    ``out`` = (phi, fx, fy, fz) accumulates elsewhere than the tree's own
    accumulators (the overlapped evaluation combines them afterwards)."""
    blo, bhi = body_range if body_range is not None else (0, tree.n)
    acc = out if out is not None else (tree.d_phi, tree.d_fx, tree.d_fy, tree.d_fz)
    if tree._L is None or tree.p is None:
        raise ValueError("local expansions not populated; run a traversal first")
    dev = tree.device
    with torch.cuda.device(dev):
        P = _lib.ptr
        _lib.call("fmm_downward", tree.p, tree.ncells, P(tree.d_parent), P(tree.d_leaf), P(tree.d_ctr),
                  P(tree.d_cells_by_level), tree.level_off_c(), len(tree.level_off) - 1, blo, bhi,
                  P(tree.d_body_leaf), P(tree.d_x), P(tree.d_y), P(tree.d_z), P(tree._L), *(P(a) for a in acc),
                  _lib.stream_handle())
        if sync:
            torch.cuda.current_stream(dev).synchronize()
    tree._results_changed()
    if stats is not None:
        stats.l2l_calls += tree.ncells - 1
        stats.l2p_calls += tree.nleaves


def check_invariants(tree: Tree) -> None:
    """Raise ValueError on any violated structural invariant (src/tree.py:491-525)."""
    b = tree.bodies
    start, end, ch, par = tree.cell_start, tree.cell_end, tree.cell_children, tree.cell_parent
    if start[0] != 0 or end[0] != tree.n:
        raise ValueError("root does not span all bodies")
    lo, hi, ctr, bmax, lvl, leaf = (tree.cell_lo, tree.cell_hi, tree.cell_center, tree.cell_bmax,
                                    tree.cell_level, tree.cell_leaf)
    eps = 1e-12 * max(1.0, float(tree.root_box.extent.max()))
    for c in range(tree.ncells):
        s, e = start[c], end[c]
        if e <= s:
            raise ValueError(f"cell {c} is empty")
        if lvl[c] > MAX_LEVEL:
            raise ValueError(f"cell {c} deeper than {MAX_LEVEL}")
        kids = ch[c][ch[c] >= 0]
        if leaf[c] != (kids.size == 0):
            raise ValueError(f"cell {c} leaf flag inconsistent")
        if kids.size:
            pos = s
            for k in kids:
                if start[k] != pos:
                    raise ValueError(f"children of cell {c} do not partition its range")
                pos = end[k]
                if par[k] != c:
                    raise ValueError(f"cell {k} has wrong parent")
            if pos != e:
                raise ValueError(f"children of cell {c} do not cover its range")
        for arr, d in ((b.x, 0), (b.y, 1), (b.z, 2)):
            seg = arr[s:e]
            if seg.min() < lo[c, d] - eps or seg.max() > hi[c, d] + eps:
                raise ValueError(f"body outside bounds of cell {c}")
        dd = np.sqrt((b.x[s:e] - ctr[c, 0]) ** 2 + (b.y[s:e] - ctr[c, 1]) ** 2 + (b.z[s:e] - ctr[c, 2]) ** 2)
        if dd.max() > bmax[c] + 1e-12:
            raise ValueError(f"bmax of cell {c} underestimates body distance")
