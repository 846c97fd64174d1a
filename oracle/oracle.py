"""ctypes front end of the C oracle (fmm_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module; the product package never does.  Every wrapper names the reference
function it restates (src/ = /root/reference/pkg/src/fmmkit/).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

MAX_LEVEL = 21

_lib = None


def build() -> str:
    """Compile liboracle.so in place (gcc; see oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


_P = C.c_void_p
_I = C.c_int64
_D = C.c_double


def _declare(L):
    L.orc_ncoef.argtypes = [C.c_int]
    L.orc_ncoef.restype = C.c_int
    L.orc_encode_points.argtypes = [_I, _P, _P, _P, _D, _D, _D, _D, _P]
    L.orc_argsort_stable.argtypes = [_I, _P, _P]
    L.orc_build_cells.argtypes = [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P]
    L.orc_build_cells.restype = _I
    L.orc_fill_geometry.argtypes = [_I, _P, _P, _P, _P, _P, _P, _P, _P, _D, _D, _D, _D, C.c_int, C.c_int, _P, _P, _P,
                                    _P, _P]
    L.orc_upward.argtypes = [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int, _P]
    L.orc_downward.argtypes = [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int, _P]
    L.orc_collect.argtypes = [_I, _P, _P, _P, _P, _P, _D, _I, _I, _I, _P, _P, _I, _P, _P, _P]
    L.orc_exec_m2l.argtypes = [_I, _P, _P, _P, _P, _P, C.c_int]
    L.orc_collect2.argtypes = [_P] * 10 + [_D, _I, _I, _I, _P, _P, _I, _P, _P, _P]
    L.orc_collect_treecode2.argtypes = [_I, _P, _P, _P, _P, _P, _P, _P, _D, _I, _P, _P, _I, _P, _P, _P]
    L.orc_exec_m2l2.argtypes = [_I, _P, _P, _P, _P, _P, _P, C.c_int]
    L.orc_exec_p2p_cross.argtypes = [_I] + [_P] * 17 + [C.c_int, _P]
    L.orc_collect_vlist.argtypes = [_I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P]
    L.orc_collect_ulist.argtypes = [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P]
    L.orc_collect_treecode.argtypes = [_I, _P, _P, _P, _P, _P, _D, _I, _P, _P, _I, _P, _P, _P]
    L.orc_exec_m2p.argtypes = [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int]
    L.orc_exec_p2p.argtypes = [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int, _P]
    L.orc_direct_subset.argtypes = [_I, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P, C.c_int]
    L.orc_partition_roots.argtypes = [_I, _P, _P, _P, _P, _P, _I, _P, _P]
    L.orc_partition_roots.restype = _I
    L.orc_collect_mutual.argtypes = [_I, _P, _P, _P, _P, _P, _P, C.c_int, _D, C.c_int, _I, _P, _P, _P, _I, _P, _P,
                                     _P, _P]
    L.orc_exec_m2l_mut.argtypes = [_I, _P, _P, _P, _P, _P, _P, C.c_int]
    L.orc_exec_p2p_mut.argtypes = [_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int, _P]
    L.orc_fmm.argtypes = [_I, _P, _P, _P, _P, _I, C.c_int, _D, C.c_int, _D,
                          _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]
    L.orc_fmm.restype = C.c_int
    L.orc_max_threads.restype = C.c_int


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def ncoef(p: int) -> int:
    return int(lib().orc_ncoef(p))


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# tree (src/geometry.py:200-206, src/tree.py:370-454)
# ---------------------------------------------------------------------------

def root_cube(x, y, z):
    """compute_bounds + cubic root (src/tree.py:387-392)."""
    lo = np.array([x.min(), y.min(), z.min()])
    hi = np.array([x.max(), y.max(), z.max()])
    size = float((hi - lo).max())
    if size == 0.0:
        size = 1.0
    return lo, size, (1 << MAX_LEVEL) / size


def encode_points(x, y, z, lo, inv_h) -> np.ndarray:
    x, y, z = f64(x), f64(y), f64(z)
    keys = np.empty(x.size, np.uint64)
    lib().orc_encode_points(x.size, _p(x), _p(y), _p(z), float(lo[0]), float(lo[1]), float(lo[2]),
                            float(inv_h), _p(keys))
    return keys


def argsort_stable(keys) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    order = np.empty(keys.size, np.int64)
    lib().orc_argsort_stable(keys.size, _p(keys), _p(order))
    return order


class OracleTree:
    """SoA tree with the reference's ``Tree`` field names (tree.py:275-302)."""


def build_tree(pos, q, ncrit=30, allow_oversized_leaves=False, shape="cubic",
               center_mode="geometric") -> OracleTree:
    """src/tree.py:370-454 (shape "cubic"/"rect", center_mode "geometric"/"com")."""
    if shape not in ("cubic", "rect") or center_mode not in ("geometric", "com"):
        raise ValueError("bad shape or center mode")
    pos = np.asarray(pos)
    x, y, z = f64(pos[:, 0]), f64(pos[:, 1]), f64(pos[:, 2])
    q = f64(q)
    n = x.size
    if n == 0:
        raise ValueError("empty particle set")
    lo, size, inv_h = root_cube(x, y, z)
    keys = encode_points(x, y, z, lo, inv_h)
    order = argsort_stable(keys)
    skeys = np.ascontiguousarray(keys[order])
    cap = max(64, 8 * (n // max(1, ncrit) + 1))
    while True:
        ch = np.empty((cap, 8), np.int64)
        par = np.empty(cap, np.int64)
        lev = np.empty(cap, np.int64)
        key = np.empty(cap, np.uint64)
        st = np.empty(cap, np.int64)
        en = np.empty(cap, np.int64)
        se = np.empty(cap, np.int64)
        flags = np.zeros(2, np.int64)
        nc = lib().orc_build_cells(_p(skeys), n, ncrit, int(allow_oversized_leaves), cap, _p(ch), _p(par),
                                   _p(lev), _p(key), _p(st), _p(en), _p(se), _p(flags))
        if nc < 0:
            cap *= 4
            continue
        break
    if flags[1]:
        raise ValueError(
            f"max depth exceeded: more than ncrit={ncrit} bodies share one depth-{MAX_LEVEL} "
            "grid cell (pass allow_oversized_leaves=True to keep them in one leaf)")
    t = OracleTree()
    t.n = n
    t.keys = skeys
    t.permutation = order
    t.x, t.y, t.z, t.q = (np.ascontiguousarray(a[order]) for a in (x, y, z, q))
    t.cell_children = np.ascontiguousarray(ch[:nc])
    t.cell_parent = par[:nc].copy()
    t.cell_level = lev[:nc].copy()
    t.cell_key = key[:nc].copy()
    t.cell_start = st[:nc].copy()
    t.cell_end = en[:nc].copy()
    t.cell_sub_end = se[:nc].copy()
    t.cell_leaf = np.ascontiguousarray((t.cell_children < 0).all(axis=1)).astype(np.uint8)
    t.ncells = int(nc)
    t.root_lo = lo
    t.root_size = size
    t.cell_lo = np.empty((nc, 3))
    t.cell_hi = np.empty((nc, 3))
    t.cell_center = np.empty((nc, 3))
    t.cell_bmax = np.empty(nc)
    t.cell_rmax = np.empty(nc)
    lib().orc_fill_geometry(nc, _p(t.cell_level), _p(t.cell_key), _p(t.cell_start), _p(t.cell_end),
                            _p(t.x), _p(t.y), _p(t.z), _p(t.q), float(lo[0]), float(lo[1]), float(lo[2]), size,
                            int(shape == "rect"), int(center_mode == "com"), _p(t.cell_lo), _p(t.cell_hi),
                            _p(t.cell_center), _p(t.cell_bmax), _p(t.cell_rmax))
    t.shape, t.center_mode = shape, center_mode
    return t


# ---------------------------------------------------------------------------
# passes, lists, executors
# ---------------------------------------------------------------------------

def upward(t: OracleTree, p: int) -> np.ndarray:
    """src/tree.py:163-174 / :457-472"""
    M = np.zeros((t.ncells, ncoef(p)))
    lib().orc_upward(t.ncells, _p(t.cell_children), _p(t.cell_start), _p(t.cell_end), _p(t.cell_leaf),
                     _p(t.cell_center), _p(t.x), _p(t.y), _p(t.z), _p(t.q), p, _p(M))
    return M


def collect_lists(t: OracleTree, theta: float):
    """Single (root, root) dual traversal (src/traversal.py:159-262).
    Returns (m2l_t, m2l_s, p2p_t, p2p_s) in DFS emission order."""
    capm = capp = max(2048, 64 * t.ncells)
    while True:
        mt = np.empty(capm, np.int64); ms = np.empty(capm, np.int64)
        pt = np.empty(capp, np.int64); ps = np.empty(capp, np.int64)
        out = np.zeros(3, np.int64)
        lib().orc_collect(t.ncells, _p(t.cell_children), _p(t.cell_leaf), _p(t.cell_center),
                          _p(t.cell_bmax), _p(t.cell_rmax), float(theta) * float(theta), 0, 0,
                          capm, _p(mt), _p(ms), capp, _p(pt), _p(ps), _p(out))
        if out[2] == 1:
            capm, capp = int(out[0]) + 1, int(out[1]) + 1
            continue
        nm, npp = int(out[0]), int(out[1])
        return mt[:nm], ms[:nm], pt[:npp], ps[:npp]


def exec_m2l(t: OracleTree, mt, ms, M, p) -> np.ndarray:
    """src/traversal.py:500-517 into zeroed locals."""
    L = np.zeros_like(M)
    mt = np.ascontiguousarray(mt, np.int64); ms = np.ascontiguousarray(ms, np.int64)
    lib().orc_exec_m2l(mt.size, _p(mt), _p(ms), _p(t.cell_center), _p(M), _p(L), p)
    return L


def exec_p2p(t: OracleTree, pt, ps, use_rsqrt=False, acc=None):
    """src/traversal.py:531-548 on zeroed accumulators (or into ``acc`` =
    (phi, fx, fy, fz), in place); returns (phi, fx, fy, fz, stats[pairs,
    skipped, flops])."""
    pt = np.ascontiguousarray(pt, np.int64); ps = np.ascontiguousarray(ps, np.int64)
    phi, fx, fy, fz = acc if acc is not None else (np.zeros(t.n) for _ in range(4))
    st = np.zeros(3, np.int64)
    lib().orc_exec_p2p(pt.size, _p(pt), _p(ps), _p(t.cell_start), _p(t.cell_end), _p(t.x), _p(t.y),
                       _p(t.z), _p(t.q), _p(phi), _p(fx), _p(fy), _p(fz), int(use_rsqrt), _p(st))
    return phi, fx, fy, fz, st


def downward(t: OracleTree, L, p, phi, fx, fy, fz):
    """src/tree.py:177-189 (accumulates into phi/f in place; L modified)."""
    lib().orc_downward(t.ncells, _p(t.cell_children), _p(t.cell_start), _p(t.cell_end),
                       _p(t.cell_leaf), _p(t.cell_center), _p(t.x), _p(t.y), _p(t.z), _p(phi), _p(fx),
                       _p(fy), _p(fz), p, _p(L))


def evaluate(t: OracleTree, p: int, theta: float):
    """evaluate_dual_tree restated sequentially (src/traversal.py:864-932).
    Returns dict with phi/fx/fy/fz (tree order), M, L, lists and stats."""
    M = upward(t, p)
    mt, ms, pt, ps = collect_lists(t, theta)
    L = exec_m2l(t, mt, ms, M, p)
    phi, fx, fy, fz, st = exec_p2p(t, pt, ps)
    Lw = L.copy()
    downward(t, Lw, p, phi, fx, fy, fz)
    return dict(phi=phi, fx=fx, fy=fy, fz=fz, M=M, L_m2l=L, m2l=(mt, ms), p2p=(pt, ps),
                p2p_pairs=int(st[0]), p2p_skipped=int(st[1]), m2l_calls=int(mt.size))


def collect_treecode(t: OracleTree, theta: float):
    """Per-target-leaf walk of the source tree (src/traversal.py:265-313),
    leaves in pre-order.  Returns (m2p_t, m2p_s, p2p_t, p2p_s)."""
    leaf_ids = np.ascontiguousarray(np.flatnonzero(t.cell_leaf), np.int64)
    capm = max(2048, 256 * leaf_ids.size)
    capp = max(2048, 64 * leaf_ids.size)
    while True:
        mt = np.empty(capm, np.int64); ms = np.empty(capm, np.int64)
        pt = np.empty(capp, np.int64); ps = np.empty(capp, np.int64)
        out = np.zeros(3, np.int64)
        lib().orc_collect_treecode(leaf_ids.size, _p(leaf_ids), _p(t.cell_children), _p(t.cell_leaf),
                                   _p(t.cell_center), _p(t.cell_bmax), float(theta) * float(theta), capm, _p(mt),
                                   _p(ms), capp, _p(pt), _p(ps), _p(out))
        if out[2] == 1:
            capm, capp = int(out[0]) + 1, int(out[1]) + 1
            continue
        nm, npp = int(out[0]), int(out[1])
        return mt[:nm], ms[:nm], pt[:npp], ps[:npp]


def exec_m2p(t: OracleTree, mt, ms, M, p, phi=None, fx=None, fy=None, fz=None):
    """src/traversal.py:520-528 -> src/_taylor.py:272-307, accumulating into
    (phi, fx, fy, fz) (zeroed when not given); returns them."""
    mt = np.ascontiguousarray(mt, np.int64); ms = np.ascontiguousarray(ms, np.int64)
    acc = [np.zeros(t.n) if a is None else a for a in (phi, fx, fy, fz)]
    lib().orc_exec_m2p(mt.size, _p(mt), _p(ms), _p(t.cell_start), _p(t.cell_end), _p(t.x), _p(t.y), _p(t.z),
                       *(_p(a) for a in acc), _p(t.cell_center), _p(M), p)
    return tuple(acc)


def evaluate_treecode(t: OracleTree, p: int, theta: float):
    """evaluate_treecode restated sequentially (src/traversal.py:1002-1046):
    M2P far field, then the P2P near field, on zeroed accumulators."""
    M = upward(t, p)
    mt, ms, pt, ps = collect_treecode(t, theta)
    acc = exec_m2p(t, mt, ms, M, p)
    phi, fx, fy, fz, st = exec_p2p(t, pt, ps, acc=acc)  # P2P adds onto the M2P sums
    return dict(phi=phi, fx=fx, fy=fy, fz=fz, M=M, m2p=(mt, ms), p2p=(pt, ps),
                p2p_pairs=int(st[0]), p2p_skipped=int(st[1]), m2p_calls=int(mt.size))


def level_tables(t: OracleTree):
    """_level_tables (src/traversal.py:1052-1058): cells sorted by
    (level, key), their keys, and level offsets."""
    order = np.ascontiguousarray(np.lexsort((t.cell_key, t.cell_level)).astype(np.int64))
    sorted_keys = np.ascontiguousarray(t.cell_key[order].astype(np.uint64))
    depth = int(t.cell_level.max())
    counts = np.bincount(t.cell_level, minlength=depth + 1)
    level_off = np.zeros(depth + 2, np.int64)
    np.cumsum(counts, out=level_off[1:])
    return order, sorted_keys, level_off


def collect_listfmm(t: OracleTree):
    """V list (src/traversal.py:341-403) over all cells and U list (:406-497)
    over all leaves: returns (m2l_t, m2l_s, p2p_t, p2p_s)."""
    order, skeys, loff = level_tables(t)
    lvl = np.ascontiguousarray(t.cell_level, np.int64)
    key = np.ascontiguousarray(t.cell_key, np.uint64)
    par = np.ascontiguousarray(t.cell_parent, np.int64)
    leaf_ids = np.ascontiguousarray(np.flatnonzero(t.cell_leaf), np.int64)
    cap = max(4096, 256 * t.ncells)
    while True:
        mt = np.empty(cap, np.int64); ms = np.empty(cap, np.int64)
        out = np.zeros(3, np.int64)
        lib().orc_collect_vlist(0, t.ncells, _p(lvl), _p(key), _p(par), _p(t.cell_children), _p(order), _p(skeys),
                                _p(loff), cap, _p(mt), _p(ms), _p(out))
        if out[2] == 1:
            cap = int(out[0]) + 1
            continue
        nm = int(out[0])
        break
    cap = max(4096, 64 * leaf_ids.size)
    while True:
        pt = np.empty(cap, np.int64); ps = np.empty(cap, np.int64)
        out = np.zeros(3, np.int64)
        lib().orc_collect_ulist(0, leaf_ids.size, _p(leaf_ids), _p(lvl), _p(key), _p(t.cell_leaf),
                                _p(np.ascontiguousarray(t.cell_sub_end, np.int64)), _p(order), _p(skeys), _p(loff),
                                cap, _p(pt), _p(ps), _p(out))
        if out[2] == 1:
            cap = int(out[1]) + 1
            continue
        npp = int(out[1])
        break
    return mt[:nm], ms[:nm], pt[:npp], ps[:npp]


def evaluate_listfmm(t: OracleTree, p: int):
    """evaluate_list_fmm restated sequentially (src/traversal.py:1127-1189)."""
    M = upward(t, p)
    mt, ms, pt, ps = collect_listfmm(t)
    L = exec_m2l(t, mt, ms, M, p)
    phi, fx, fy, fz, st = exec_p2p(t, pt, ps)
    downward(t, L.copy(), p, phi, fx, fy, fz)
    return dict(phi=phi, fx=fx, fy=fy, fz=fz, m2l=(mt, ms), p2p=(pt, ps), p2p_pairs=int(st[0]),
                p2p_skipped=int(st[1]), m2l_calls=int(mt.size))


# ---- cross-tree evaluation (targets of A, sources of B) -------------------
def collect_cross(A: OracleTree, B: OracleTree, theta: float):
    """Dual traversal from (root_A, root_B) (src/traversal.py:159-262 with a
    source tree): (m2l_t, m2l_s, p2p_t, p2p_s), targets in A, sources in B."""
    capm = capp = max(2048, 64 * (A.ncells + B.ncells))
    while True:
        mt = np.empty(capm, np.int64); ms = np.empty(capm, np.int64)
        pt = np.empty(capp, np.int64); ps = np.empty(capp, np.int64)
        out = np.zeros(3, np.int64)
        lib().orc_collect2(*(_p(a) for a in (A.cell_children, A.cell_leaf, A.cell_center, A.cell_bmax, A.cell_rmax,
                                              B.cell_children, B.cell_leaf, B.cell_center, B.cell_bmax, B.cell_rmax)),
                           float(theta) * float(theta), 0, 0, capm, _p(mt), _p(ms), capp, _p(pt), _p(ps), _p(out))
        if out[2] == 1:
            capm, capp = int(out[0]) + 1, int(out[1]) + 1
            continue
        return mt[:int(out[0])], ms[:int(out[0])], pt[:int(out[1])], ps[:int(out[1])]


def collect_treecode_cross(A: OracleTree, B: OracleTree, theta: float):
    """Treecode walk of A's leaves over B's tree (src/traversal.py:265-313)."""
    leaf_ids = np.ascontiguousarray(np.flatnonzero(A.cell_leaf), np.int64)
    capm = max(2048, 256 * leaf_ids.size)
    capp = max(2048, 64 * leaf_ids.size)
    while True:
        mt = np.empty(capm, np.int64); ms = np.empty(capm, np.int64)
        pt = np.empty(capp, np.int64); ps = np.empty(capp, np.int64)
        out = np.zeros(3, np.int64)
        lib().orc_collect_treecode2(leaf_ids.size, _p(leaf_ids), _p(A.cell_center), _p(A.cell_bmax),
                                    _p(B.cell_children), _p(B.cell_leaf), _p(B.cell_center), _p(B.cell_bmax),
                                    float(theta) * float(theta), capm, _p(mt), _p(ms), capp, _p(pt), _p(ps), _p(out))
        if out[2] == 1:
            capm, capp = int(out[0]) + 1, int(out[1]) + 1
            continue
        return mt[:int(out[0])], ms[:int(out[0])], pt[:int(out[1])], ps[:int(out[1])]


def exec_p2p_cross(A: OracleTree, B: OracleTree, pt, ps, acc=None, use_rsqrt=False):
    """src/traversal.py:552-597 into (phi, fx, fy, fz) of A (zeroed unless
    given); returns them and stats[pairs, skipped, flops]."""
    pt = np.ascontiguousarray(pt, np.int64); ps = np.ascontiguousarray(ps, np.int64)
    phi, fx, fy, fz = acc if acc is not None else (np.zeros(A.n) for _ in range(4))
    st = np.zeros(3, np.int64)
    lib().orc_exec_p2p_cross(pt.size, _p(pt), _p(ps), _p(A.cell_start), _p(A.cell_end), _p(A.x), _p(A.y), _p(A.z),
                             _p(phi), _p(fx), _p(fy), _p(fz), _p(B.cell_start), _p(B.cell_end), _p(B.x), _p(B.y),
                             _p(B.z), _p(B.q), int(use_rsqrt), _p(st))
    return phi, fx, fy, fz, st


def evaluate_cross(A: OracleTree, B: OracleTree, p: int, theta: float):
    """evaluate_dual_tree(A, source_tree=B) restated sequentially."""
    MB = upward(B, p)
    mt, ms, pt, ps = collect_cross(A, B, theta)
    L = np.zeros((A.ncells, ncoef(p)))
    mt64, ms64 = np.ascontiguousarray(mt, np.int64), np.ascontiguousarray(ms, np.int64)
    lib().orc_exec_m2l2(mt.size, _p(mt64), _p(ms64), _p(A.cell_center), _p(B.cell_center), _p(MB), _p(L), p)
    phi, fx, fy, fz, st = exec_p2p_cross(A, B, pt, ps)
    downward(A, L.copy(), p, phi, fx, fy, fz)
    return dict(phi=phi, fx=fx, fy=fy, fz=fz, m2l=(mt, ms), p2p=(pt, ps), p2p_pairs=int(st[0]),
                p2p_skipped=int(st[1]))


def evaluate_treecode_cross(A: OracleTree, B: OracleTree, p: int, theta: float):
    """evaluate_treecode(A, source_tree=B) restated sequentially."""
    MB = upward(B, p)
    mt, ms, pt, ps = collect_treecode_cross(A, B, theta)
    acc = [np.zeros(A.n) for _ in range(4)]
    mt64, ms64 = np.ascontiguousarray(mt, np.int64), np.ascontiguousarray(ms, np.int64)
    lib().orc_exec_m2p(mt.size, _p(mt64), _p(ms64), _p(A.cell_start), _p(A.cell_end), _p(A.x), _p(A.y), _p(A.z),
                       *(_p(a) for a in acc), _p(B.cell_center), _p(MB), p)
    phi, fx, fy, fz, st = exec_p2p_cross(A, B, pt, ps, acc=acc)
    return dict(phi=phi, fx=fx, fy=fy, fz=fz, m2p=(mt, ms), p2p=(pt, ps), p2p_pairs=int(st[0]),
                p2p_skipped=int(st[1]))


def direct(x, y, z, q, idx=None, threads=0):
    """src/kernels.py:208-228 / src/_taylor.py:496-528."""
    x, y, z, q = f64(x), f64(y), f64(z), f64(q)
    idx = np.arange(x.size, dtype=np.int64) if idx is None else np.ascontiguousarray(idx, np.int64)
    out = [np.zeros(idx.size) for _ in range(4)]
    lib().orc_direct_subset(x.size, _p(x), _p(y), _p(z), _p(q), idx.size, _p(idx), *(_p(o) for o in out),
                            int(threads))
    return tuple(out)


def error_sample_idx(n: int, sample: int = 1000, seed: int = 0) -> np.ndarray:
    """src/tuner.py:30-39: sorted tree-order sample indices."""
    if sample >= n:
        return np.arange(n, dtype=np.int64)
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=sample, replace=False)).astype(np.int64)


def fmm(pos, q, ncrit, p, theta, threads=0, tfrac=1.0):
    """Whole-FMM CPU run (the bench.py CPU baseline); see orc_fmm."""
    pos = np.asarray(pos)
    xin, yin, zin = f64(pos[:, 0]), f64(pos[:, 1]), f64(pos[:, 2])
    qin = f64(q)
    n = xin.size
    perm = np.empty(n, np.int64)
    arrs = [np.empty(n) for _ in range(8)]
    times = np.zeros(6)
    stats = np.zeros(6, np.int64)
    lib().orc_fmm(n, _p(xin), _p(yin), _p(zin), _p(qin), int(ncrit), int(p), float(theta), int(threads),
                  float(tfrac), _p(perm), *(_p(a) for a in arrs), _p(times), _p(stats))
    x, y, z, qq, phi, fx, fy, fz = arrs
    return dict(perm=perm, x=x, y=y, z=z, q=qq, phi=phi, fx=fx, fy=fy, fz=fz,
                times=dict(zip(("build", "upward", "lists", "m2l", "p2p", "downward"), times.tolist())),
                p2p_pairs=int(stats[0]), p2p_skipped=int(stats[1]), m2l_calls=int(stats[2]),
                leaves_done=int(stats[3]), bodies_done=int(stats[4]), ncells=int(stats[5]))


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ---------------------------------------------------------------------------
# mutual dual traversal
# ---------------------------------------------------------------------------
MAC_CODES = {"bh": 0, "bmax": 1, "fmm": 2}


def partition_roots(t: OracleTree, grain: int):
    """src/traversal.py:621-640: (sorted partition roots, owner map)."""
    roots = np.empty(t.ncells, np.int64)
    owner = np.empty(t.ncells, np.int64)
    nr = lib().orc_partition_roots(t.ncells, _p(t.cell_children), _p(t.cell_leaf), _p(t.cell_start),
                                   _p(t.cell_end), _p(np.ascontiguousarray(t.cell_sub_end, np.int64)), int(grain),
                                   _p(roots), _p(owner))
    return roots[:nr].copy(), owner


def collect_mutual(t: OracleTree, theta: float, grain: int, mac: str = "fmm", mutual: bool = True):
    """Driver + per-bucket _collect_units with (target, source, mut) entries
    (src/traversal.py:159-262, :704-791).  Returns (mt, ms, mm, pt, ps, pm)
    in the reference's execution order."""
    _, owner = partition_roots(t, grain)
    capm = capp = max(2048, 64 * t.ncells)
    while True:
        mt = np.empty(capm, np.int64); ms = np.empty(capm, np.int64); mm = np.empty(capm, np.uint8)
        pt = np.empty(capp, np.int64); ps = np.empty(capp, np.int64); pm = np.empty(capp, np.uint8)
        out = np.zeros(3, np.int64)
        lib().orc_collect_mutual(t.ncells, _p(t.cell_children), _p(t.cell_leaf), _p(t.cell_center),
                                 _p(t.cell_bmax), _p(t.cell_rmax), _p(owner), MAC_CODES[mac],
                                 float(theta) * float(theta), int(mutual), capm, _p(mt), _p(ms), _p(mm), capp,
                                 _p(pt), _p(ps), _p(pm), _p(out))
        if out[2] == 1:
            capm, capp = int(out[0]) + 1, int(out[1]) + 1
            continue
        nm, npp = int(out[0]), int(out[1])
        return mt[:nm], ms[:nm], mm[:nm], pt[:npp], ps[:npp], pm[:npp]


def expand_mutual(t, s, m):
    """Directed events of (target, source, mut) entries, as the reference's
    trace lists them (src/traversal.py:644-650): a mutual entry (a, b),
    a != b, also stands for (b, a)."""
    t, s, m = (np.asarray(a) for a in (t, s, m))
    rev = (m != 0) & (t != s)
    return np.concatenate([t, s[rev]]), np.concatenate([s, t[rev]])


def evaluate_mutual(t: OracleTree, p: int, theta: float, grain: int, mac: str = "fmm"):
    """evaluate_dual_tree(..., mutual=True) restated sequentially."""
    M = upward(t, p)
    mt, ms, mm, pt, ps, pm = collect_mutual(t, theta, grain, mac)
    L = np.zeros_like(M)
    lib().orc_exec_m2l_mut(mt.size, _p(mt), _p(ms), _p(mm), _p(t.cell_center), _p(M), _p(L), p)
    phi, fx, fy, fz = (np.zeros(t.n) for _ in range(4))
    st = np.zeros(3, np.int64)
    lib().orc_exec_p2p_mut(pt.size, _p(pt), _p(ps), _p(pm), _p(t.cell_start), _p(t.cell_end), _p(t.x), _p(t.y),
                           _p(t.z), _p(t.q), _p(phi), _p(fx), _p(fy), _p(fz), 0, _p(st))
    downward(t, L.copy(), p, phi, fx, fy, fz)
    m2l = expand_mutual(mt, ms, mm)
    return dict(phi=phi, fx=fx, fy=fy, fz=fz, m2l=m2l, p2p=expand_mutual(pt, ps, pm), p2p_pairs=int(st[0]),
                p2p_skipped=int(st[1]), m2l_calls=int(m2l[0].size))
