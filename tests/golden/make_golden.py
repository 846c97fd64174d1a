"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container only (the reference is not present on the GPU
box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports ``fmmkit`` from /root/reference/pkg/src and records, per case,
the per-stage outputs the B200 path must reproduce:

* depth-21 Morton keys (sorted) and ``tree.permutation``  (bit-exact)
* every ``cell_*`` array of the tree                       (bit-exact)
* the M2L and P2P pair sets from a single-root ``_collect_units`` call
  (``traversal.py:159-262``), checked here to equal the threaded
  ``evaluate_dual_tree(trace=True)`` event sets             (bit-exact)
* multipoles after ``upward_pass``                          (<= 1e-12)
* locals after ``_exec_m2l`` only (before the downward pass)
* P2P-only accumulators from ``_exec_p2p`` on zeroed bodies
* final ``phi, fx, fy, fz`` of ``evaluate_dual_tree``       (FP64 bar)
* direct-summation references and the reference's own errors.

Large list sets are stored as a count plus a SHA-256 of the canonical
encoding (sorted int64 ``t << 32 | s``) to keep fixtures small.
Inputs are regenerated from ``paper_1209_3516_b200.workloads`` seeds; a
SHA-256 of the float64 input bytes is stored to detect RNG drift.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import fmmkit as fk  # noqa: E402
from fmmkit import traversal as tv  # noqa: E402
from fmmkit import tuner as tu  # noqa: E402

from paper_1209_3516_b200 import workloads as wl  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def canon_pairs(t, s) -> np.ndarray:
    t = np.asarray(t, dtype=np.int64)
    s = np.asarray(s, dtype=np.int64)
    return np.sort((t << 32) | s)


def input_sha(pos, q) -> str:
    pos = np.asarray(pos, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    return sha(np.concatenate([pos[:, 0], pos[:, 1], pos[:, 2], q]))


def single_root_lists(tree, theta):
    """M2L/P2P pairs of the whole dual traversal from (root, root)."""
    ch, lf, ctr, bm, rm = (tree.cell_children, tree.cell_leaf, tree.cell_center,
                           tree.cell_bmax, tree.cell_rmax)
    cap = 1 << 16
    srows = 1 << 14
    while True:
        m2l_t = np.empty(cap, np.int64); m2l_s = np.empty(cap, np.int64); m2l_m = np.empty(cap, np.uint8)
        p2p_t = np.empty(cap, np.int64); p2p_s = np.empty(cap, np.int64); p2p_m = np.empty(cap, np.uint8)
        stack = np.empty((srows, 2), np.int64)
        out = np.zeros(3, np.int64)
        tv._collect_units(np.array([[0, 0, 0]], np.int64), ch, lf, ctr, bm, rm,
                          ch, lf, ctr, bm, rm, 2, theta * theta,
                          m2l_t, m2l_s, m2l_m, p2p_t, p2p_s, p2p_m, stack, out)
        if out[2] == 2:
            srows *= 4
            continue
        if out[0] > cap or out[1] > cap:
            cap = int(max(out[0], out[1])) + 1
            continue
        nm, npp = int(out[0]), int(out[1])
        return (m2l_t[:nm].copy(), m2l_s[:nm].copy(), p2p_t[:npp].copy(), p2p_s[:npp].copy())


def run_case(name, pos, q, p, theta, ncrit, *, full=True, allow=False,
             direct_all=True, check_trace=True, stored_inputs=False,
             results=False):
    pos = np.asarray(pos)
    q = np.asarray(q)
    ps = fk.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q)
    tree = fk.build_tree(ps, ncrit=ncrit, allow_oversized_leaves=allow)
    meta = dict(name=name, n=int(ps.n), p=p, theta=theta, ncrit=ncrit,
                allow_oversized_leaves=allow, input_sha=input_sha(pos, q),
                ncells=int(tree.ncells), nleaves=int(tree.nleaves), depth=int(tree.depth))
    arrs = {}
    if stored_inputs:
        arrs["in_pos"] = pos.astype(np.float64)
        arrs["in_q"] = q.astype(np.float64)

    # --- keys and permutation
    from fmmkit.geometry import _encode_points, compute_bounds
    b = compute_bounds(ps)
    size = float(b.extent.max()) or 1.0
    keys = _encode_points(ps.x, ps.y, ps.z, b.lo[0], b.lo[1], b.lo[2], (1 << 21) / size)
    skeys = keys[tree.permutation]
    meta["keys_sha"] = sha(skeys.astype(np.uint64))
    meta["perm_sha"] = sha(tree.permutation.astype(np.int64))
    meta["root_lo"] = [float(v) for v in tree.root_box.lo]
    meta["root_size"] = size

    cells = dict(children=tree.cell_children.astype(np.int32),
                 parent=tree.cell_parent.astype(np.int32),
                 level=tree.cell_level.astype(np.int8),
                 key=tree.cell_key.astype(np.uint64),
                 start=tree.cell_start.astype(np.int32),
                 end=tree.cell_end.astype(np.int32),
                 sub_end=tree.cell_sub_end.astype(np.int32),
                 lo=tree.cell_lo, hi=tree.cell_hi, center=tree.cell_center,
                 bmax=tree.cell_bmax, rmax=tree.cell_rmax,
                 leaf=tree.cell_leaf.astype(np.uint8))
    meta["cells_sha"] = {k: sha(v) for k, v in cells.items()}
    if full:
        arrs["keys"] = skeys.astype(np.uint64)
        arrs["perm"] = tree.permutation.astype(np.int32)
        for k, v in cells.items():
            arrs["cell_" + k] = v

    # --- lists
    mt, ms, pt, pp = single_root_lists(tree, theta)
    m2l = canon_pairs(mt, ms)
    p2p = canon_pairs(pt, pp)
    meta["n_m2l"] = int(m2l.size)
    meta["n_p2p"] = int(p2p.size)
    meta["m2l_sha"] = sha(m2l)
    meta["p2p_sha"] = sha(p2p)
    if full:
        arrs["m2l_pairs"] = m2l
        arrs["p2p_pairs"] = p2p

    # --- upward
    st = fk.KernelStats()
    fk.upward_pass(tree, p, st)
    M = tree.multipole.copy()
    if full or results:
        arrs["multipole"] = M
    meta["multipole_norm"] = float(np.linalg.norm(M))

    # --- M2L-only locals in single-root list order
    L = np.zeros_like(M)
    tv._exec_m2l(mt, ms, np.zeros(mt.size, np.uint8), mt.size, tree.cell_center,
                 tree.cell_center, M, M, L, L, p)
    if full or results:
        arrs["local_m2l"] = L
    meta["local_m2l_norm"] = float(np.linalg.norm(L))

    # --- P2P-only accumulators
    bd = tree.bodies.copy()
    bd.reset_accumulators()
    s3 = np.zeros(3, np.int64)
    tv._exec_p2p(pt, pp, np.zeros(pt.size, np.uint8), pt.size, tree.cell_start, tree.cell_end,
                 bd.x, bd.y, bd.z, bd.q, bd.phi, bd.fx, bd.fy, bd.fz, False, s3)
    if full:
        arrs["p2p_phi"], arrs["p2p_fx"], arrs["p2p_fy"], arrs["p2p_fz"] = bd.phi, bd.fx, bd.fy, bd.fz
    else:
        meta["p2p_norm"] = [float(np.linalg.norm(v)) for v in (bd.phi, bd.fx, bd.fy, bd.fz)]

    # --- full evaluation (threaded, the reference's own path)
    tree.multipole = None
    cfg = fk.EvalConfig(strategy="dualtree", mac=fk.MacConfig("fmm", theta), p=p)
    rep = fk.evaluate_on_tree(tree, cfg, threads=4, trace=check_trace)
    if check_trace:
        ev_m = canon_pairs([a for k, a, _ in rep.trace if k == "m2l"], [s for k, _, s in rep.trace if k == "m2l"])
        ev_p = canon_pairs([a for k, a, _ in rep.trace if k == "p2p"], [s for k, _, s in rep.trace if k == "p2p"])
        assert np.array_equal(ev_m, m2l), name
        assert np.array_equal(ev_p, p2p), name
    counts = {k: v for k, v in rep.stats.as_dict().items() if k != "times"}
    meta["stats"] = counts
    bo = tree.bodies
    if full or results:
        arrs["phi"], arrs["fx"], arrs["fy"], arrs["fz"] = bo.phi, bo.fx, bo.fy, bo.fz

    # --- direct references and the reference's own errors
    if direct_all:
        idx = np.arange(bo.n, dtype=np.int64)
    else:
        idx, _ = tu.error_sample(tree, 1000, 0)
    dphi, dfx, dfy, dfz = fk.direct(bo, idx)
    arrs["direct_idx"] = idx.astype(np.int32)
    arrs["direct_phi"], arrs["direct_fx"], arrs["direct_fy"], arrs["direct_fz"] = dphi, dfx, dfy, dfz
    if not full:
        arrs["sample_phi"] = bo.phi[idx]
        arrs["sample_fx"], arrs["sample_fy"], arrs["sample_fz"] = bo.fx[idx], bo.fy[idx], bo.fz[idx]
    fref = np.stack([dfx, dfy, dfz], 1)
    fgot = np.stack([bo.fx[idx], bo.fy[idx], bo.fz[idx]], 1)
    meta["force_err"] = float(np.sqrt(((fgot - fref) ** 2).sum() / (fref ** 2).sum()))
    meta["pot_err"] = float(np.sqrt(((bo.phi[idx] - dphi) ** 2).sum() / (dphi ** 2).sum()))
    print(f"{name}: n={bo.n} cells={tree.ncells} m2l={m2l.size} p2p={p2p.size} "
          f"ferr={meta['force_err']:.3e} perr={meta['pot_err']:.3e}")
    return meta, arrs


def save(meta, arrs):
    np.savez_compressed(os.path.join(HERE, meta["name"] + ".npz"), **arrs)
    return meta


def main():
    index = {}

    def add(meta, arrs):
        index[meta["name"]] = save(meta, arrs)

    # C1 exactly as BASELINE.json configs[0]
    pos, q = wl.config1(10_000, 0)
    add(*run_case("c1", pos, q, 4, 0.4, 64))

    # reference fixture tree_2k (conftest.py:43-52) at the accuracy test's p/theta
    pos, q = wl.uniform_unit(2000, 11)
    add(*run_case("u2k_p5", pos, q, 5, 0.5, 30))

    # clustered fixture (conftest.py:61-65)
    pos, q = wl.clustered_points(3000, 7)
    add(*run_case("clustered3k", pos, q, 5, 0.5, 20))

    # completeness case (test_traversal.py:50-59)
    pos, q = wl.uniform_unit(300, 5)
    add(*run_case("u300_ncrit8", pos, q, 4, 0.7, 8))

    # coincident bodies: duplicate groups of 4 inside ncrit=8 leaves
    rng = np.random.default_rng(42)
    base = rng.random((400, 3))
    dup = np.repeat(base[:5], 3, axis=0)
    pos = np.concatenate([base, dup])
    q = rng.uniform(-1, 1, pos.shape[0])
    add(*run_case("coincident", pos, q, 4, 0.6, 8, stored_inputs=True))

    # all bodies at one point (test_tree.py:141-150), kept with oversized leaves
    pos = np.zeros((40, 3))
    q = np.ones(40)
    ps = fk.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q)
    try:
        fk.build_tree(ps, ncrit=8)
        raise SystemExit("expected max depth error")
    except ValueError as e:
        index["max_depth_message"] = str(e)
    add(*run_case("all_coincident", pos, q, 3, 0.6, 8, allow=True, stored_inputs=True))

    # one body per octant, ncrit=1 (test_tree.py:25-34)
    grid = np.array([[x, y, z] for x in (0.25, 0.75) for y in (0.25, 0.75) for z in (0.25, 0.75)])
    add(*run_case("octants", grid, np.ones(8), 2, 0.6, 1, stored_inputs=True))

    # tiny theta degenerates to direct (test_traversal.py:153-163)
    pos, q = wl.uniform_unit(1000, 14)
    add(*run_case("tiny_theta", pos, q, 4, 1e-6, 30))

    # order sweep on one tree
    pos, q = wl.config1(400, 3)
    for p in (1, 2, 3, 6, 8, 10, 12):
        add(*run_case(f"order_p{p}", pos, q, p, 0.6, 12, check_trace=False,
                      full=(p == 1), results=True))

    # C2 law at reduced N (FP32-rounded inputs), hashes only
    pos, q = wl.config2(1 << 15, 0)
    add(*run_case("c2_32k", pos, q, 4, 0.4, 64, full=False, direct_all=False))

    # Plummer (C3 law) at reduced N: adaptive depth
    pos, q = wl.plummer(1 << 15, 0)
    add(*run_case("plummer_32k", pos, q, 5, 0.5, 64, full=False, direct_all=False))

    # C5 leaf size at reduced N
    pos, q = wl.config5(1 << 16, 1)
    add(*run_case("c5_64k_ncrit128", pos, q, 4, 0.4, 128, full=False, direct_all=False,
                  check_trace=False))

    with open(os.path.join(HERE, "index.json"), "w") as fh:
        json.dump(index, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
