"""Golden fixtures for the treecode strategy, generated
from the REAL reference in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_treecode.py

Per case (inputs regenerated from paper_1209_3516_b200.workloads seeds,
SHA-256 of the float64 inputs stored):

* the M2P and P2P pair sets of one ``_collect_treecode`` call over all
  leaves (src/traversal.py:265-313), checked to equal the threaded
  ``evaluate_treecode(trace=True)`` event sets                (bit-exact)
* M2P-only accumulators from ``_exec_m2p`` on zeroed bodies     (<= 1e-12)
* final ``phi, fx, fy, fz`` of ``evaluate_treecode`` and its counters
* the reference's own errors against direct summation.
Written to tests/golden/tc_<name>.npz and tests/golden/index_treecode.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import canon_pairs, fk, input_sha, sha, tu, tv, wl  # noqa: E402


def treecode_lists(tree, theta):
    leaf_ids = tree.leaves().astype(np.int64)
    ch, lf, ctr, bm, rm = (tree.cell_children, tree.cell_leaf, tree.cell_center, tree.cell_bmax,
                           tree.cell_rmax)
    capm = capp = 1 << 16
    srows = 1 << 12
    while True:
        m2p_t = np.empty(capm, np.int64); m2p_s = np.empty(capm, np.int64)
        p2p_t = np.empty(capp, np.int64); p2p_s = np.empty(capp, np.int64)
        stack = np.empty(srows, np.int64)
        out = np.zeros(3, np.int64)
        tv._collect_treecode(leaf_ids, 0, leaf_ids.size, ctr, bm, ch, lf, ctr, bm, rm, 2, theta * theta,
                             m2p_t, m2p_s, p2p_t, p2p_s, stack, out)
        if out[2] == 2:
            srows *= 4
            continue
        if out[0] > capm or out[1] > capp:
            capm, capp = int(out[0]) + 1, int(out[1]) + 1
            continue
        nm, npp = int(out[0]), int(out[1])
        return m2p_t[:nm].copy(), m2p_s[:nm].copy(), p2p_t[:npp].copy(), p2p_s[:npp].copy()


def run_case(name, pos, q, p, theta, ncrit, *, full=True, direct_all=True, stored_inputs=False):
    pos = np.asarray(pos)
    q = np.asarray(q)
    ps = fk.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q)
    tree = fk.build_tree(ps, ncrit=ncrit)
    meta = dict(name=name, n=int(ps.n), p=p, theta=theta, ncrit=ncrit, allow_oversized_leaves=False,
                input_sha=input_sha(pos, q), ncells=int(tree.ncells), nleaves=int(tree.nleaves))
    arrs = {}
    if stored_inputs:
        arrs["in_pos"] = pos.astype(np.float64)
        arrs["in_q"] = q.astype(np.float64)
    mt, ms, pt, pp = treecode_lists(tree, theta)
    m2p = canon_pairs(mt, ms)
    p2p = canon_pairs(pt, pp)
    meta.update(n_m2p=int(m2p.size), n_p2p=int(p2p.size), m2p_sha=sha(m2p), p2p_sha=sha(p2p))
    if full:
        arrs["m2p_pairs"] = m2p
        arrs["p2p_pairs"] = p2p

    fk.upward_pass(tree, p, fk.KernelStats())
    bd = tree.bodies.copy()
    bd.reset_accumulators()
    tv._exec_m2p(mt, ms, mt.size, tree.cell_start, tree.cell_end, bd.x, bd.y, bd.z, bd.phi, bd.fx, bd.fy,
                 bd.fz, tree.cell_center, tree.multipole, p)
    if full:
        arrs["m2p_phi"], arrs["m2p_fx"], arrs["m2p_fy"], arrs["m2p_fz"] = bd.phi, bd.fx, bd.fy, bd.fz
    meta["m2p_norm"] = [float(np.linalg.norm(v)) for v in (bd.phi, bd.fx, bd.fy, bd.fz)]

    tree.multipole = None
    cfg = fk.EvalConfig(strategy="treecode", mac=fk.MacConfig("fmm", theta), p=p)
    rep = fk.evaluate_on_tree(tree, cfg, threads=4, trace=True)
    ev_m = canon_pairs([a for k, a, _ in rep.trace if k == "m2p"], [s for k, _, s in rep.trace if k == "m2p"])
    ev_p = canon_pairs([a for k, a, _ in rep.trace if k == "p2p"], [s for k, _, s in rep.trace if k == "p2p"])
    assert np.array_equal(ev_m, m2p), name
    assert np.array_equal(ev_p, p2p), name
    meta["stats"] = {k: v for k, v in rep.stats.as_dict().items() if k != "times"}
    bo = tree.bodies
    if full:
        arrs["phi"], arrs["fx"], arrs["fy"], arrs["fz"] = bo.phi, bo.fx, bo.fy, bo.fz
    if direct_all:
        idx = np.arange(bo.n, dtype=np.int64)
    else:
        idx, _ = tu.error_sample(tree, 1000, 0)
    dphi, dfx, dfy, dfz = fk.direct(bo, idx)
    arrs["direct_idx"] = idx.astype(np.int32)
    arrs["direct_phi"], arrs["direct_fx"], arrs["direct_fy"], arrs["direct_fz"] = dphi, dfx, dfy, dfz
    arrs["sample_phi"] = bo.phi[idx]
    arrs["sample_fx"], arrs["sample_fy"], arrs["sample_fz"] = bo.fx[idx], bo.fy[idx], bo.fz[idx]
    fref = np.stack([dfx, dfy, dfz], 1)
    fgot = np.stack([bo.fx[idx], bo.fy[idx], bo.fz[idx]], 1)
    meta["force_err"] = float(np.sqrt(((fgot - fref) ** 2).sum() / (fref ** 2).sum()))
    meta["pot_err"] = float(np.sqrt(((bo.phi[idx] - dphi) ** 2).sum() / (dphi ** 2).sum()))
    print(f"tc_{name}: n={bo.n} m2p={m2p.size} p2p={p2p.size} ferr={meta['force_err']:.3e} "
          f"perr={meta['pot_err']:.3e}")
    np.savez_compressed(os.path.join(HERE, "tc_" + name + ".npz"), **arrs)
    return meta


def main():
    index = {}
    pos, q = wl.config1(10_000, 0)
    index["c1"] = run_case("c1", pos, q, 4, 0.4, 64)
    pos, q = wl.uniform_unit(2000, 11)
    index["u2k_p5"] = run_case("u2k_p5", pos, q, 5, 0.5, 30)
    pos, q = wl.clustered_points(3000, 7)
    index["clustered3k"] = run_case("clustered3k", pos, q, 5, 0.5, 20)
    rng = np.random.default_rng(42)
    base = rng.random((400, 3))
    pos = np.concatenate([base, np.repeat(base[:5], 3, axis=0)])
    q = rng.uniform(-1, 1, pos.shape[0])
    index["coincident"] = run_case("coincident", pos, q, 4, 0.6, 8, stored_inputs=True)
    pos, q = wl.config1(400, 3)
    for p in (1, 8, 12):
        index[f"order_p{p}"] = run_case(f"order_p{p}", pos, q, p, 0.6, 12)
    pos, q = wl.config2(1 << 15, 0)
    index["c2_32k"] = run_case("c2_32k", pos, q, 4, 0.4, 64, full=False, direct_all=False)
    with open(os.path.join(HERE, "index_treecode.json"), "w") as fh:
        json.dump(index, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
