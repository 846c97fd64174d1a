"""Golden fixtures for the listfmm strategy, generated
from the REAL reference in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_listfmm.py

Per case: the V-list (M2L) pair set of ``_collect_vlist`` over all cells and
the U-list (P2P) pair set of ``_collect_ulist`` over all leaves
(src/traversal.py:342-497), checked to equal the threaded
``evaluate_list_fmm(trace=True)`` event sets; the final phi/f and counters;
the reference's own error against direct summation.  Written to
tests/golden/lf_<name>.npz and tests/golden/index_listfmm.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import canon_pairs, fk, input_sha, sha, tu, tv, wl  # noqa: E402


def lists(tree):
    order, sorted_keys, level_off = tv._level_tables(tree)
    cap = 1 << 16
    while True:
        m2l_t = np.empty(cap, np.int64); m2l_s = np.empty(cap, np.int64)
        out = np.zeros(3, np.int64)
        tv._collect_vlist(tree.cell_level, tree.cell_key, tree.cell_parent, tree.cell_children, order,
                          sorted_keys, level_off, 0, tree.ncells, m2l_t, m2l_s, out)
        if out[0] > cap:
            cap = int(out[0]) + 1
            continue
        nm = int(out[0])
        break
    leaf_ids = tree.leaves().astype(np.int64)
    cap = 1 << 16
    while True:
        p2p_t = np.empty(cap, np.int64); p2p_s = np.empty(cap, np.int64)
        out = np.zeros(3, np.int64)
        tv._collect_ulist(tree.cell_level, tree.cell_key, tree.cell_leaf, tree.cell_sub_end, order, sorted_keys,
                          level_off, leaf_ids, 0, leaf_ids.size, p2p_t, p2p_s, out)
        if out[1] > cap:
            cap = int(out[1]) + 1
            continue
        npp = int(out[1])
        break
    return m2l_t[:nm], m2l_s[:nm], p2p_t[:npp], p2p_s[:npp]


def run_case(name, pos, q, p, ncrit, *, full=True, direct_all=True, stored_inputs=False):
    pos = np.asarray(pos)
    q = np.asarray(q)
    ps = fk.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q)
    tree = fk.build_tree(ps, ncrit=ncrit)
    meta = dict(name=name, n=int(ps.n), p=p, theta=0.5, ncrit=ncrit, allow_oversized_leaves=False,
                input_sha=input_sha(pos, q), ncells=int(tree.ncells), nleaves=int(tree.nleaves))
    arrs = {}
    if stored_inputs:
        arrs["in_pos"] = pos.astype(np.float64)
        arrs["in_q"] = q.astype(np.float64)
    mt, ms, pt, pp = lists(tree)
    m2l, p2p = canon_pairs(mt, ms), canon_pairs(pt, pp)
    assert np.unique(p2p).size == p2p.size and np.unique(m2l).size == m2l.size, name
    meta.update(n_m2l=int(m2l.size), n_p2p=int(p2p.size), m2l_sha=sha(m2l), p2p_sha=sha(p2p))
    if full:
        arrs["m2l_pairs"], arrs["p2p_pairs"] = m2l, p2p
    cfg = fk.EvalConfig(strategy="listfmm", mac=fk.MacConfig("fmm", 0.5), p=p)
    rep = fk.evaluate_on_tree(tree, cfg, threads=4, trace=True)
    ev_m = canon_pairs([a for k, a, _ in rep.trace if k == "m2l"], [s for k, _, s in rep.trace if k == "m2l"])
    ev_p = canon_pairs([a for k, a, _ in rep.trace if k == "p2p"], [s for k, _, s in rep.trace if k == "p2p"])
    assert np.array_equal(ev_m, m2l) and np.array_equal(ev_p, p2p), name
    meta["stats"] = {k: v for k, v in rep.stats.as_dict().items() if k != "times"}
    bo = tree.bodies
    if full:
        arrs["phi"], arrs["fx"], arrs["fy"], arrs["fz"] = bo.phi, bo.fx, bo.fy, bo.fz
    idx = np.arange(bo.n, dtype=np.int64) if direct_all else tu.error_sample(tree, 1000, 0)[0]
    dphi, dfx, dfy, dfz = fk.direct(bo, idx)
    arrs["direct_idx"] = idx.astype(np.int32)
    arrs["direct_phi"], arrs["direct_fx"], arrs["direct_fy"], arrs["direct_fz"] = dphi, dfx, dfy, dfz
    arrs["sample_phi"] = bo.phi[idx]
    arrs["sample_fx"], arrs["sample_fy"], arrs["sample_fz"] = bo.fx[idx], bo.fy[idx], bo.fz[idx]
    fref = np.stack([dfx, dfy, dfz], 1)
    fgot = np.stack([bo.fx[idx], bo.fy[idx], bo.fz[idx]], 1)
    meta["force_err"] = float(np.sqrt(((fgot - fref) ** 2).sum() / (fref ** 2).sum()))
    meta["pot_err"] = float(np.sqrt(((bo.phi[idx] - dphi) ** 2).sum() / (dphi ** 2).sum()))
    print(f"lf_{name}: n={bo.n} m2l={m2l.size} p2p={p2p.size} ferr={meta['force_err']:.3e} "
          f"perr={meta['pot_err']:.3e}")
    np.savez_compressed(os.path.join(HERE, "lf_" + name + ".npz"), **arrs)
    return meta


def main():
    index = {}
    pos, q = wl.config1(10_000, 0)
    index["c1"] = run_case("c1", pos, q, 4, 64)
    pos, q = wl.uniform_unit(2000, 11)
    index["u2k_p5"] = run_case("u2k_p5", pos, q, 5, 30)
    pos, q = wl.clustered_points(3000, 7)
    index["clustered3k"] = run_case("clustered3k", pos, q, 5, 20)
    rng = np.random.default_rng(42)
    base = rng.random((400, 3))
    pos = np.concatenate([base, np.repeat(base[:5], 3, axis=0)])
    q = rng.uniform(-1, 1, pos.shape[0])
    index["coincident"] = run_case("coincident", pos, q, 4, 8, stored_inputs=True)
    pos, q = wl.config1(400, 3)
    index["order_p8"] = run_case("order_p8", pos, q, 8, 12)
    pos, q = wl.plummer(1 << 15, 0)
    index["plummer_32k"] = run_case("plummer_32k", pos, q, 5, 64, full=False, direct_all=False)
    pos, q = wl.config2(1 << 15, 0)
    index["c2_32k"] = run_case("c2_32k", pos, q, 4, 64, full=False, direct_all=False)
    with open(os.path.join(HERE, "index_listfmm.json"), "w") as fh:
        json.dump(index, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
