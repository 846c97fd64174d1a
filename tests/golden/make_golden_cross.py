"""Golden fixtures for cross-tree evaluation (targets of one tree, sources of
another; src/traversal.py:864-932 and :1002-1046 with
``source_tree``), from the REAL reference:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_cross.py

Per case: the dual-tree M2L/P2P pair sets of a single (root_A, root_B)
``_collect_units`` call, the treecode M2P/P2P sets, counters and final
phi/f of both strategies (in target-tree order), and direct sums of the
sources at the targets.  Written to tests/golden/cx_<name>.npz and
tests/golden/index_cross.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import canon_pairs, fk, sha, tv, wl  # noqa: E402
from make_golden_treecode import treecode_lists  # noqa: E402,F401


def cross_lists(A, B, theta):
    cap, srows = 1 << 16, 1 << 14
    while True:
        m2l_t = np.empty(cap, np.int64); m2l_s = np.empty(cap, np.int64); m2l_m = np.empty(cap, np.uint8)
        p2p_t = np.empty(cap, np.int64); p2p_s = np.empty(cap, np.int64); p2p_m = np.empty(cap, np.uint8)
        stack = np.empty((srows, 2), np.int64)
        out = np.zeros(3, np.int64)
        tv._collect_units(np.array([[0, 0, 0]], np.int64), A.cell_children, A.cell_leaf, A.cell_center,
                          A.cell_bmax, A.cell_rmax, B.cell_children, B.cell_leaf, B.cell_center, B.cell_bmax,
                          B.cell_rmax, 2, theta * theta, m2l_t, m2l_s, m2l_m, p2p_t, p2p_s, p2p_m, stack, out)
        if out[2] == 2:
            srows *= 4
            continue
        if out[0] > cap or out[1] > cap:
            cap = int(max(out[0], out[1])) + 1
            continue
        nm, npp = int(out[0]), int(out[1])
        return m2l_t[:nm], m2l_s[:nm], p2p_t[:npp], p2p_s[:npp]


def cross_treecode_lists(A, B, theta):
    leaf_ids = A.leaves().astype(np.int64)
    capm = capp = 1 << 16
    while True:
        m2p_t = np.empty(capm, np.int64); m2p_s = np.empty(capm, np.int64)
        p2p_t = np.empty(capp, np.int64); p2p_s = np.empty(capp, np.int64)
        stack = np.empty(1 << 12, np.int64)
        out = np.zeros(3, np.int64)
        tv._collect_treecode(leaf_ids, 0, leaf_ids.size, A.cell_center, A.cell_bmax, B.cell_children, B.cell_leaf,
                             B.cell_center, B.cell_bmax, B.cell_rmax, 2, theta * theta, m2p_t, m2p_s, p2p_t, p2p_s,
                             stack, out)
        if out[0] > capm or out[1] > capp:
            capm, capp = int(out[0]) + 1, int(out[1]) + 1
            continue
        nm, npp = int(out[0]), int(out[1])
        return m2p_t[:nm], m2p_s[:nm], p2p_t[:npp], p2p_s[:npp]


def run_case(name, pa, qa, pb, qb, p, theta, ncrit_a, ncrit_b):
    A = fk.build_tree(fk.ParticleSet(pa[:, 0], pa[:, 1], pa[:, 2], qa), ncrit=ncrit_a)
    B = fk.build_tree(fk.ParticleSet(pb[:, 0], pb[:, 1], pb[:, 2], qb), ncrit=ncrit_b)
    meta = dict(name=name, p=p, theta=theta, ncrit_a=ncrit_a, ncrit_b=ncrit_b, na=int(A.n), nb=int(B.n))
    arrs = {"a_pos": pa.astype(np.float64), "a_q": qa.astype(np.float64), "b_pos": pb.astype(np.float64),
            "b_q": qb.astype(np.float64)}
    mt, ms, pt, ps = cross_lists(A, B, theta)
    meta.update(n_m2l=int(mt.size), n_p2p=int(pt.size), m2l_sha=sha(canon_pairs(mt, ms)),
                p2p_sha=sha(canon_pairs(pt, ps)))
    tmt, tms, tpt, tps = cross_treecode_lists(A, B, theta)
    meta.update(n_m2p=int(tmt.size), tc_p2p_n=int(tpt.size), m2p_sha=sha(canon_pairs(tmt, tms)),
                tc_p2p_sha=sha(canon_pairs(tpt, tps)))
    for strategy in ("dualtree", "treecode"):
        B.multipole = None
        A.multipole = None
        rep = fk.evaluate_on_tree(A, fk.EvalConfig(strategy=strategy, mac=fk.MacConfig("fmm", theta), p=p),
                                  source_tree=B, threads=4, trace=True)
        if strategy == "dualtree":
            ev_m = canon_pairs([a for k, a, _ in rep.trace if k == "m2l"], [s for k, _, s in rep.trace if k == "m2l"])
            ev_p = canon_pairs([a for k, a, _ in rep.trace if k == "p2p"], [s for k, _, s in rep.trace if k == "p2p"])
            assert sha(ev_m) == meta["m2l_sha"] and sha(ev_p) == meta["p2p_sha"], name
        meta["stats_" + strategy] = {k: v for k, v in rep.stats.as_dict().items() if k != "times"}
        for k in ("phi", "fx", "fy", "fz"):
            arrs[f"{strategy}_{k}"] = getattr(A.bodies, k).copy()
    # direct sums of all sources at every target (tree order of A)
    ba, bb = A.bodies, B.bodies
    dx = ba.x[:, None] - bb.x[None, :]
    dy = ba.y[:, None] - bb.y[None, :]
    dz = ba.z[:, None] - bb.z[None, :]
    r2 = dx * dx + dy * dy + dz * dz
    with np.errstate(divide="ignore"):
        rinv = np.where(r2 > 0, 1.0 / np.sqrt(r2), 0.0)
    qr = bb.q[None, :] * rinv
    qr3 = qr * rinv * rinv
    arrs["direct_phi"] = qr.sum(1)
    arrs["direct_fx"], arrs["direct_fy"], arrs["direct_fz"] = (qr3 * dx).sum(1), (qr3 * dy).sum(1), (qr3 * dz).sum(1)
    print(name, A.ncells, B.ncells, mt.size, pt.size, tmt.size, tpt.size, meta["stats_dualtree"]["p2p_skipped"])
    np.savez_compressed(os.path.join(HERE, "cx_" + name + ".npz"), **arrs)
    return meta


def main():
    index = {}
    pa, qa = wl.uniform_unit(2000, 1)
    pb, qb = wl.clustered_points(3000, 7)
    index["uniform_vs_clustered"] = run_case("uniform_vs_clustered", pa, qa, pb, qb, 5, 0.5, 30, 20)
    pa, qa = wl.config1(1500, 2)
    pb, qb = wl.uniform_unit(4000, 9)
    pb = pb * 2.0 - 0.5  # a larger source cube around the targets
    index["inside_bigger"] = run_case("inside_bigger", pa, qa, pb, qb, 4, 0.6, 16, 40)
    rng = np.random.default_rng(21)
    pa = rng.random((800, 3))
    pb = np.concatenate([rng.random((700, 3)), pa[::8]])  # 100 targets coincide with sources
    qa = rng.uniform(-1, 1, pa.shape[0])
    qb = rng.uniform(-1, 1, pb.shape[0])
    index["coincident"] = run_case("coincident", pa, qa, pb, qb, 4, 0.5, 12, 12)
    with open(os.path.join(HERE, "index_cross.json"), "w") as fh:
        json.dump(index, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
