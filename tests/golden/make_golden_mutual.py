"""Golden fixtures for the mutual dual traversal (
src/traversal.py:159-262 with mutual units, :704-791 driver, :621-639
partition roots; src/_taylor.py:191-217, :410-493 symmetric kernels), from
the REAL reference:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_mutual.py

The mutual list sets depend on the target partition (``task_grain``): a
mutual pair straddling two partition roots is demoted to two directed
pairs.  Per case: the partition roots, the directed-expanded M2L / P2P event
sets of ``evaluate_dual_tree(..., mutual=True, trace=True)``, the counters,
final phi/f (tree order) and direct sums.  Written to
tests/golden/mu_<name>.npz and tests/golden/index_mutual.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import canon_pairs, fk, sha, tv, wl  # noqa: E402


def run_case(name, pos, q, *, p, theta, ncrit, grain, mac="fmm"):
    pos = np.asarray(pos, np.float64)
    q = np.asarray(q, np.float64)
    tree = fk.build_tree(fk.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q), ncrit=ncrit)
    roots = tv._partition_roots(tree, grain)
    cfg = fk.EvalConfig(strategy="dualtree", mac=fk.MacConfig(mac, theta), p=p, mutual=True, task_grain=grain)
    rep = fk.evaluate_on_tree(tree, cfg, threads=4, trace=True)
    ev = {k: [(a, b) for kk, a, b in rep.trace if kk == k] for k in ("m2l", "p2p")}
    meta = dict(name=name, p=p, theta=theta, ncrit=ncrit, grain=grain, mac=mac, n=int(tree.n),
                ncells=int(tree.ncells), n_roots=int(roots.size))
    for k, v in ev.items():
        t = np.array([a for a, _ in v], np.int64)
        s = np.array([b for _, b in v], np.int64)
        c = canon_pairs(t, s)
        assert np.unique(c).size == c.size, (name, k, "duplicate directed events")
        meta[f"n_{k}"] = int(c.size)
        meta[f"{k}_sha"] = sha(c)
    meta["stats"] = {k: v for k, v in rep.stats.as_dict().items() if k != "times"}
    arrs = {"pos": pos, "q": q, "roots": roots.astype(np.int64)}
    b = tree.bodies
    for k in ("phi", "fx", "fy", "fz"):
        arrs[k] = getattr(b, k).copy()
    # the directed evaluation's lists for contrast (mutual sets must differ
    # somewhere for the case to pin anything beyond the directed traversal)
    tree.reset_accumulators()
    rep_d = fk.evaluate_on_tree(tree, fk.EvalConfig(strategy="dualtree", mac=fk.MacConfig(mac, theta), p=p),
                                threads=1, trace=True)
    dm = canon_pairs([a for k, a, _ in rep_d.trace if k == "m2l"], [s for k, _, s in rep_d.trace if k == "m2l"])
    meta["differs_from_directed"] = bool(sha(dm) != meta["m2l_sha"])
    # direct sums at every body (tree order)
    dx = b.x[:, None] - b.x[None, :]
    dy = b.y[:, None] - b.y[None, :]
    dz = b.z[:, None] - b.z[None, :]
    r2 = dx * dx + dy * dy + dz * dz
    with np.errstate(divide="ignore"):
        rinv = np.where(r2 > 0, 1.0 / np.sqrt(r2), 0.0)
    qr = b.q[None, :] * rinv
    qr3 = qr * rinv * rinv
    arrs["direct_phi"] = qr.sum(1)
    arrs["direct_fx"], arrs["direct_fy"], arrs["direct_fz"] = (qr3 * dx).sum(1), (qr3 * dy).sum(1), (qr3 * dz).sum(1)
    print(name, tree.ncells, roots.size, meta["n_m2l"], meta["n_p2p"], meta["stats"]["p2p_pairs"],
          meta["differs_from_directed"])
    np.savez_compressed(os.path.join(HERE, "mu_" + name + ".npz"), **arrs)
    return meta


def main():
    index = {}
    ps = fk.generate_distribution("uniform", 512, seed=9)  # tests/test_traversal.py:62-68
    pos = np.stack([ps.x, ps.y, ps.z], 1)
    for grain in (1, 64, 10 ** 9):
        nm = f"u512_g{grain if grain < 10 ** 9 else 'inf'}"
        index[nm] = run_case(nm, pos, ps.q, p=4, theta=0.6, ncrit=8, grain=grain)
    pos, q = wl.config1(4000, 3)
    index["c1_4k_g5000"] = run_case("c1_4k_g5000", pos, q, p=4, theta=0.4, ncrit=32, grain=5000)
    index["c1_4k_g700"] = run_case("c1_4k_g700", pos, q, p=5, theta=0.5, ncrit=32, grain=700)
    pos, q = wl.clustered_points(3000, 7)
    index["clustered_bh"] = run_case("clustered_bh", pos, q, p=5, theta=0.5, ncrit=20, grain=300, mac="bh")
    index["clustered_bmax"] = run_case("clustered_bmax", pos, q, p=4, theta=0.6, ncrit=20, grain=1000, mac="bmax")
    rng = np.random.default_rng(33)
    pos = rng.random((600, 3))
    pos = np.concatenate([pos, pos[::6]])  # 100 bodies coincide with another
    q = rng.uniform(-1, 1, pos.shape[0])
    index["coincident"] = run_case("coincident", pos, q, p=4, theta=0.5, ncrit=12, grain=100)
    with open(os.path.join(HERE, "index_mutual.json"), "w") as fh:
        json.dump(index, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
