"""Golden fixtures for rect / center-of-mass trees (SURVEY.md §8(f) 4,
src/tree.py:80-160 with rect=True and/or com=True), from the REAL reference:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_geometry.py

Per (case, shape, center_mode): SHA-256 of every cell_* array, the dual-tree
M2L/P2P pair sets (single-root ``_collect_units``), the dual-tree and
treecode counters and final phi/f.  Written to tests/golden/geo_<key>.npz
and tests/golden/index_geometry.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import canon_pairs, fk, input_sha, sha, single_root_lists, wl  # noqa: E402

FIELDS = ("children", "parent", "level", "key", "start", "end", "sub_end", "lo", "hi", "center", "bmax", "rmax",
          "leaf")
DT = dict(children=np.int32, parent=np.int32, level=np.int8, key=np.uint64, start=np.int32, end=np.int32,
          sub_end=np.int32, leaf=np.uint8)


def run(name, pos, q, shape, center, p, theta, ncrit, stored=False):
    ps = fk.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q)
    tree = fk.build_tree(ps, ncrit=ncrit, shape=shape, center_mode=center)
    key = f"{name}_{shape}_{center}"
    meta = dict(name=name, key=key, shape=shape, center_mode=center, n=int(ps.n), p=p, theta=theta, ncrit=ncrit,
                input_sha=input_sha(pos, q), ncells=int(tree.ncells))
    meta["cells_sha"] = {f: sha(getattr(tree, "cell_" + f).astype(DT.get(f, np.float64))) for f in FIELDS}
    mt, ms, pt, pp = single_root_lists(tree, theta)
    meta["m2l_sha"], meta["p2p_sha"] = sha(canon_pairs(mt, ms)), sha(canon_pairs(pt, pp))
    meta["n_m2l"], meta["n_p2p"] = int(mt.size), int(pt.size)
    arrs = {"in_pos": pos.astype(np.float64), "in_q": q.astype(np.float64)} if stored else {}
    for strategy in ("dualtree", "treecode"):
        tree.multipole = None
        rep = fk.evaluate_on_tree(tree, fk.EvalConfig(strategy=strategy, mac=fk.MacConfig("fmm", theta), p=p),
                                  threads=4)
        meta["stats_" + strategy] = {k: v for k, v in rep.stats.as_dict().items() if k != "times"}
        b = tree.bodies
        for k in ("phi", "fx", "fy", "fz"):
            arrs[f"{strategy}_{k}"] = getattr(b, k).copy()
    np.savez_compressed(os.path.join(HERE, "geo_" + key + ".npz"), **arrs)
    print(key, tree.ncells, mt.size, pt.size)
    return key, meta


def main():
    index = {}
    cases = []
    pos, q = wl.clustered_points(3000, 7)
    cases.append(("clustered3k", pos, q, 5, 0.5, 20, False))
    pos, q = wl.uniform_unit(2000, 11)
    cases.append(("u2k_p5", pos, q, 5, 0.5, 30, False))
    rng = np.random.default_rng(5)
    pz = rng.random((600, 3))
    cases.append(("zero_q", pz, np.zeros(600), 4, 0.6, 16, True))  # every cell: sum q == 0 -> box midpoint
    for name, pos, q, p, theta, ncrit, stored in cases:
        for shape, center in (("rect", "geometric"), ("cubic", "com"), ("rect", "com")):
            k, m = run(name, np.asarray(pos), np.asarray(q), shape, center, p, theta, ncrit, stored)
            index[k] = m
    with open(os.path.join(HERE, "index_geometry.json"), "w") as fh:
        json.dump(index, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
