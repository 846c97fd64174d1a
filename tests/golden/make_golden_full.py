"""Full-size golden pins for the BASELINE configurations, from the REAL reference.

Run in the build container only (the reference is absent on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_full.py [case ...]

Cases (BASELINE.json configs):

* ``c2_full``  -- 2^20 uniform FP32, q ~ U[0,1), P=4, theta=0.4, ncrit=64
* ``c3_full``  -- Plummer 2^22, q = 1/N, P=5, theta=0.5, ncrit=64
* ``c5_full``  -- 2^24 uniform FP32, q ~ U[0,1), P=4, theta=0.4, ncrit=128
* ``c4_full_p{8,10}_t{0.3,0.4}`` -- the C4 high-order corner at 2^20
* ``c4_64k_p{P}_t{T}`` -- the C4 law at 2^16 over P in {3,4,6,8,10} and
  theta in {0.3,0.4,0.5,0.6} (reduced-N accuracy grid for the GPU test)

Per case it records SHA-256 of: the sorted depth-21 Morton keys, the
permutation, each of the 13 ``cell_*`` arrays, and the canonical M2L / P2P
pair sets of a single-root ``_collect_units`` (src/traversal.py:159-262);
the reference's ``KernelStats`` counters; and, on the 1000-body error
sample (src/tuner.py:30-39, tree order, seed 0), the reference FMM's own
float64 phi/f, the direct sums and the reference's errors.  Everything goes
to ``tests/golden/full/<case>.json`` (+ a small ``.npz`` of the sample), so
large cases stay a few kB.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import canon_pairs, fk, input_sha, sha, single_root_lists, tu, wl  # noqa: E402

OUT = os.path.join(HERE, "full")
THREADS = os.cpu_count() or 1


def cases():
    c = {
        "c2_full": (lambda: wl.config2(1 << 20, 0), 4, 0.4, 64),
        "c3_full": (lambda: wl.plummer(1 << 22, 0), 5, 0.5, 64),
        "c5_full": (lambda: wl.config5(1 << 24, 0), 4, 0.4, 128),
    }
    for p in (8, 10):
        for t in (0.3, 0.4):
            c[f"c4_full_p{p}_t{t}"] = (lambda: wl.config4(1 << 20, 0), p, t, 64)
    for p in (3, 4, 6, 8, 10):
        for t in (0.3, 0.4, 0.5, 0.6):
            c[f"c4_64k_p{p}_t{t}"] = (lambda: wl.config4(1 << 16, 0), p, t, 64)
    return c


def run(name, gen, p, theta, ncrit):
    t0 = time.time()
    pos, q = gen()
    ps = fk.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q)
    tree = fk.build_tree(ps, ncrit=ncrit)
    meta = dict(name=name, n=int(ps.n), p=p, theta=theta, ncrit=ncrit, input_sha=input_sha(pos, q),
                ncells=int(tree.ncells), nleaves=int(tree.nleaves), depth=int(tree.depth))
    from fmmkit.geometry import _encode_points, compute_bounds
    b = compute_bounds(ps)
    size = float(b.extent.max()) or 1.0
    keys = _encode_points(ps.x, ps.y, ps.z, b.lo[0], b.lo[1], b.lo[2], (1 << 21) / size)
    meta["keys_sha"] = sha(keys[tree.permutation].astype(np.uint64))
    meta["perm_sha"] = sha(tree.permutation.astype(np.int64))
    cells = dict(children=tree.cell_children.astype(np.int32), parent=tree.cell_parent.astype(np.int32),
                 level=tree.cell_level.astype(np.int8), key=tree.cell_key.astype(np.uint64),
                 start=tree.cell_start.astype(np.int32), end=tree.cell_end.astype(np.int32),
                 sub_end=tree.cell_sub_end.astype(np.int32), lo=tree.cell_lo, hi=tree.cell_hi,
                 center=tree.cell_center, bmax=tree.cell_bmax, rmax=tree.cell_rmax,
                 leaf=tree.cell_leaf.astype(np.uint8))
    meta["cells_sha"] = {k: sha(v) for k, v in cells.items()}
    del keys, cells
    mt, ms, pt, pp = single_root_lists(tree, theta)
    m2l = canon_pairs(mt, ms)
    del mt, ms
    meta["n_m2l"], meta["m2l_sha"] = int(m2l.size), sha(m2l)
    del m2l
    p2p = canon_pairs(pt, pp)
    del pt, pp
    meta["n_p2p"], meta["p2p_sha"] = int(p2p.size), sha(p2p)
    del p2p
    t_lists = time.time()
    cfg = fk.EvalConfig(strategy="dualtree", mac=fk.MacConfig("fmm", theta), p=p)
    rep = fk.evaluate_on_tree(tree, cfg, threads=THREADS)
    meta["stats"] = {k: v for k, v in rep.stats.as_dict().items() if k != "times"}
    meta["ref_times_ms"] = rep.to_dict()["times_ms"]
    meta["ref_threads"] = THREADS
    idx, _ = tu.error_sample(tree, 1000, 0)
    bo = tree.bodies
    dphi, dfx, dfy, dfz = fk.direct(bo, idx)
    fref = np.stack([dfx, dfy, dfz], 1)
    fgot = np.stack([bo.fx[idx], bo.fy[idx], bo.fz[idx]], 1)
    meta["force_err"] = float(np.sqrt(((fgot - fref) ** 2).sum() / (fref ** 2).sum()))
    meta["pot_err"] = float(np.sqrt(((bo.phi[idx] - dphi) ** 2).sum() / (dphi ** 2).sum()))
    meta["wall_s"] = {"lists": t_lists - t0, "total": time.time() - t0}
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), idx=idx.astype(np.int32),
                        phi=bo.phi[idx], fx=bo.fx[idx], fy=bo.fy[idx], fz=bo.fz[idx],
                        direct_phi=dphi, direct_fx=dfx, direct_fy=dfy, direct_fz=dfz)
    with open(os.path.join(OUT, name + ".json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(f"{name}: cells={meta['ncells']} m2l={meta['n_m2l']} p2p={meta['n_p2p']} "
          f"pairs={meta['stats']['p2p_pairs']} ferr={meta['force_err']:.3e} "
          f"perr={meta['pot_err']:.3e} {meta['wall_s']['total']:.1f}s", flush=True)


def main(argv):
    cs = cases()
    names = argv or list(cs)
    for n in names:
        if os.path.exists(os.path.join(OUT, n + ".json")) and not argv:
            continue
        run(n, *cs[n])


if __name__ == "__main__":
    main(sys.argv[1:])
