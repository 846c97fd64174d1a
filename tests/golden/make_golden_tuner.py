"""Golden answers for the tuner from the REAL reference:
``max_theta_for_error`` per order and the errors of the tuned angles, on the
reference's tree_2k fixture cloud (uniform 2000, seed 11, ncrit 30).

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_tuner.py

Writes tests/golden/index_tuner.json.  (Timings, and therefore
``select_p_theta``'s winner, are host-dependent; the angles are not.)
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import fk, input_sha, tu, wl  # noqa: E402


def main():
    pos, q = wl.uniform_unit(2000, 11)
    ps = fk.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q)
    tree = fk.build_tree(ps, ncrit=30)
    oracle = tu.error_sample(tree, 1000, 0)
    out = {"name": "u2k", "input_sha": input_sha(pos, q), "ncrit": 30, "cases": []}
    for target in (1e-3, 1e-4, 1e-6):
        for p in (2, 3, 4, 5, 6):
            try:
                theta = tu.max_theta_for_error(tree, p, target, "fmm", threads=4, oracle=oracle)
            except ValueError as e:
                out["cases"].append({"target": target, "p": p, "theta": None, "error": str(e)})
                continue
            cfg = fk.EvalConfig(strategy="dualtree", mac=fk.MacConfig("fmm", theta), p=p)
            fk.evaluate_dual_tree(tree, cfg, threads=4)
            err = tu.sampled_force_error(tree, *oracle)
            out["cases"].append({"target": target, "p": p, "theta": theta, "tuned_error": err})
            print(target, p, theta, err)
    with open(os.path.join(HERE, "index_tuner.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
