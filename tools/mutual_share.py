"""Share of the directed near-field work that sits in symmetric (mutual)
leaf pairs, from the oracle's mutual lists (the reference's
`_collect_units` with mutual units, src/traversal.py:159-262).  This bounds
what a symmetric P2P kernel could save ("Symmetric P2P").

    python tools/mutual_share.py [--n 1048576] [--theta 0.4] [--grain 5000]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (test infrastructure: a measurement, not the product)

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 20)
ap.add_argument("--theta", type=float, default=0.4)
ap.add_argument("--grain", type=int, default=5000)
ap.add_argument("--ncrit", type=int, default=64)
a = ap.parse_args()
rng = np.random.default_rng(0)
pos = rng.random((a.n, 3)).astype(np.float32).astype(np.float64)
t = O.build_tree(pos, rng.random(a.n), ncrit=a.ncrit)
_, _, _, pt, ps, pm = O.collect_mutual(t, a.theta, a.grain)
cnt = (t.cell_end - t.cell_start).astype(np.int64)
w = cnt[pt] * cnt[ps]
sym = (pm != 0) & (pt != ps)
directed = np.where(sym, 2 * w, w).sum()
share = 2 * w[sym].sum() / directed
print(f"n={a.n} theta={a.theta} grain={a.grain}: {share:.4f} of the directed body pairs are in symmetric leaf pairs; "
      f"a symmetric kernel (19 instead of 2x13 FP32 operations per pair) saves at most {share * 7 / 26:.4f} of P2P")
