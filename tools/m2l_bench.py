"""M2L-only microbenchmark: builds the tree, multipoles and lists once,
then times the M2L kernel alone (CUDA events, L2 flushed between launches)
and checks the locals against a reference launch of the in-tree library.

    FMM_B200_LIB=... python tools/m2l_bench.py [--config C3] [--p 5] [--reps 10]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import workloads  # noqa: E402
from paper_1209_3516_b200.kernels import ncoef  # noqa: E402
from paper_1209_3516_b200.traversal import run_m2l  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--p", type=int, default=0)
ap.add_argument("--theta", type=float, default=0.0)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--mode", default="both", choices=["both", "pairs", "grouped"])
args = ap.parse_args()
gen, n, solver = workloads.CONFIGS[args.config]
p = args.p or solver["p"]
theta = args.theta or solver["theta"]
pos, q = gen(n, 0)
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))
tree = fb.build_tree(ps, ncrit=solver["ncrit"])
fb.upward_pass(tree, p)
lists = fb.interaction_lists(tree, fb.MacConfig("fmm", theta))
nm2l = lists.n_m2l
tree._L = torch.zeros((tree.ncells, ncoef(p)), dtype=torch.float64, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
from paper_1209_3516_b200 import traversal as trv  # noqa: E402


def timed(min_p):
    trv.M2L_GROUPED_MIN_P = min_p
    ts = []
    for r in range(args.reps + 1):
        tree._L.zero_()
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_m2l(tree, lists, p)
        e1.record()
        e1.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), tree._L.double().cpu().numpy()


modes = {"pairs": 99, "grouped": 6} if args.mode == "both" else {args.mode: 99 if args.mode == "pairs" else 6}
out = {}
base = None
for name, mp in modes.items():
    ms, L = timed(mp)
    if base is None:
        base = L
    rel = float(np.linalg.norm(L - base) / np.linalg.norm(base))
    out[name] = {"ms": ms, "calls_per_s": nm2l / ms * 1e3, "rel_l2_vs_first": rel}
print(json.dumps({"config": args.config, "p": p, "theta": theta, "m2l_calls": nm2l, **out,
                  "lib": os.environ.get("FMM_B200_LIB", "default")}))
