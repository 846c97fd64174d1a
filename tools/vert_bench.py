"""Vertical-pass microbenchmark: P2M + M2M (upward_pass) and L2L + L2P
(downward_pass) alone on one tree, CUDA events, median of --reps.

    python tools/vert_bench.py [--config C3] [--p 5]
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

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--p", type=int, default=0)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
gen, n, solver = workloads.CONFIGS[args.config]
p = args.p or solver["p"]
pos, q = gen(n, 0)
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))
tree = fb.build_tree(ps, ncrit=solver["ncrit"])


def timed(fn):
    ts = []
    for r in range(args.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


up = timed(lambda: fb.upward_pass(tree, p, sync=False))
M = tree.multipole.copy()
tree._L = torch.ones((tree.ncells, ncoef(p)), dtype=torch.float64, device="cuda") * 1e-3
down = timed(lambda: fb.downward_pass(tree, sync=False))
print(json.dumps({"config": args.config, "p": p, "ncells": tree.ncells, "upward_ms": up, "downward_ms": down,
                  "M_norm": float(np.linalg.norm(M))}))
