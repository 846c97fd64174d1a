"""P2P-plan microbenchmark: builds the tree and the P2P CSR once, then times
fmm_p2p_plan alone (CUDA events) and checks the runs against the in-tree
library's (row ranges and run contents equal).

    FMM_B200_LIB=... python tools/plan_bench.py [--config C3] [--reps 10]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import _lib, workloads  # noqa: E402
from paper_1209_3516_b200.traversal import _p2p_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
gen, n, solver = workloads.CONFIGS[args.config]
pos, q = gen(n, 0)
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))
tree = fb.build_tree(ps, ncrit=solver["ncrit"])
lists = fb.interaction_lists(tree, fb.MacConfig("fmm", solver["theta"]), defer=False)
n_p2p = lists.n_p2p
wsp, wsb = _lib.workspace(max(n_p2p, tree.n, tree.ncells + 1), tree.device)
st = _lib.stream_handle()
ts = []
for r in range(args.reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan = _p2p_plan(tree, lists.p2p_grp, lists.p2p_rows, n_p2p, 0, tree.n, wsp, wsb, st)
    e1.record()
    e1.synchronize()
    if r:
        ts.append(e0.elapsed_time(e1))
nrows = int(plan["dev_nrows"].item())
rng = plan["run_off"][:2 * tree.ncells].view(-1, 2)
lr = plan["leaf_rows"][:nrows].long()
runs = plan["runs"]
# digest of every row's runs in row order (runs are stored row-locally)
import hashlib  # noqa: E402
rr = rng[:nrows].cpu().numpy()
ru = runs.cpu().numpy()
dig = hashlib.sha256(lr.cpu().numpy().tobytes())
for a, b in rr:
    dig.update(ru[a:b, :3].tobytes())
digest = dig.hexdigest()
ref_path = f"/tmp/plan_ref_{args.config}.txt"
if os.environ.get("FMM_B200_LIB"):
    same = open(ref_path).read() == digest if os.path.exists(ref_path) else None
else:
    open(ref_path, "w").write(digest)
    same = True
print(json.dumps({"config": args.config, "rows": nrows, "p2p_leaf_pairs": n_p2p, "ms": float(np.median(ts)),
                  "stats": plan["dev_stats"].tolist(), "runs_equal_default": same,
                  "lib": os.environ.get("FMM_B200_LIB", "default")}))
