"""P2P-only microbenchmark on the C2 leaf lists (BASELINE.json configs[1]:
"also reported separately: a P2P-only microbenchmark using the same leaf
lists").  Builds the tree and lists once, then times the P2P kernel alone
with CUDA events (L2 flushed between launches) and checks its FP32 output
against the FP64 kernel on the same lists.

    python tools/p2p_bench.py [--config C2] [--reps 20]
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
from paper_1209_3516_b200.traversal import run_p2p  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--precision", default="fp32")
ap.add_argument("--dump", default="", help="save the P2P outputs (torch.save) for a bitwise A/B")
args = ap.parse_args()
gen, n, solver = workloads.CONFIGS[args.config]
n = args.n or n
pos, q = gen(n, 0)
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))
tree = fb.build_tree(ps, ncrit=solver["ncrit"])
lists = fb.interaction_lists(tree, fb.MacConfig("fmm", solver["theta"]))
pairs = int(lists.dev_stats[0].item())
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
run_p2p(tree, lists, "fp64", flag=flag)
ref = [a.clone() for a in (tree.d_phi, tree.d_fx, tree.d_fy, tree.d_fz)]
for _ in range(3):
    run_p2p(tree, lists, args.precision, flag=flag)
times = []
for _ in range(args.reps):
    flush.fill_(0.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run_p2p(tree, lists, args.precision, flag=flag)
    e1.record()
    e1.synchronize()
    times.append(e0.elapsed_time(e1) * 1e-3)
got = [tree.d_phi, tree.d_fx, tree.d_fy, tree.d_fz]
if args.dump:
    torch.save([g.cpu() for g in got], args.dump)
rel = [float(torch.linalg.norm(g - r) / torch.linalg.norm(r)) for g, r in zip(got, ref)]
t = float(np.median(times))
print(json.dumps({"config": args.config, "n": n, "precision": args.precision, "p2p_pairs": pairs,
                  "nrows": int(lists.dev_nrows.item()), "ms": 1e3 * t, "min_ms": 1e3 * min(times),
                  "ginteractions_per_s": pairs / t / 1e9, "tflops_20": 20 * pairs / t / 1e12,
                  "rel_l2_vs_fp64": rel, "lib": os.environ.get("FMM_B200_LIB", "default")}))
