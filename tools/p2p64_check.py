"""FP64 P2P check: the streamed double4 kernel against the SoA kernel (IEEE
1/sqrt) on the same plan -- relative L2 difference and kernel times.

    python tools/p2p64_check.py [--config C2] [--n N] [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import _lib, workloads  # noqa: E402
from paper_1209_3516_b200.traversal import _packed_f64  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=10)
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
P = _lib.ptr


def run(packed):
    _lib.call("fmm_p2p", _lib.PREC_FP64, 0, 0, 0, lists.nrows, P(lists.dev_nrows), P(lists.leaf_rows),
              P(tree.d_start), P(tree.d_end), P(lists.run_off), P(lists.runs), P(tree.d_x), P(tree.d_y),
              P(tree.d_z), P(tree.d_q), P(packed), None, P(tree.d_phi), P(tree.d_fx), P(tree.d_fy), P(tree.d_fz),
              None, _lib.stream_handle())


def timed(packed):
    run(packed)
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(packed)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2], [a.clone() for a in (tree.d_phi, tree.d_fx, tree.d_fy, tree.d_fz)]


b64 = _packed_f64(tree)
t_soa, ref = timed(None)
t_str, got = timed(b64)
rel = [float(torch.linalg.norm(g - r) / torch.linalg.norm(r)) for g, r in zip(got, ref)]
mx = [float(((g - r).abs() / r.abs().clamp_min(1e-300)).max()) for g, r in zip(got, ref)]
print(json.dumps({"config": args.config, "n": n, "p2p_pairs": pairs, "soa_ms": t_soa, "streamed_ms": t_str,
                  "streamed_gpairs_per_s": pairs / t_str / 1e6, "speedup": t_soa / t_str,
                  "rel_l2_vs_soa": rel, "max_rel_vs_soa": mx,
                  "newton_steps": os.environ.get("FMM_RSQ64_NEWTON", "build default")}))
