"""Near-field arithmetic at the C4 corner: for each (p, theta) point and
each near-field mode (fp32, fp32acc = float32 terms + float64 sums, fp64),
the relative L2 force/potential error against direct summation on the
reference's 1000-body sample and the step time (C4: N=2^20 FP32 uniform,
q ~ U[-1,1), ncrit=64; whole FMM per step, CUDA events).

    python tools/nearfield_sweep.py [--points 8:0.3,10:0.4] > gpurun_out/nearfield.jsonl
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
from paper_1209_3516_b200.tuner import potential_sample, sampled_potential_error  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--points", default="6:0.3,8:0.3,8:0.4,10:0.3,10:0.4,10:0.5")
ap.add_argument("--modes", default="fp32,fp32acc,fp64")
ap.add_argument("--n", type=int, default=1 << 20)
args = ap.parse_args()
pos, q = workloads.config4(args.n, 0)
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))
tree = fb.build_tree(ps, ncrit=64)
idx, fref, pref = potential_sample(tree, 1000, 0)
for pt in args.points.split(","):
    p, th = int(pt.split(":")[0]), float(pt.split(":")[1])
    for mode in args.modes.split(","):
        os.environ["FMM_B200_NEAR_FIELD"] = mode
        cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", th), p=p, precision="fp32")
        times = []
        for r in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t = fb.build_tree(ps, ncrit=64)
            rep = fb.evaluate_on_tree(t, cfg)
            e1.record()
            e1.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        rec = {"p": p, "theta": th, "near_field": rep.near_field, "force_err": fb.sampled_force_error(t, idx, fref),
               "pot_err": sampled_potential_error(t, idx, pref), "ms": float(np.median(times)),
               "p2p_ms": rep.stats.times.get("p2p")}
        print(json.dumps(rec), flush=True)
os.environ.pop("FMM_B200_NEAR_FIELD", None)
