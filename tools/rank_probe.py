"""Per-rank device time of the Morton-partitioned evaluation, one rank at a
time on one GPU: for W in {1, 2, 4, 8} and every rank r < W, the bench step
(build_tree + evaluate_partitioned(rank=r, world=W)) timed with CUDA events,
with the exchanges replaced by no-ops (no rank ever waits on another, so
nothing here needs W GPUs).  max over r of the rank times is the step a
W-GPU run would take without its collectives (one multipole all-gather of
ncells x ncoef doubles and one result gather of 32 B/body over NVLink); the
projected strong-scaling efficiency is T_1 / (W * max_r T_r).

    python tools/rank_probe.py [--config C2] [--worlds 1,2,4,8]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import distributed as fd, workloads  # noqa: E402
from rank_probe_comm import NoComm  # noqa: E402


ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
gen, n, solver = workloads.CONFIGS[args.config]
pos, q = gen(n, 0)
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))
cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision="fp32")
flush = torch.empty(2 * 126 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
comm = NoComm()
out = {}
for world in [int(w) for w in args.worlds.split(",")]:
    ranks = []
    for r in range(world):
        def step():
            t = fb.build_tree(ps, ncrit=solver["ncrit"])
            if world == 1:
                fb.evaluate_on_tree(t, cfg)
            else:
                fd.evaluate_partitioned(t, cfg, r, world, comm=comm, results="root")
        for _ in range(5):
            step()
        ts = []
        for _ in range(args.reps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ranks.append(float(np.median(ts)))
    out[world] = {"rank_ms": ranks, "max_ms": max(ranks)}
    t1 = out[1]["max_ms"] if 1 in out else None
    eff = (t1 / (world * max(ranks))) if t1 else None
    print(json.dumps({"config": args.config, "world": world, "rank_ms": [round(x, 3) for x in ranks],
                      "step_ms_max_over_ranks": round(max(ranks), 3),
                      "projected_particles_per_s": n / (max(ranks) * 1e-3),
                      "projected_strong_efficiency": eff}), flush=True)
