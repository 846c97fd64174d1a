"""C4 accuracy/speed sweep (BASELINE.json configs[3]): N=2^20 FP32 uniform,
q ~ U[-1,1), ncrit=64, P in {3,4,6,8,10} x theta in {0.3,0.4,0.5,0.6}.
Per point: relative L2 force/potential error against direct summation on
the reference's 1000-body sample (tree order, seed 0), and particles/s
(device-resident cloud, whole FMM per step, CUDA events)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import workloads  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
pos, q = workloads.config4(1 << 20, 0)
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))
tree = fb.build_tree(ps, ncrit=64)
from paper_1209_3516_b200.tuner import potential_sample  # noqa: E402
idx, fref, pref = potential_sample(tree, 1000, 0)
out = []
for p in (3, 4, 6, 8, 10):
    for th in (0.3, 0.4, 0.5, 0.6):
        cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", th), p=p, precision=prec)
        for _ in range(2):
            t = fb.build_tree(ps, ncrit=64)
            fb.evaluate_on_tree(t, cfg)
        times = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            t = fb.build_tree(ps, ncrit=64)
            rep = fb.evaluate_on_tree(t, cfg)
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3)
        ferr = fb.sampled_force_error(t, idx, fref)
        from paper_1209_3516_b200.tuner import sampled_potential_error
        perr = sampled_potential_error(t, idx, pref)
        rec = {"p": p, "theta": th, "precision": prec, "force_err": ferr, "pot_err": perr,
               "particles_per_s": (1 << 20) / float(np.median(times)), "ms": 1e3 * float(np.median(times)),
               "p2p_pairs": rep.stats.p2p_pairs, "m2l_calls": rep.stats.m2l_calls}
        print(json.dumps(rec), flush=True)
        out.append(rec)
json.dump(out, open(f"gpurun_out/c4_sweep_{prec}.json", "w"), indent=1)
