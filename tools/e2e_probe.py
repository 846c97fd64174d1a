"""Time the pieces of the e2e (host buffers) path on C2:
ParticleSet -> build_tree -> evaluate_on_tree -> results_in_input_order."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import workloads  # noqa: E402

gen, n, solver = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
pos, q = gen(n, 0)
hx, hy, hz = (np.ascontiguousarray(pos[:, k]) for k in range(3))
hq = np.ascontiguousarray(q)
cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision="fp32")
for it in range(6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    ps = fb.ParticleSet(hx, hy, hz, hq)
    t.append(time.perf_counter())
    tr = fb.build_tree(ps, ncrit=solver["ncrit"])
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    rep = fb.evaluate_on_tree(tr, cfg)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    res = tr.results_in_input_order()
    t.append(time.perf_counter())
    _ = res.phi[0]
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"iter {it}: particleset {d[0]:.2f}  build {d[1]:.2f}  evaluate {d[2]:.2f}  results {d[3]:.2f} "
          f"touch {d[4]:.2f}  total {sum(d):.2f} ms", flush=True)
