"""Fine-grained timing of the host-buffer (e2e) path on C2."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import tree as ftree  # noqa: E402
from paper_1209_3516_b200 import workloads  # noqa: E402

gen, n, solver = workloads.CONFIGS["C2"]
pos, q = gen(n, 0)
hx, hy, hz = (np.ascontiguousarray(pos[:, k]) for k in range(3))
hq = np.ascontiguousarray(q)
cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision="fp32")
T = {}


def tick(name, t0):
    torch.cuda.synchronize()
    T.setdefault(name, []).append((time.perf_counter() - t0) * 1e3)
    return time.perf_counter()


for it in range(8):
    torch.cuda.synchronize()
    t = time.perf_counter()
    a = [ftree._to_device(v, torch.device("cuda", 0)) for v in (hx, hy, hz, hq)]
    t = tick("to_device x4", t)
    ps = fb.ParticleSet(hx, hy, hz, hq)
    t = tick("ParticleSet", t)
    tr = fb.build_tree(ps, ncrit=solver["ncrit"])
    t = tick("build_tree", t)
    fb.evaluate_on_tree(tr, cfg)
    t = tick("evaluate", t)
    acc = tr.device_results_in_input_order()
    t = tick("unpermute", t)
    host = []
    for v in acc:
        h = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
        h.copy_(v, non_blocking=True)
        host.append(h)
    t = tick("d2h pinned x4", t)
    src = [np.array(v) for v in ps.host_inputs()]
    t = tick("np.array inputs", t)
    r = fb.ParticleSet(*src, *(h.numpy() for h in host))
    t = tick("result ParticleSet", t)
    res = tr.results_in_input_order()
    t = tick("results_in_input_order (all)", t)
    del a, res, r
for k, v in T.items():
    print(f"{k:32s} median {np.median(v[2:]):7.3f} ms   min {min(v[2:]):7.3f}")
