"""Host-side trace of one step without a profiler: every C-ABI call
(_lib.call) and Python phase with perf_counter stamps, so the host time
between the build's synchronisation and the P2P launch can be attributed.

    python tools/host_trace.py [--config C2] > gpurun_out/host_trace.txt
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import _lib, traversal, tree, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
args = ap.parse_args()
gen, n, solver = workloads.CONFIGS[args.config]
pos, q = gen(n, 0)
cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision="fp32")
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))
log = []
pc = time.perf_counter


def wrap(mod, name, label):
    f = getattr(mod, name)

    def g(*a, **k):
        t0 = pc()
        try:
            return f(*a, **k)
        finally:
            log.append((t0, pc(), label(a)))
    setattr(mod, name, g)


wrap(_lib, "call", lambda a: "call:" + a[0])
for nm in ("interaction_lists", "run_m2l", "run_p2p", "upward_pass", "downward_pass", "evaluate_dual_tree"):
    wrap(traversal, nm, lambda a, nm=nm: "py:" + nm)
wrap(tree, "build_tree", lambda a: "py:build_tree")
fb.build_tree = tree.build_tree
fb.evaluate_dual_tree = traversal.evaluate_dual_tree


def step():
    t = fb.build_tree(ps, ncrit=solver["ncrit"])
    fb.evaluate_on_tree(t, cfg)


for _ in range(5):
    step()
torch.cuda.synchronize()
for rep in range(3):
    log.clear()
    t0 = pc()
    step()
    t1 = pc()
    log.sort()
    print(f"--- step {rep}: host wall {1e3 * (t1 - t0):.2f} ms")
    prev = t0
    for s, e, nm in log:
        gap = s - prev
        print(f"{1e6 * (s - t0):9.1f} {1e6 * (e - s):8.1f} us  (+{1e6 * gap:7.1f} before)  {nm}")
        prev = max(prev, e) if not nm.startswith("py:") else s
