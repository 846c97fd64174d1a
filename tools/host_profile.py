"""Host-side (Python) cost of one C2 step: cProfile of build_tree +
evaluate_on_tree after warm-up, sorted by own time.

    python tools/host_profile.py [--config C2] > gpurun_out/host_profile.txt
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
args = ap.parse_args()
gen, n, solver = workloads.CONFIGS[args.config]
pos, q = gen(n, 0)
cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision="fp32")
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))


def step():
    t = fb.build_tree(ps, ncrit=solver["ncrit"])
    fb.evaluate_on_tree(t, cfg)


for _ in range(4):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
step()
print(f"step wall {1e3 * (time.perf_counter() - t0):.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
