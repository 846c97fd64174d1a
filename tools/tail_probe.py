"""Host time after the evaluation's final synchronisation (the step's tail:
the GPU is idle while the report is assembled) and before the build's first
kernel.  Wraps Event.synchronize / Event.elapsed_time to timestamp them.

    python tools/tail_probe.py [--config C2]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=30)
    args = ap.parse_args()
    gen, n, solver = workloads.CONFIGS[args.config]
    pos, q = gen(n, 0)
    dev = torch.device("cuda", 0)
    dt = torch.float32 if pos.dtype == np.float32 else torch.float64
    dpos = torch.as_tensor(pos, device=dev).to(dt)
    ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                        torch.as_tensor(q, device=dev).to(dt))
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision="fp32")
    marks = {"sync_end": 0.0, "n_elapsed": 0, "t_elapsed": 0.0}
    sync0, el0 = torch.cuda.Event.synchronize, torch.cuda.Event.elapsed_time

    def sync(self):
        sync0(self)
        marks["sync_end"] = time.perf_counter()

    def elapsed(self, other):
        t = time.perf_counter()
        r = el0(self, other)
        marks["n_elapsed"] += 1
        marks["t_elapsed"] += time.perf_counter() - t
        return r

    torch.cuda.Event.synchronize, torch.cuda.Event.elapsed_time = sync, elapsed
    tails, nel, tel, builds = [], [], [], []
    for i in range(args.steps + 5):
        torch.cuda.synchronize()
        marks.update(n_elapsed=0, t_elapsed=0.0)
        t0 = time.perf_counter()
        tree = fb.build_tree(ps, ncrit=solver["ncrit"])
        t1 = time.perf_counter()
        fb.evaluate_on_tree(tree, cfg)
        t2 = time.perf_counter()
        if i >= 5:
            tails.append(t2 - marks["sync_end"])
            nel.append(marks["n_elapsed"])
            tel.append(marks["t_elapsed"])
            builds.append(t1 - t0)
    us = lambda v: round(1e6 * float(np.median(v)), 1)  # noqa: E731
    print(f"{args.config}: host tail after the last synchronisation {us(tails)} us "
          f"(of which {int(np.median(nel))} Event.elapsed_time calls: {us(tel)} us); build_tree host {us(builds)} us")


if __name__ == "__main__":
    main()
