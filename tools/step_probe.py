"""Step-time probe for host-side effects: CUDA-event time of build_tree +
evaluate_on_tree (bench-style, L2 flushed outside the bracket) with the
caching allocator's segment counters, optionally with the cyclic GC off.

    python tools/step_probe.py [--config C2] [--nogc] [--steps 20]
"""
import argparse
import gc
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--nogc", action="store_true")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--strategy", default="dualtree")
ap.add_argument("--mutual", action="store_true")
ap.add_argument("--all", action="store_true", help="print every step time")
ap.add_argument("--warmup", type=int, default=4)
args = ap.parse_args()
gen, n, solver = workloads.CONFIGS[args.config]
pos, q = gen(n, 0)
cfg = fb.EvalConfig(strategy=args.strategy, mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision="fp32",
                    mutual=args.mutual)
dpos = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                    torch.as_tensor(q, device="cuda"))
flush = torch.empty(2 * 126 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def step():
    t = fb.build_tree(ps, ncrit=solver["ncrit"])
    fb.evaluate_on_tree(t, cfg)
    return t


tree = None
for _ in range(args.warmup):
    tree = step()
torch.cuda.synchronize()
if args.nogc:
    gc.collect()
    gc.disable()
s0 = torch.cuda.memory_stats()
ts, pre, p2p, post = [], [], [], []
for _ in range(args.steps):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tree = step()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
    if args.strategy == "dualtree":
        ev0, pev, eend = fb.traversal.last_events
        pre.append(e0.elapsed_time(pev[0][0]))
        p2p.append(pev[0][0].elapsed_time(pev[-1][1]))
        post.append(pev[-1][1].elapsed_time(e1))
s1 = torch.cuda.memory_stats()
d = {k: s1[k] - s0.get(k, 0) for k in ("segment.all.allocated", "num_alloc_retries", "num_device_alloc")
     if k in s1}
print(f"{args.config} nogc={args.nogc} ms/step median {np.median(ts):.3f} mean {np.mean(ts):.3f} "
      f"min {np.min(ts):.3f} allocator deltas {d}")
if args.all:
    print("  steps:", " ".join(f"{t:.2f}" for t in ts))
if pre:
  print(f"  step start -> P2P start {np.median(pre):.3f} ms, P2P {np.median(p2p):.3f} ms, P2P end -> step end "
      f"{np.median(post):.3f} ms")
