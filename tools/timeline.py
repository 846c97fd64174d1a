"""Kernel timeline of one bench step (build_tree + evaluate_on_tree) from
torch.profiler (CUPTI): every kernel / memcpy / memset with its stream,
start and duration, plus the idle gaps of the GPU on the critical path.

    python tools/timeline.py --config C2 [--mutual] > gpurun_out/timeline.txt
"""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1209_3516_b200 as fb  # noqa: E402
from paper_1209_3516_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--mutual", action="store_true")
    ap.add_argument("--gap-us", type=float, default=8.0)
    args = ap.parse_args()
    gen, n, solver = workloads.CONFIGS[args.config]
    pos, q = gen(n, 0)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision=args.precision,
                        mutual=args.mutual)
    dpos = torch.as_tensor(pos, device="cuda")
    ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                        torch.as_tensor(q, device="cuda"))

    def step():
        t = fb.build_tree(ps, ncrit=solver["ncrit"])
        fb.evaluate_on_tree(t, cfg)

    for _ in range(4):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        step()
        torch.cuda.synchronize()
    ev = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            ev.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", -1), e.name))
    ev.sort()
    t0 = ev[0][0]
    print(f"{len(ev)} device events, span {(ev[-1][1] - t0):.1f} us")
    busy_end = t0
    idle = 0.0
    for s, e, st, name in ev:
        gap = s - busy_end
        mark = ""
        if gap > args.gap_us:
            idle += gap
            mark = f"   <-- idle {gap:.1f} us"
        print(f"{s - t0:9.1f} {e - s:9.1f}  s{st:<3} {name[:90]}{mark}")
        busy_end = max(busy_end, e)
    print(f"idle (gaps > {args.gap_us} us): {idle:.1f} us of {(ev[-1][1] - t0):.1f} us")
    by = {}
    for s, e, st, name in ev:
        by.setdefault(name[:60], [0, 0.0])
        by[name[:60]][0] += 1
        by[name[:60]][1] += e - s
    for k, (c, d) in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"{d:9.1f} us {c:4d}  {k}")
    _ = np


if __name__ == "__main__":
    main()
