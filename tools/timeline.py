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
    ap.add_argument("--world", type=int, default=1, help="time rank --rank of a W-rank partitioned evaluation "
                    "(exchanges as no-ops, tools/rank_probe.py)")
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--gap-us", type=float, default=8.0)
    ap.add_argument("--host", action="store_true", help="interleave host events: every C-ABI call (call:NAME) "
                    "and Python phase (py:NAME) with the device kernels")
    args = ap.parse_args()
    if args.host:
        _instrument()
    gen, n, solver = workloads.CONFIGS[args.config]
    pos, q = gen(n, 0)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision=args.precision,
                        mutual=args.mutual)
    dpos = torch.as_tensor(pos, device="cuda")
    ps = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                        torch.as_tensor(q, device="cuda"))

    def step():
        t = fb.build_tree(ps, ncrit=solver["ncrit"])
        if args.world > 1:
            from paper_1209_3516_b200 import distributed as fd
            sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
            from rank_probe_comm import NoComm
            fd.evaluate_partitioned(t, cfg, args.rank, args.world, comm=NoComm(), results="root")
        else:
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
    if args.host:
        _print_host(prof, ev)
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


def _instrument():
    """Wrap the C-ABI entry and the Python phases in profiler ranges."""
    from torch.profiler import record_function

    from paper_1209_3516_b200 import _lib, traversal, tree

    def wrap(mod, name, label):
        f = getattr(mod, name)

        def g(*a, **k):
            with record_function(label(a)):
                return f(*a, **k)
        setattr(mod, name, g)

    wrap(_lib, "call", lambda a: "call:" + a[0])
    for n in ("interaction_lists", "run_m2l", "run_p2p", "upward_pass", "downward_pass", "evaluate_dual_tree"):
        if hasattr(traversal, n):
            wrap(traversal, n, lambda a, n=n: "py:" + n)
    wrap(tree, "build_tree", lambda a: "py:build_tree")
    fb.build_tree = tree.build_tree
    fb.evaluate_dual_tree = traversal.evaluate_dual_tree


def _print_host(prof, dev_ev):
    """Host ranges (call:/py:, torch ops, syncs) beside device kernels, in
    time order up to the first P2P kernel."""
    host = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CPU:
            nm = e.name
            if nm.startswith(("call:", "py:", "aten::zeros", "aten::empty", "cudaStreamSynchronize",
                              "cudaEventSynchronize", "cudaMemcpy", "aten::item", "aten::_local_scalar")):
                host.append((e.time_range.start, e.time_range.end, nm))
    t0 = min(x[0] for x in dev_ev + host)
    stop = next((s for s, _, _, n in sorted(dev_ev) if "p2p_f" in n), None)
    rows = [(s, e, "H", n) for s, e, n in host] + [(s, e, "D", n) for s, e, _, n in dev_ev]
    rows.sort()
    print("---- host (H) and device (D) events up to the first P2P kernel ----")
    for s, e, k, n in rows:
        if stop is not None and s > stop:
            break
        print(f"{k} {s - t0:9.1f} {e - s:8.1f}  {n[:80]}")
    print("----")


if __name__ == "__main__":
    main()
