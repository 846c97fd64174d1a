"""Caching-allocator settling: new device segments per evaluation of the
same workload (two trees alive while the next builds, as in the bench loop).

    python tools/alloc_probe.py [C3]
"""
import os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1209_3516_b200 as fb
from paper_1209_3516_b200 import workloads
gen, n, solver = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
pos, q = gen(n, 0)
cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"], precision="fp32")
d = torch.as_tensor(pos, device="cuda")
ps = fb.ParticleSet(d[:, 0].contiguous(), d[:, 1].contiguous(), d[:, 2].contiguous(), torch.as_tensor(q, device="cuda"))
flush = torch.empty(2 * 126 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
def segs():
    return {(s["address"], s["total_size"]) for s in torch.cuda.memory_snapshot()}
prev = segs()
tree = None
for i in range(8):
    tree2 = fb.build_tree(ps, ncrit=solver["ncrit"])
    fb.evaluate_on_tree(tree2, cfg)
    tree = tree2
    torch.cuda.synchronize()
    now = segs()
    new = sorted(sz for _, sz in now - prev)
    print(i, "reserved MB", torch.cuda.memory_reserved() >> 20, "new segments MB", [x >> 20 for x in new])
    prev = now
