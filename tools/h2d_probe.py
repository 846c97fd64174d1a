"""Host -> device staging of the C2 input (4 x 4 MB float32 arrays): the
current pinned-bounce copy, the same with the bounce copies on threads,
a direct pageable copy, and pinning the caller's pages in place."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_3516_b200 import workloads  # noqa: E402

pos, q = workloads.config2(1 << 20, 0)
arrs = [np.ascontiguousarray(pos[:, k]) for k in range(3)] + [np.ascontiguousarray(q)]
dev = torch.device("cuda", 0)
pool = ThreadPoolExecutor(4)


def bounce(a):
    h = torch.from_numpy(a)
    p = torch.empty(h.shape, dtype=h.dtype, pin_memory=True)
    p.copy_(h)
    return p.to(dev, non_blocking=True)


def serial():
    return [bounce(a) for a in arrs]


def threaded():
    return list(pool.map(bounce, arrs))


def pageable():
    return [torch.from_numpy(a).to(dev, non_blocking=True) for a in arrs]


def registered():
    cr = torch.cuda.cudart()
    out = []
    for a in arrs:
        cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        out.append(torch.from_numpy(a).to(dev, non_blocking=True))
    torch.cuda.synchronize()
    for a in arrs:
        cr.cudaHostUnregister(a.ctypes.data)
    return out


for name, fn in [("serial", serial), ("threaded", threaded), ("pageable", pageable), ("registered", registered)]:
    ts = []
    for it in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name:10s} median {1e3 * np.median(ts[2:]):.3f} ms  min {1e3 * min(ts[2:]):.3f} ms", flush=True)
