"""FP32 pipe probes (see fmm_ffma_probe in include/fmm_b200.h)."""
import ctypes as C, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1209_3516_b200 import _lib
sink = torch.zeros(148 * 64, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
names = {0: "ffma_imm", 1: "ffma2_imm", 2: "ffma_reg", 3: "ffma2_reg", 4: "fmul_fadd_reg", 5: "p2p_mix", 6: "p2p_mix_nomufu", 7: "p2p_mix_packed"}
out = {}
for mode, nm in names.items():
    for blocks in (148 * 8, 148 * 16):
        fl = C.c_double(0)
        iters = 4096 if mode < 5 else 2048
        for _ in range(2):
            _lib.call("fmm_ffma_probe", mode, blocks, iters, _lib.ptr(sink), C.byref(fl), st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            _lib.call("fmm_ffma_probe", mode, blocks, iters, _lib.ptr(sink), C.byref(fl), st)
        e1.record(); e1.synchronize()
        out[f"{nm}@{blocks}"] = 5 * fl.value / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(json.dumps(out))
