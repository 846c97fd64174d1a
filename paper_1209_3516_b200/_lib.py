"""ctypes binding of libfmm_b200.so (the C ABI declared in include/fmm_b200.h).

This is the only door to the compute path: there is no CPU fallback.  When
the library is missing or no CUDA device is visible the calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# FMM_B200_LIB selects an alternative in-tree build (kernel A/B experiments)
LIB_PATH = os.environ.get("FMM_B200_LIB") or os.path.join(HERE, "libfmm_b200.so")

FMM_OK, FMM_ERR_CAPACITY, FMM_ERR_MAX_DEPTH, FMM_ERR_INVALID, FMM_ERR_CUDA = range(5)
DTYPE_F64, DTYPE_F32 = 0, 1
PREC_FP64, PREC_FP32, PREC_FP32_ANCHORED, PREC_FP32_ACC64 = 0, 1, 2, 3

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
INT = C.c_int
DBL = C.c_double
SZ = C.c_size_t

# name -> argtypes (every function returns int status, except where noted)
SIGNATURES = {
    "fmm_abi_version": [],
    "fmm_last_error": [],
    "fmm_launch_count": [],
    "fmm_device_sm_count": [],
    "fmm_workspace_bytes": [I64, P],
    "fmm_ingest_bounds": [P, P, P, P, INT, I64, P, P, P, P, P, P, SZ, P],
    "fmm_morton_keys": [P, P, P, I64, P, P, P, P],
    "fmm_sort_pairs_u64": [P, P, P, P, I64, INT, P, SZ, P],
    "fmm_permute_bodies": [P, P, P, P, P, I64, P, P, P, P, P, P, P, P],
    "fmm_carve_count": [P, I64, I32, INT, P, P, P, P, P, P, P, SZ, P],
    "fmm_carve_emit": [P, I64, P, P, I32, P, P, P, P, P, P, P, P, P, P, P, P, SZ, P],
    "fmm_cell_geometry": [I32, P, P, P, P, P, P, P, P, INT, INT, P, P, P, P, P, P, P, SZ, P],
    "fmm_cell_bmax_range": [I32, P, P, P, P, P, P, I32, I32, P, P, SZ, P],
    "fmm_upward": [INT, I32, P, P, P, P, P, P, P, P, P, P, P, INT, P, P],
    "fmm_downward": [INT, I32, P, P, P, P, P, INT, I64, I64, P, P, P, P, P, P, P, P, P, P],
    "fmm_traverse_step": [P, P, I64, INT, P, P, P, P, P, P, P, P, P, P, P, P, I32, I32, INT, INT, DBL, P, P, I64,
                          P, P, I64, P, P, I64, P, P],
    "fmm_traverse": [P, P, P, P, I64, INT, P, P, P, P, P, P, P, P, P, P, P, P, I32, I32, P, INT, INT, DBL, P, P, I64,
                     P, P, I64, P, P],
    "fmm_pairs_to_rows": [P, P, P, I64, I32, I32, INT, P, P, P, SZ, P],
    "fmm_partition_plan": [I32, I64, INT, INT, P, P, P, P, P, P, P, P, P, SZ, P],
    "fmm_partition_owner": [I32, P, P, P, P, I64, P, P],
    "fmm_traverse_mutual": [P, P, P, P, I64, INT, P, P, P, P, P, P, P, P, I32, I32, INT, DBL, P, P, I64, P, P, I64,
                            P, P],
    "fmm_traverse_mutual_sym": [P, P, P, P, I64, INT, P, P, P, P, P, P, P, P, I32, I32, INT, DBL, P, P, I64, P, P,
                                I64, P, P, P, I64, P, P, I64, P, P],
    "fmm_treecode_traverse": [P, P, P, P, I64, INT, I32, P, P, P, P, P, P, P, P, P, P, P, P, I32, I32, INT, DBL, P, P,
                              I64, P, P, I64, P, P, SZ, P],
    "fmm_listfmm_lists": [I32, INT, P, P, P, P, P, P, P, P, P, I32, I32, P, P, I64, P, P, I64, P, P, SZ, P],
    "fmm_pairs_to_csr": [P, P, I64, I32, P, P, P, SZ, P],
    "fmm_p2p_plan": [I32, P, P, P, I32, I32, P, P, P, P, P, P, P, P, I32, P, P, I32, P, P, P, I64, P, P, P, P, P,
                     SZ, P],
    "fmm_sort_rows": [I32, P, P, P, P, SZ, P],
    "fmm_m2l_csr": [INT, I32, P, P, P, P, P, P, P],
    "fmm_m2l_grouped_bytes": [INT, I32, I64, P],
    "fmm_m2l_grouped": [INT, I32, P, P, I64, P, P, P, P, P, P, P, SZ, P],
    "fmm_m2p_csr": [INT, INT, I32, P, P, P, P, P, P, P, P, P, P, P, P, P, P],
    "fmm_p2p": [INT, INT, INT, INT, I32, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P],
    "fmm_p2p_sym": [INT, I32, I32, I32, P, P, P, P, P, I64, P, P, P, P, P, P, P, P, P],
    "fmm_m2l_sym": [INT, I32, I32, I32, P, P, P, P, I64, P, P, P, P, P],
    "fmm_pack_bodies_f64": [I64, P, P, P, P, P, P],
    "fmm_p2p_coincident": [I32, P, P, P, P, P, P, P, P, P, P, P],
    "fmm_unpermute": [P, I64, P, P, P, P, P, P, P, P, P],
    "fmm_combine": [I64, P, P, P, P, P, P, P, P, P],
    "fmm_direct": [I64, P, P, P, P, I64, P, P, P, P, P, P],
    "fmm_ffma_probe": [INT, INT, INT, P, P, P],
}

_lib = None
_lock = threading.Lock()


class FmmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class CapacityError(FmmError):
    pass


def load():
    """Load (not build) the library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1209_3516_b200._build` "
                    "(the B200 path has no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, argt in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argt
                fn.restype = {"fmm_last_error": C.c_char_p, "fmm_launch_count": C.c_longlong}.get(name, C.c_int)
            if lib.fmm_abi_version() != 1:
                raise RuntimeError("libfmm_b200.so ABI mismatch")
            _lib = lib
    return _lib


def launch_count() -> int:
    """Kernels launched by libfmm_b200.so so far (its own, not CUB's)."""
    return int(load().fmm_launch_count())


def exported_symbols():
    return sorted(SIGNATURES)


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 FMM path needs a CUDA device (no CPU fallback)")


def call(name: str, *args):
    """Invoke ``name``; raise FmmError / CapacityError on a non-zero status."""
    lib = load()
    st = getattr(lib, name)(*args)
    if st == FMM_OK:
        return
    msg = lib.fmm_last_error().decode(errors="replace")
    if st == FMM_ERR_CAPACITY:
        raise CapacityError(st, msg)
    if st in (FMM_ERR_MAX_DEPTH, FMM_ERR_INVALID):
        raise ValueError(msg)
    raise FmmError(st, f"{name}: {msg}")


def ptr(t) -> int:
    """Device pointer of a tensor (0 for None)."""
    return 0 if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ---------------------------------------------------------------------------
# workspace cache (caller-owned scratch for the C ABI)
# ---------------------------------------------------------------------------
_ws = {}


def workspace(items: int, device, slot: int = 0, stream=None) -> tuple[int, int]:
    """(pointer, bytes) of a scratch buffer valid for ``items`` elements
    (``slot`` separates buffers used concurrently on different streams; with
    ``stream`` (a torch stream other than the allocating one) the buffer is
    recorded on it, so a later reallocation cannot recycle it under that
    stream's pending work)."""
    need = C.c_size_t(0)
    call("fmm_workspace_bytes", int(max(items, 1)), C.byref(need))
    key = (torch.device(device).index or 0, threading.get_ident(), slot)  # per thread: calls may overlap
    buf = _ws.get(key)
    if buf is None or buf.numel() < need.value:
        _ws[key] = None
        buf = torch.empty(int(need.value * 1.25) + 4096, dtype=torch.uint8, device=device)
        _ws[key] = buf
    if stream is not None:
        buf.record_stream(stream)
    return buf.data_ptr(), buf.numel()
