"""The NCCL code path on a one-GPU box: a ONE-rank NCCL communicator on
cuda:0 (NCCL refuses two ranks on one device, and the box has one GPU).
Every collective the multi-GPU paths issue -- the padded row all-gather and
gather of ``distributed.py`` (device tensors, ``all_gather_into_tensor``),
the MIN all-reduce, and ``sharded.py``'s size / variable all-gathers,
all-reduces and all-to-alls -- runs through the real NCCL backend with the
dtypes and stream usage of the product path, and the sharded build and
evaluation (world = 1: the rank's shard is the whole input) must reproduce
the single-GPU tree bit for bit and its results to 1e-12.  What this cannot
show is a transfer between two GPUs; the 2- and 4-rank runs of the same code
are in test_gpu_multiprocess.py / test_gpu_sharded.py (gloo)."""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CELLS = ("children", "parent", "level", "key", "start", "end", "sub_end", "leaf", "ctr", "bmax", "rmax", "lo",
         "hi")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _digest(t):
    return {k: hashlib.sha256(getattr(t, "d_" + k).contiguous().cpu().numpy().tobytes()).hexdigest()
            for k in CELLS + ("keys", "perm")}


def _worker(rank, port, out):
    import paper_1209_3516_b200 as fb
    from goldens import Case
    from paper_1209_3516_b200 import distributed as fd
    from paper_1209_3516_b200 import sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        assert dist.get_backend() == "nccl"
        # distributed.py: padded row exchanges on device tensors, from a side stream as the product issues them
        side = torch.cuda.Stream()
        for dtype in (torch.float64, torch.int32, torch.int64):
            full = (torch.arange(7 * 5, device=dev).reshape(7, 5) * 3).to(dtype)
            keep = full.clone()
            with torch.cuda.stream(side):
                fd.allgather_rows(full, [0, 7], 0, 1)
                fd.gather_rows(full, [0, 7], 0, 1)
            side.synchronize()
            assert torch.equal(full, keep)
        comm = fd.TorchDistComm()
        assert comm.all_true(True, 0, 1) and not comm.all_true(False, 0, 1)
        # sharded.py: its collectives one by one
        c = sharded._Comm(None, dev)
        assert c.nccl
        v = torch.tensor([3.0, -1.0], dtype=torch.float64, device=dev)
        assert torch.equal(c.all_reduce(v, dist.ReduceOp.MAX), v)
        assert c.all_gather_sizes(11, 1) == [11]
        keys = torch.arange(9, dtype=torch.int64, device=dev) * 1000003
        assert torch.equal(c.all_gather_var(keys, [9]), keys)
        rows = torch.rand((6, 4), dtype=torch.float64, device=dev)
        got, counts = c.all_to_all_var(rows, [6])
        assert counts == [6] and torch.equal(got, rows)
        empty, counts = c.all_to_all_var(rows[:0], [0])
        assert counts == [0] and empty.shape[0] == 0
        # the sharded build + evaluation end to end over the NCCL communicator
        for name, precision, mutual in (("c2_32k", "fp32", False), ("plummer_32k", "fp64", False),
                                        ("c1", "fp64", True)):
            cs = Case(name)
            pos, qq = np.asarray(cs.pos), np.asarray(cs.q)
            cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", cs.theta), p=cs.p, precision=precision, mutual=mutual,
                                task_grain=1500)
            ref = fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], qq), ncrit=cs.ncrit)
            rrep = fb.evaluate_on_tree(ref, cfg)
            want = ref.results_in_input_order()
            t = sharded.build_tree_sharded(pos[:, 0], pos[:, 1], pos[:, 2], qq, cs.ncrit, 0, 1)
            same = _digest(t) == _digest(ref)
            rep, res = sharded.evaluate_sharded(t, cfg)
            err = max(float(np.linalg.norm(g.cpu().numpy() - np.asarray(getattr(want, k))) /
                            max(np.linalg.norm(np.asarray(getattr(want, k))), 1e-300))
                      for g, k in zip(res, ("phi", "fx", "fy", "fz")))
            out[name] = (same, err, int(rep.stats.p2p_pairs), int(rrep.stats.p2p_pairs))
        out["ok"] = True
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_one_rank_nccl_communicator():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(_free_port(), out), nprocs=1, join=True, start_method="spawn")
    assert out.get("ok")
    for name in ("c2_32k", "plummer_32k", "c1"):
        same, err, pairs, ref_pairs = out[name]
        assert same, name
        assert err <= 1e-12, (name, err)
        assert pairs == ref_pairs, name
