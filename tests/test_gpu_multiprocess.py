"""The multi-GPU path as real processes: W = 2 and 4 ranks launched through
``torch.distributed`` (gloo: collectives staged through the host, so no
rank's kernel ever waits on another's), all on cuda:0 -- the GPU box has one
GPU.  Each rank runs ``evaluate_partitioned`` (dual tree FP64/FP32, mutual,
treecode, listfmm; every result mode) and must reproduce the single-GPU
evaluation on its rows to 1e-12; the per-rank P2P pair counts must sum to
the single-GPU count exactly (src/traversal.py:19-26, :621-639: disjoint
target ownership)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = [("c2_32k", "fp64", "dualtree", "all"), ("plummer_32k", "fp32", "dualtree", "root"),
         ("c1", "fp64", "mutual", "local"), ("c1", "fp64", "treecode", "all"),
         ("c2_32k", "fp32", "listfmm", "root")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import paper_1209_3516_b200 as fb
    from goldens import Case
    from paper_1209_3516_b200 import distributed as fd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for name, precision, strategy, results in CASES:
            c = Case(name)
            pos = np.asarray(c.pos, np.float64)
            mutual = strategy == "mutual"
            cfg = fb.EvalConfig(strategy="dualtree" if mutual else strategy, mac=fb.MacConfig("fmm", c.theta),
                                p=c.p, precision=precision, mutual=mutual, task_grain=1500)
            ref = fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q), ncrit=c.ncrit)
            rrep = fb.evaluate_on_tree(ref, cfg)
            want = torch.stack([ref.d_phi, ref.d_fx, ref.d_fy, ref.d_fz]).cpu().numpy()
            t = fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q), ncrit=c.ncrit)
            rep = fd.evaluate_partitioned(t, cfg, rank, world, results=results)
            got = torch.stack([t.d_phi, t.d_fx, t.d_fy, t.d_fz]).cpu().numpy()
            lo, hi = t.owned_range
            err = max(float(np.linalg.norm(g[lo:hi] - w[lo:hi]) / max(np.linalg.norm(w[lo:hi]), 1e-300))
                      for g, w in zip(got, want))
            pairs = torch.tensor([rep.stats.p2p_pairs], dtype=torch.int64)
            dist.all_reduce(pairs)
            full = (lo, hi) == (0, t.n)
            out[(rank, name, strategy)] = (err, int(pairs.item()), int(rrep.stats.p2p_pairs), full,
                                           hi - lo, rep.total_time > 0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_processes_match_single_gpu(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    for name, precision, strategy, results in CASES:
        owned = 0
        for r in range(world):
            err, pairs, ref_pairs, full, nown, timed = out[(r, name, strategy)]
            assert err <= 1e-12, (name, strategy, r, err)
            assert pairs == ref_pairs, (name, strategy)
            assert timed
            want_full = results == "all" or (results == "root" and r == 0)
            assert full == want_full, (name, results, r)
            owned += nown if not full else 0
        if results == "local":  # the ranks' own rows tile the body set
            from goldens import Case
            assert owned == Case(name).n
