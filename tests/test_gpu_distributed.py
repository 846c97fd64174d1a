"""Multi-GPU evaluation path on one device: W ranks emulated as host
threads, each with its own tree, exchanging through a host-side all-gather
(no kernel ever waits on another rank's kernel).  The partitioned result
must equal the single-GPU result, and the per-rank P2P/M2L work must add up
to the single-GPU lists (P2P rows are never shared)."""

import threading

import numpy as np
import pytest
import torch

import paper_1209_3516_b200 as fb
from goldens import Case
from paper_1209_3516_b200 import distributed as fd

pytestmark = pytest.mark.gpu


class ThreadComm:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.bufs = [None] * world

    def allgather_rows(self, full, chunks, rank, world):
        torch.cuda.current_stream().synchronize()
        self.bufs[rank] = full[int(chunks[rank]):int(chunks[rank + 1])].clone()
        torch.cuda.current_stream().synchronize()
        self.barrier.wait()
        for r in range(world):
            full[int(chunks[r]):int(chunks[r + 1])].copy_(self.bufs[r])
        torch.cuda.current_stream().synchronize()
        self.barrier.wait()

    def all_true(self, ok, rank, world):
        self.bufs[rank] = bool(ok)
        self.barrier.wait()
        res = all(self.bufs[r] for r in range(world))
        self.barrier.wait()
        return res

    def gather_rows(self, full, chunks, rank, world, root=0):
        torch.cuda.current_stream().synchronize()
        self.bufs[rank] = full[int(chunks[rank]):int(chunks[rank + 1])].clone()
        torch.cuda.current_stream().synchronize()
        self.barrier.wait()
        if rank == root:
            for r in range(world):
                full[int(chunks[r]):int(chunks[r + 1])].copy_(self.bufs[r])
            torch.cuda.current_stream().synchronize()
        self.barrier.wait()


def _ps(c):
    pos = np.asarray(c.pos, np.float64)
    return fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q)


@pytest.mark.parametrize("name,world,precision,strategy", [
    ("c2_32k", 2, "fp64", "dualtree"), ("plummer_32k", 4, "fp64", "dualtree"), ("c1", 3, "fp64", "dualtree"),
    ("c2_32k", 8, "fp32", "dualtree"), ("c1", 3, "fp64", "treecode"), ("c2_32k", 4, "fp32", "treecode"),
    ("c1", 2, "fp64", "listfmm"), ("plummer_32k", 4, "fp64", "listfmm"), ("c1", 3, "fp64", "mutual"),
    ("c2_32k", 4, "fp32", "mutual")])
def test_partitioned_equals_single(name, world, precision, strategy):
    c = Case(name)
    mutual = strategy == "mutual"
    cfg = fb.EvalConfig(strategy="dualtree" if mutual else strategy, mac=fb.MacConfig("fmm", c.theta), p=c.p,
                        precision=precision, mutual=mutual, task_grain=1500)
    ref_tree = fb.build_tree(_ps(c), ncrit=c.ncrit)
    ref = fb.evaluate_on_tree(ref_tree, cfg)
    want = [a.clone() for a in (ref_tree.d_phi, ref_tree.d_fx, ref_tree.d_fy, ref_tree.d_fz)]
    comm = ThreadComm(world)
    trees = [fb.build_tree(_ps(c), ncrit=c.ncrit) for _ in range(world)]
    reps = [None] * world
    errs = []

    def run(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                reps[r] = fd.evaluate_partitioned(trees[r], cfg, r, world, comm=comm)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            comm.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert sum(rp.stats.p2p_pairs for rp in reps) == ref.stats.p2p_pairs
    assert sum(rp.stats.p2p_skipped for rp in reps) == ref.stats.p2p_skipped
    assert sum(rp.stats.m2l_calls for rp in reps) >= ref.stats.m2l_calls  # shared top rows repeat
    assert sum(rp.stats.m2p_calls for rp in reps) == ref.stats.m2p_calls  # leaf targets: never shared
    for r in range(world):
        got = (trees[r].d_phi, trees[r].d_fx, trees[r].d_fy, trees[r].d_fz)
        for g, w in zip(got, want):
            rel = float(torch.linalg.norm(g - w) / torch.linalg.norm(w))
            assert rel <= 1e-12, (r, rel)


def _run_ranks(cfg, trees, comm, world):
    reps, errs = [None] * world, []

    def run(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                reps[r] = fd.evaluate_partitioned(trees[r], cfg, r, world, comm=comm)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            comm.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    return reps


@pytest.mark.parametrize("mutual", [False, True])
def test_partitioned_redo_when_one_rank_overflows(mutual):
    """Hinted (deferred) lists: when one rank's lists outgrow its capacity
    hint, every rank redoes the step (comm.all_true) and the result is
    exact."""
    from paper_1209_3516_b200 import traversal as trv
    c = Case("c2_32k")
    world = 3
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", c.theta), p=c.p, precision="fp64", mutual=mutual, task_grain=1500)
    ref_tree = fb.build_tree(_ps(c), ncrit=c.ncrit)
    ref = fb.evaluate_on_tree(ref_tree, cfg)
    want = [a.clone() for a in (ref_tree.d_phi, ref_tree.d_fx, ref_tree.d_fy, ref_tree.d_fz)]
    comm = ThreadComm(world)
    trees = [fb.build_tree(_ps(c), ncrit=c.ncrit) for _ in range(world)]
    _run_ranks(cfg, trees, comm, world)  # leaves capacity hints behind
    lo1, hi1 = (int(x) for x in trees[1]._dist_plan.cuts[1:3])
    shrunk = 0
    for k in list(trv._hint):
        # rank 1's keys carry its body range (lo, hi): shrink only those
        rng = k[5:7] if k[0] == "mutual" else k[4:6]
        if tuple(rng) == (lo1, hi1):
            trv._hint[k] = (64, 64, 64)
            shrunk += 1
    assert shrunk
    trees = [fb.build_tree(_ps(c), ncrit=c.ncrit) for _ in range(world)]
    reps = _run_ranks(cfg, trees, comm, world)
    assert sum(rp.stats.p2p_pairs for rp in reps) == ref.stats.p2p_pairs
    for r in range(world):
        got = (trees[r].d_phi, trees[r].d_fx, trees[r].d_fy, trees[r].d_fz)
        for g, w in zip(got, want):
            assert float(torch.linalg.norm(g - w) / torch.linalg.norm(w)) <= 1e-12


@pytest.mark.parametrize("world", [2, 3, 8])
def test_device_plan_matches_host_rules(world):
    """The per-step device plan equals the host functions' cuts, chunks,
    shared top and owned cells (fd.body_cuts / cell_chunks / shared_cells)."""
    c = Case("plummer_32k")
    t = fb.build_tree(_ps(c), ncrit=c.ncrit)
    leaf = t.cell_leaf
    cuts = fd.body_cuts(t.cell_start[leaf], t.cell_end[leaf], t.n, world)
    chunks = fd.cell_chunks(t.cell_start, cuts)
    shared = fd.shared_cells(t.cell_start, t.cell_end, cuts)
    for rank in range(world):
        plan = fd._Plan(t, world, rank)
        assert np.array_equal(plan.cuts, cuts) and np.array_equal(plan.chunks, chunks)
        lo, hi = cuts[rank], cuts[rank + 1]
        own = np.flatnonzero((t.cell_start >= lo) & (t.cell_end <= hi))
        ids, off = plan.owned
        assert sorted(ids.cpu().tolist()) == own.tolist() and off[-1] == own.size
        tids, toff = plan.top
        assert sorted(tids.cpu().tolist()) == np.flatnonzero(shared).tolist() and toff[-1] == shared.sum()
        lev = t.cell_level[ids.cpu().numpy()]
        assert np.all(np.diff(lev) >= 0)  # grouped by level, as fmm_upward needs
