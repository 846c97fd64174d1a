"""Multi-GPU partition logic on CPU: cut points, cell chunks, the shared
top, and the padded all-gather exchange over torch.distributed (gloo,
world_size 2, real processes)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from goldens import Case
from oracle import oracle as orc
from paper_1209_3516_b200 import distributed as fd


def _tree(name="c2_32k"):
    c = Case(name)
    return c, orc.build_tree(c.pos, c.q, c.ncrit, c.allow)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_cuts_on_leaf_boundaries_and_balanced(world):
    c, t = _tree()
    leaf = t.cell_leaf.astype(bool)
    cuts = fd.body_cuts(t.cell_start[leaf], t.cell_end[leaf], t.n, world)
    assert cuts[0] == 0 and cuts[-1] == t.n and np.all(np.diff(cuts) > 0)
    starts = set(t.cell_start[leaf].tolist()) | {t.n}
    assert all(int(x) in starts for x in cuts)
    share = np.diff(cuts) / t.n
    assert share.max() <= 1.0 / world + 64 / t.n  # within one leaf of equal
    # every leaf belongs to exactly one rank
    owner = np.searchsorted(cuts, t.cell_start[leaf], side="right") - 1
    assert np.all(t.cell_end[leaf] <= cuts[owner + 1])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_chunks_and_shared_top(world):
    c, t = _tree("plummer_32k")
    leaf = t.cell_leaf.astype(bool)
    cuts = fd.body_cuts(t.cell_start[leaf], t.cell_end[leaf], t.n, world)
    ch = fd.cell_chunks(t.cell_start, cuts)
    assert ch[0] == 0 and ch[-1] == t.ncells and np.all(np.diff(ch) >= 0)
    shared = fd.shared_cells(t.cell_start, t.cell_end, cuts)
    assert not np.any(shared[leaf])               # cuts never split a leaf
    assert shared[0] or world == 1                 # the root straddles every cut
    # every non-shared cell lies inside exactly one rank's body range
    for cidx in np.flatnonzero(~shared):
        r = np.searchsorted(cuts, t.cell_start[cidx], side="right") - 1
        assert t.cell_end[cidx] <= cuts[r + 1]
    # shared cells are ancestors-only: their parents are shared too
    par = t.cell_parent[shared]
    assert np.all(shared[par[par >= 0]])


def test_target_filter_union_equals_full_list():
    """Per-rank traversal restricted to the rank's targets (the oracle's
    pair sets filtered the way csrc/traverse.cu filters) unions to the
    single-GPU list, and P2P rows are never shared."""
    c, t = _tree()
    mt, ms, pt, ps = orc.collect_lists(t, c.theta)
    leaf = t.cell_leaf.astype(bool)
    world = 4
    cuts = fd.body_cuts(t.cell_start[leaf], t.cell_end[leaf], t.n, world)
    m_union, p_union, p_total = set(), set(), 0
    for r in range(world):
        lo, hi = cuts[r], cuts[r + 1]
        keep_m = (t.cell_end[mt] > lo) & (t.cell_start[mt] < hi)
        keep_p = (t.cell_end[pt] > lo) & (t.cell_start[pt] < hi)
        m_union |= set(zip(mt[keep_m].tolist(), ms[keep_m].tolist()))
        p_union |= set(zip(pt[keep_p].tolist(), ps[keep_p].tolist()))
        p_total += int(keep_p.sum())
    assert m_union == set(zip(mt.tolist(), ms.tolist()))
    assert p_union == set(zip(pt.tolist(), ps.tolist()))
    assert p_total == pt.size  # no P2P row on two ranks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ncells, nc = 37, 5
        chunks = np.array([0, 11, 11, 37][: world + 1]) if world == 3 else np.array([0, 16, 37])
        full = torch.full((ncells, nc), -1.0, dtype=torch.float64)
        lo, hi = int(chunks[rank]), int(chunks[rank + 1])
        full[lo:hi] = torch.arange(lo * nc, hi * nc, dtype=torch.float64).reshape(-1, nc)
        mine = full.clone()
        fd.allgather_rows(full, chunks, rank, world)
        out[rank] = full.numpy().tolist()
        fd.gather_rows(mine, chunks, rank, world, root=0)
        out[(rank, "gather")] = mine.numpy().tolist()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allgather_rows_gloo(world):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    want = np.arange(37 * 5, dtype=np.float64).reshape(37, 5)
    for r in range(world):
        assert np.array_equal(np.array(out[r]), want)
    assert np.array_equal(np.array(out[(0, "gather")]), want)  # only the root receives
    for r in range(1, world):
        assert (np.array(out[(r, "gather")]) == -1.0).sum() > 0


def test_sharded_host_logic():
    from paper_1209_3516_b200.sharded import halo_ranges, owner_of, shard_offsets
    assert shard_offsets([3, 0, 5]).tolist() == [0, 3, 3, 8]
    assert owner_of([0, 2, 3, 7], [0, 3, 3, 8]).tolist() == [0, 0, 2, 2]
    cuts = [0, 10, 20, 30]
    # own range [10, 20): runs inside it vanish, the rest merge and split at the cuts
    out = halo_ranges([12, 5, 8, 18, 25, 28, 0], [15, 9, 12, 24, 27, 29, 0], 10, 20, cuts)
    assert out[0].tolist() == [[5, 10]]
    assert out[1].tolist() == []
    assert out[2].tolist() == [[20, 24], [25, 27], [28, 29]]
    # a run crossing two foreign ranges is split per owner
    out = halo_ranges([5], [25], 30, 30, cuts)
    assert [o.tolist() for o in out] == [[[5, 10]], [[10, 20]], [[20, 25]]]
    assert all(o.size == 0 for o in halo_ranges([], [], 0, 10, cuts))
