"""Multi-GPU evaluation: Morton-partitioned targets, NCCL all-gather of
multipoles.

One process per GPU (``torch.distributed``, backend "nccl" on the B200
box, "gloo" in the CPU tests).  Every rank holds the full input and builds
the identical tree (the build is deterministic and bit-exact, ~1 ms at
N=2^20), then:

1. **Partition.**  The leaves, in pre-order (= Morton order), are cut into
   ``world`` contiguous ranges of ~N/world bodies; cuts fall on leaf
   boundaries, so P2P rows are never shared.  Rank r owns bodies
   ``[cut[r], cut[r+1])``, every cell whose body range lies inside that
   range, and the pre-order cell chunk ``[c_lo, c_hi)`` of cells that START
   inside it.  Cells straddling a cut (the tree top) are shared.
2. **Upward.**  Each rank runs P2M/M2M on the cells it owns, the chunks are
   all-gathered (one ``all_gather_into_tensor`` of padded chunks over
   NVLink), and the shared top cells are rebuilt redundantly by M2M.
3. **Traversal.**  Each rank runs the dual traversal from (root, root) but
   keeps only pairs whose target meets its body range
   (csrc/traverse.cu); the union over ranks is the single-GPU list (shared
   top cells' M2L rows appear on several ranks and are computed
   redundantly and identically).
4. **Near/far field.**  M2L, P2P and L2P for the rank's targets; L2L runs
   on all cells (cheap, redundant).
5. **Results.**  One all-gather of (phi, fx, fy, fz) chunks, so every rank
   ends with the full Morton-ordered result.

Host helpers here are pure NumPy/torch so the partition and exchange logic
is tested on CPU with ``gloo`` (tests/test_distributed.py).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["body_cuts", "cell_chunks", "shared_cells", "allgather_rows", "TorchDistComm",
           "evaluate_partitioned"]


def body_cuts(leaf_start: np.ndarray, leaf_end: np.ndarray, n: int, world: int) -> np.ndarray:
    """Cut points ``cuts[0]=0 < ... < cuts[world]=n`` on leaf boundaries,
    closest to the equal split ``r * n / world`` (leaves in Morton order)."""
    bounds = np.concatenate([np.sort(np.asarray(leaf_start, np.int64)), [n]])
    cuts = [0]
    for r in range(1, world):
        target = r * n / world
        k = int(np.searchsorted(bounds, target))
        cand = [bounds[max(0, k - 1)], bounds[min(len(bounds) - 1, k)]]
        c = int(min(cand, key=lambda v: abs(v - target)))
        c = max(c, cuts[-1])
        cuts.append(c)
    cuts.append(n)
    return np.asarray(cuts, np.int64)


def cell_chunks(cell_start: np.ndarray, cuts: np.ndarray) -> np.ndarray:
    """Pre-order cell chunk boundaries: rank r's chunk is
    ``[chunks[r], chunks[r+1])``, the cells whose first body lies in its
    range (``cell_start`` is non-decreasing in pre-order)."""
    return np.searchsorted(np.asarray(cell_start, np.int64), cuts, side="left").astype(np.int64)


def shared_cells(cell_start: np.ndarray, cell_end: np.ndarray, cuts: np.ndarray) -> np.ndarray:
    """Boolean mask of cells straddling an interior cut (the shared top)."""
    s = np.asarray(cell_start, np.int64)
    e = np.asarray(cell_end, np.int64)
    m = np.zeros(s.shape, bool)
    for c in cuts[1:-1]:
        m |= (s < c) & (e > c)
    return m


def allgather_rows(full: torch.Tensor, chunks, rank: int, world: int, group=None) -> None:
    """Replace ``full[chunks[r]:chunks[r+1]]`` with rank r's rows, for every r
    (one padded all-gather; works with NCCL on GPU and gloo on CPU)."""
    sizes = [int(chunks[r + 1] - chunks[r]) for r in range(world)]
    width = int(np.prod(full.shape[1:])) if full.dim() > 1 else 1
    rows = max(max(sizes), 1)
    send = torch.zeros((rows, width), dtype=full.dtype, device=full.device)
    mine = full[int(chunks[rank]):int(chunks[rank + 1])].reshape(-1, width)
    send[:mine.shape[0]].copy_(mine)
    recv = torch.empty((world * rows, width), dtype=full.dtype, device=full.device)
    if hasattr(dist, "all_gather_into_tensor") and full.is_cuda:
        dist.all_gather_into_tensor(recv, send, group=group)
    else:
        parts = list(recv.split(rows))
        dist.all_gather(parts, send, group=group)
    for r in range(world):
        if sizes[r]:
            full[int(chunks[r]):int(chunks[r + 1])].reshape(-1, width).copy_(recv[r * rows:r * rows + sizes[r]])


class _Plan:
    """Per-tree partition plan (host arrays + device cell lists)."""

    def __init__(self, tree, world: int):
        from .tree import Tree  # noqa: F401
        leaf = tree.cell_leaf
        start, end, level = tree.cell_start, tree.cell_end, tree.cell_level
        self.cuts = body_cuts(start[leaf], end[leaf], tree.n, world)
        self.chunks = cell_chunks(start, self.cuts)
        self.shared = shared_cells(start, end, self.cuts)
        bfs = tree.d_cells_by_level.cpu().numpy()  # pre-order ids grouped by level
        nlev = len(tree.level_off) - 1
        self.owned = []
        for r in range(world):
            lo, hi = self.cuts[r], self.cuts[r + 1]
            own = (start >= lo) & (end <= hi)
            self.owned.append(self._by_level(bfs, own, tree.level_off, nlev, tree.device))
        self.top = self._by_level(bfs, self.shared, tree.level_off, nlev, tree.device)

    @staticmethod
    def _by_level(bfs, mask, level_off, nlev, dev):
        ids, off = [], [0]
        for L in range(nlev):
            seg = bfs[level_off[L]:level_off[L + 1]]
            sel = seg[mask[seg]]
            ids.append(sel)
            off.append(off[-1] + sel.size)
        arr = np.concatenate(ids).astype(np.int32) if ids else np.zeros(0, np.int32)
        return torch.as_tensor(arr, device=dev), off


def _upward_cells(tree, p, cells, off, M):
    import ctypes as C
    from . import _lib
    P = _lib.ptr
    offc = (C.c_int32 * len(off))(*off)
    _lib.call("fmm_upward", p, tree.ncells, P(tree.d_children), P(tree.d_start), P(tree.d_end), P(tree.d_leaf),
              P(tree.d_ctr), P(tree.d_x), P(tree.d_y), P(tree.d_z), P(tree.d_q), P(cells), offc, len(off) - 1,
              P(M), _lib.stream_handle())


class TorchDistComm:
    """Exchange through ``torch.distributed`` (NCCL over NVLink on the box)."""

    def __init__(self, group=None):
        self.group = group

    def allgather_rows(self, full, chunks, rank, world):
        allgather_rows(full, chunks, rank, world, self.group)


def evaluate_partitioned(tree, cfg, rank: int, world: int, group=None, comm=None):
    """Evaluate ``tree`` with targets Morton-partitioned over ``world`` ranks.

    Every rank returns the same full results in ``tree`` (after the final
    all-gather) and an ``EvalReport`` whose counters cover its own rows.
    ``comm`` defaults to :class:`TorchDistComm`; tests pass an in-process
    exchange to emulate ranks on one device."""
    comm = comm or TorchDistComm(group)
    from . import _lib
    from .kernels import KernelStats, ncoef
    from .traversal import (EvalReport, interaction_lists, listfmm_lists, run_m2l, run_m2p, run_p2p,
                            treecode_lists)
    from .tree import downward_pass

    if world == 1:
        from .traversal import evaluate_on_tree
        return evaluate_on_tree(tree, cfg)
    treecode = cfg.strategy == "treecode"
    if cfg.mutual and cfg.strategy == "dualtree":
        raise NotImplementedError("mutual traversal is outside the B200 hot path")
    plan = getattr(tree, "_dist_plan", None)
    if plan is None or len(plan.cuts) != world + 1:
        plan = _Plan(tree, world)
        tree._dist_plan = plan
    lo, hi = int(plan.cuts[rank]), int(plan.cuts[rank + 1])
    dev = tree.device
    stats = KernelStats()
    stream = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record(stream)
    nc = ncoef(cfg.p)
    # upward: owned cells, all-gather, shared top rebuilt redundantly
    M = torch.zeros((tree.ncells, nc), dtype=torch.float64, device=dev)
    cells, off = plan.owned[rank]
    _upward_cells(tree, cfg.p, cells, off, M)
    comm.allgather_rows(M, plan.chunks, rank, world)
    top, toff = plan.top
    if top.numel():
        M[top.long()] = 0.0
        _upward_cells(tree, cfg.p, top, toff, M)
    tree._M, tree.p = M, cfg.p
    tree._L = torch.zeros((tree.ncells, nc), dtype=torch.float64, device=dev)
    ev[1].record(stream)
    if treecode:
        # the rank's target leaves walk the whole (replicated) tree
        lists = treecode_lists(tree, cfg.mac, body_range=(lo, hi))
        ev[2].record(stream)
        far = torch.zeros((4, tree.n), dtype=torch.float64, device=dev)
        run_m2p(tree, lists, cfg.p, tuple(far))
    else:
        if cfg.strategy == "listfmm":
            lists = listfmm_lists(tree, body_range=(lo, hi))
        else:
            lists = interaction_lists(tree, cfg.mac, body_range=(lo, hi))
        ev[2].record(stream)
        run_m2l(tree, lists, cfg.p)
    ev[3].record(stream)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    run_p2p(tree, lists, cfg.precision, cfg.use_rsqrt, False, flag)
    if cfg.precision == "fp32" and int(flag.item()) != 0:
        run_p2p(tree, lists, cfg.precision, cfg.use_rsqrt, True, flag)
    ev[4].record(stream)
    if treecode:
        P = _lib.ptr
        _lib.call("fmm_combine", tree.n, *(P(a) for a in far), P(tree.d_phi), P(tree.d_fx), P(tree.d_fy),
                  P(tree.d_fz), _lib.stream_handle())
    else:
        downward_pass(tree, None, sync=False, body_range=(lo, hi))
    ev[5].record(stream)
    res = torch.stack([tree.d_phi, tree.d_fx, tree.d_fy, tree.d_fz], 1)
    comm.allgather_rows(res, plan.cuts, rank, world)
    for k, a in enumerate((tree.d_phi, tree.d_fx, tree.d_fy, tree.d_fz)):
        a.copy_(res[:, k])
    ev[6].record(stream)
    ev[6].synchronize()
    pairs, skipped = lists.dev_stats.tolist()
    stats.p2p_pairs, stats.p2p_skipped, stats.p2p_flops = int(pairs), int(skipped), 20 * int(pairs)
    stats.m2l_calls = lists.n_m2l
    stats.m2p_calls = getattr(lists, "n_m2p", 0)
    stats.add_time("list", ev[1].elapsed_time(ev[2]) * 1e-3)
    stats.add_time("m2p" if treecode else "m2l", ev[2].elapsed_time(ev[3]) * 1e-3)
    stats.add_time("p2p", ev[3].elapsed_time(ev[4]) * 1e-3)
    stats.add_time("allgather", ev[5].elapsed_time(ev[6]) * 1e-3)
    tree._results_changed()
    del _lib
    return EvalReport(strategy=cfg.strategy, n=tree.n, n_sources=tree.n, p=cfg.p, mac_kind=cfg.mac.kind,
                      theta=cfg.mac.theta, mutual=False, threads=world, task_grain=cfg.task_grain, stats=stats,
                      build_time=tree.build_time, upward_time=ev[0].elapsed_time(ev[1]) * 1e-3,
                      traversal_time=ev[1].elapsed_time(ev[4]) * 1e-3,
                      downward_time=0.0 if treecode else ev[4].elapsed_time(ev[6]) * 1e-3)
