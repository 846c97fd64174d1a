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

__all__ = ["body_cuts", "cell_chunks", "shared_cells", "allgather_rows", "gather_rows", "TorchDistComm",
           "evaluate_partitioned", "RESULTS"]


def body_cuts(leaf_start: np.ndarray, leaf_end: np.ndarray, n: int, world: int) -> np.ndarray:
    """Cut points ``cuts[0]=0 <= ... <= cuts[world]=n`` on leaf boundaries:
    cut r is the start of the leaf holding body ``r * n // world`` (leaves in
    Morton order), within one leaf of the equal split."""
    starts = np.sort(np.asarray(leaf_start, np.int64))
    cuts = [0]
    for r in range(1, world):
        k = int(np.searchsorted(starts, r * n // world, side="right")) - 1
        cuts.append(max(int(starts[max(k, 0)]), cuts[-1]))
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


def _device_collectives(t: torch.Tensor, group=None) -> bool:
    """True when the group's backend moves CUDA tensors itself (NCCL over
    NVLink); gloo moves host tensors, so device rows are staged through the
    host."""
    return t.is_cuda and dist.get_backend(group) == "nccl"


def _padded_rows(full: torch.Tensor, chunks, rank: int, world: int):
    sizes = [int(chunks[r + 1] - chunks[r]) for r in range(world)]
    width = int(np.prod(full.shape[1:])) if full.dim() > 1 else 1
    rows = max(max(sizes), 1)
    send = torch.zeros((rows, width), dtype=full.dtype, device=full.device)
    mine = full[int(chunks[rank]):int(chunks[rank + 1])].reshape(-1, width)
    send[:mine.shape[0]].copy_(mine)
    return sizes, width, rows, send


def allgather_rows(full: torch.Tensor, chunks, rank: int, world: int, group=None) -> None:
    """Replace ``full[chunks[r]:chunks[r+1]]`` with rank r's rows, for every r:
    one padded all-gather (``all_gather_into_tensor`` on device tensors under
    NCCL; host-staged ``all_gather`` under gloo)."""
    sizes, width, rows, send = _padded_rows(full, chunks, rank, world)
    if _device_collectives(full, group):
        recv = torch.empty((world * rows, width), dtype=full.dtype, device=full.device)
        dist.all_gather_into_tensor(recv, send, group=group)
    else:
        send = send.cpu()
        recv = torch.empty((world * rows, width), dtype=full.dtype)
        dist.all_gather(list(recv.split(rows)), send, group=group)
    recv = recv.to(full.device, non_blocking=True)
    for r in range(world):
        if sizes[r]:
            full[int(chunks[r]):int(chunks[r + 1])].reshape(-1, width).copy_(recv[r * rows:r * rows + sizes[r]])


def gather_rows(full: torch.Tensor, chunks, rank: int, world: int, root: int = 0, group=None) -> None:
    """Like ``allgather_rows`` but only ``root`` receives the other ranks'
    rows (one padded gather: (world - 1) / world of the all-gather's
    traffic stays off the other ranks)."""
    sizes, width, rows, send = _padded_rows(full, chunks, rank, world)
    dev = _device_collectives(full, group)
    if not dev:
        send = send.cpu()
    recv = None
    if rank == root:
        recv = torch.empty((world * rows, width), dtype=full.dtype, device=send.device)
    dist.gather(send, list(recv.split(rows)) if recv is not None else None, dst=root, group=group)
    if rank != root:
        return
    recv = recv.to(full.device, non_blocking=True)
    for r in range(world):
        if sizes[r] and r != rank:
            full[int(chunks[r]):int(chunks[r + 1])].reshape(-1, width).copy_(recv[r * rows:r * rows + sizes[r]])


class _Plan:
    """This rank's share of the tree, computed on the device each step
    (``body_cuts``, ``cell_chunks`` and ``shared_cells`` above state the same
    rules on NumPy arrays):

    * ``cuts``: body cut points on leaf boundaries (the start of the leaf
      holding body r * n / world), ``chunks``: the cells whose first body
      lies in each rank's range (pre-order cell starts are non-decreasing);
    * ``owned``: this rank's cells (body range inside its own), grouped by
      level, ``top``: cells straddling an interior cut, grouped by level --
      both as (device id list, host level offsets) for ``fmm_upward``.
    One small device-to-host read, no host copies of cell arrays."""

    def __init__(self, tree, world: int, rank: int):
        from . import _lib
        P = _lib.ptr
        dev, ncells = tree.device, tree.ncells
        own = torch.empty(ncells, dtype=torch.int32, device=dev)
        top = torch.empty(ncells, dtype=torch.int32, device=dev)
        nl = 32
        host = np.zeros(2 * (world + 1) + 3 * nl, np.int64)
        wsp, wsb = _lib.workspace(ncells + 1, dev)
        _lib.call("fmm_partition_plan", ncells, tree.n, world, rank, P(tree.d_start), P(tree.d_end),
                  P(tree.d_body_leaf), P(tree.d_cells_by_level), P(tree.d_level), P(own), P(top),
                  host.ctypes.data, wsp, wsb, _lib.stream_handle())
        self.cuts = host[:world + 1].copy()
        self.chunks = host[world + 1:2 * world + 2].copy()
        cnt = host[2 * world + 2:].reshape(3, nl)
        depth = len(tree.level_off) - 2
        self.lists = [own[:int(cnt[0].sum())], top[:int(cnt[1].sum())]]
        self.owned = (self.lists[0], [0] + list(np.cumsum(cnt[0][:depth + 1]).astype(int)))
        self.top = (self.lists[1], [0] + list(np.cumsum(cnt[1][:depth + 1]).astype(int)))


def _upward_cells(tree, p, cells, off, M):
    import ctypes as C
    from . import _lib
    P = _lib.ptr
    offc = (C.c_int32 * len(off))(*off)
    _lib.call("fmm_upward", p, tree.ncells, P(tree.d_children), P(tree.d_start), P(tree.d_end), P(tree.d_leaf),
              P(tree.d_ctr), P(tree.d_x), P(tree.d_y), P(tree.d_z), P(tree.d_q), P(cells), offc, len(off) - 1,
              P(M), _lib.stream_handle())


class TorchDistComm:
    """Exchange through ``torch.distributed`` (NCCL over NVLink on the box,
    gloo with host staging elsewhere)."""

    def __init__(self, group=None):
        self.group = group

    def allgather_rows(self, full, chunks, rank, world):
        allgather_rows(full, chunks, rank, world, self.group)

    def gather_rows(self, full, chunks, rank, world, root=0):
        gather_rows(full, chunks, rank, world, root, self.group)

    def all_true(self, ok: bool, rank: int, world: int) -> bool:
        """Whether ``ok`` holds on every rank (one MIN all-reduce)."""
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(ok)], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return bool(int(t.item()))


RESULTS = ("all", "root", "local")


def evaluate_partitioned(tree, cfg, rank: int, world: int, group=None, comm=None, results: str = "all",
                         before_p2p=None):
    """Evaluate ``tree`` with targets Morton-partitioned over ``world`` ranks.

    ``results`` picks where the (phi, f) rows end up: "all" (one all-gather:
    every rank holds the full result), "root" (one gather to rank 0; the
    other ranks keep their own rows) or "local" (no exchange: each rank's
    tree is valid on its own bodies ``tree.owned_range`` only).  The
    ``EvalReport`` counters cover the rank's own rows.  ``comm`` defaults to
    :class:`TorchDistComm`; tests pass an in-process exchange to emulate
    ranks on one device.  ``before_p2p(lists)`` runs once the rank's lists
    exist, before its near field (``sharded`` fetches its halo there)."""
    if results not in RESULTS:
        raise ValueError(f"results must be one of {RESULTS}, got {results!r}")
    comm = comm or TorchDistComm(group)
    from . import _lib
    from .kernels import KernelStats, ncoef
    from .traversal import (EndReadback, EvalReport, _EventPool, critical_path, interaction_lists, listfmm_lists,
                            m2l_grouped, mutual_lists, _near_field, run_m2l, run_m2p, run_p2p, treecode_lists)
    from .tree import downward_pass

    if world == 1:
        from .traversal import evaluate_on_tree
        return evaluate_on_tree(tree, cfg)
    treecode = cfg.strategy == "treecode"
    nf = _near_field(cfg, tree)
    defer = hasattr(comm, "all_true")  # a collective decision on list overflows is available
    plan = getattr(tree, "_dist_plan", None)
    if plan is None or len(plan.cuts) != world + 1 or plan.rank != rank:
        plan = _Plan(tree, world, rank)
        plan.rank = rank
        tree._dist_plan = plan
    lo, hi = int(plan.cuts[rank]), int(plan.cuts[rank + 1])
    dev = tree.device
    stats = KernelStats()
    from .traversal import _side_stream
    main = torch.cuda.current_stream(dev)
    side = _side_stream(dev)
    E = _EventPool(dev)
    ev = [E() for _ in range(9)]
    ev[0].record(main)
    nc = ncoef(cfg.p)
    # the expansions, the far-field accumulators and the flag share one fill
    nm = tree.ncells * nc
    buf = torch.zeros(2 * nm + 4 * tree.n + 1, dtype=torch.float64, device=dev)
    M = buf[:nm].view(tree.ncells, nc)
    L = buf[nm:2 * nm].view(tree.ncells, nc)
    far = buf[2 * nm:2 * nm + 4 * tree.n].view(4, tree.n)
    flag = buf[-1:].view(torch.int32)[:1]
    # far field, side stream: owned upward, all-gather, shared top rebuilt
    # redundantly -- beside the main stream's traversal, which needs no moments
    side.wait_event(ev[0])
    with torch.cuda.stream(side):
        cells, off = plan.owned
        _upward_cells(tree, cfg.p, cells, off, M)
        comm.allgather_rows(M, plan.chunks, rank, world)
        top, toff = plan.top
        if top.numel():
            M[top.long()] = 0.0
            _upward_cells(tree, cfg.p, top, toff, M)
        ev[1].record(side)
    tree._M, tree.p, tree._L = M, cfg.p, L
    ready = E()
    sort_far = not m2l_grouped(tree, cfg.p)  # (the grouped M2L orders its pairs itself)
    if treecode:  # the rank's target leaves walk the whole (replicated) tree
        lists = treecode_lists(tree, cfg.mac, body_range=(lo, hi), m2p_ready=ready, side=side)
    elif cfg.strategy == "listfmm":
        lists = listfmm_lists(tree, body_range=(lo, hi), m2l_ready=ready, side=side, sort_far=sort_far)
    elif cfg.mutual:  # the rank's targets of the mutual lists (directed-expanded)
        lists = mutual_lists(tree, cfg.mac, cfg.task_grain, body_range=(lo, hi), m2l_ready=ready, side=side,
                             defer=defer, sort_far=sort_far)
    else:
        # hinted lists do not wait for their counters; an overflow on any rank
        # is caught at the end and every rank redoes the step (comm.all_true)
        lists = interaction_lists(tree, cfg.mac, body_range=(lo, hi), m2l_ready=ready, side=side, defer=defer,
                                  sort_far=sort_far)
    ev[2].record(main)
    side.wait_event(ready)
    with torch.cuda.stream(side):
        ev[3].record(side)
        if treecode:
            run_m2p(tree, lists, cfg.p, tuple(far), precision=nf)
        else:
            run_m2l(tree, lists, cfg.p)
        ev[4].record(side)
        if not treecode:
            downward_pass(tree, None, sync=False, body_range=(lo, hi), out=tuple(far))
        ev[5].record(side)
    if before_p2p is not None:  # the sharded path's halo exchange (sharded.py)
        before_p2p(lists)
    ev[6].record(main)
    run_p2p(tree, lists, nf, cfg.use_rsqrt, False, flag)
    ev[7].record(main)
    main.wait_event(ev[5])
    P = _lib.ptr
    combine = lambda: _lib.call("fmm_combine", tree.n, *(P(a) for a in far), P(tree.d_phi),  # noqa: E731
                                P(tree.d_fx), P(tree.d_fy), P(tree.d_fz), _lib.stream_handle())
    combine()
    # one read-back of the FP32 flag and the list / pair counters
    rb = EndReadback([flag] + lists.device_counters())
    done = E()
    done.record(main)
    done.synchronize()
    host = rb.parts()
    ok = lists.settle(host[1:])
    if defer and not comm.all_true(ok, rank, world):
        # a hinted list outgrew its buffer on some rank: every rank redoes the
        # step (the overflowing rank's hint is gone, so it counts exactly)
        return evaluate_partitioned(tree, cfg, rank, world, group=group, comm=comm, results=results,
                                    before_p2p=before_p2p)
    if nf in ("fp32", "fp32acc") and int(host[0][0]) != 0:
        run_p2p(tree, lists, nf, cfg.use_rsqrt, True, flag)  # rewrites the near field: add the far field again
        combine()
    tree.owned_range = (lo, hi)
    if results != "local":
        res = torch.stack([tree.d_phi, tree.d_fx, tree.d_fy, tree.d_fz], 1)
        if results == "all":
            comm.allgather_rows(res, plan.cuts, rank, world)
        else:
            comm.gather_rows(res, plan.cuts, rank, world, 0)
        if results == "all" or rank == 0:
            tree.owned_range = (0, tree.n)
            for k, a in enumerate((tree.d_phi, tree.d_fx, tree.d_fy, tree.d_fz)):
                a.copy_(res[:, k])
    ev[8].record(main)
    ev[8].synchronize()
    pairs, skipped = host[1].tolist()
    stats.p2p_pairs, stats.p2p_skipped, stats.p2p_flops = int(pairs), int(skipped), 20 * int(pairs)
    stats.m2l_calls = lists.n_m2l
    stats.m2p_calls = getattr(lists, "n_m2p", 0)
    stats.add_time("list", ev[0].elapsed_time(ev[2]) * 1e-3)
    stats.add_time("m2p" if treecode else "m2l", ev[3].elapsed_time(ev[4]) * 1e-3)
    stats.add_time("p2p", ev[6].elapsed_time(ev[7]) * 1e-3)
    stats.add_time("allgather", ev[7].elapsed_time(ev[8]) * 1e-3)
    tree._results_changed()
    del _lib
    ms = lambda a, b: ev[a].elapsed_time(ev[b]) * 1e-3  # noqa: E731
    up, trav, down = critical_path(ms(0, 7), ms(0, 1), ms(0, 4), ms(0, 8))
    if treecode:
        trav, down = trav + down, 0.0
    spans = {"lists": ms(0, 2), "upward_allgather": ms(0, 1), "m2p" if treecode else "m2l": ms(3, 4),
             "downward": ms(4, 5), "p2p": ms(6, 7), "result_allgather": ms(7, 8), "wall": ms(0, 8)}
    return EvalReport(strategy=cfg.strategy, n=tree.n, n_sources=tree.n, p=cfg.p, mac_kind=cfg.mac.kind,
                      theta=cfg.mac.theta, mutual=cfg.mutual, threads=world, task_grain=cfg.task_grain, stats=stats,
                      build_time=tree.build_time, upward_time=up, traversal_time=trav, downward_time=down,
                      spans=spans, near_field=nf)
