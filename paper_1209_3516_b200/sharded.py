"""Sharded multi-GPU evaluation: every rank holds only its share of the
input, and after the build only the bodies its own targets and their near
field need ("each GPU handles only the near-field sources
its own targets need").

The replicated path (``distributed.evaluate_partitioned``) gives every rank
the whole cloud.  Here rank r is handed the r-th contiguous block of the
caller's input (global input indices ``[offsets[r], offsets[r+1])``) and

1. **Root cube.**  Local min/max, one MIN all-reduce: the same root cube as
   a single-GPU build (src/geometry.py:200-206, src/tree.py:387-392).
2. **Keys.**  Local depth-21 Morton keys, all-gathered in rank order (= the
   global input order), so the replicated stable radix sort gives the
   single-GPU permutation and the replicated carve the single-GPU cells, bit
   for bit.  Keys are 8 B per body; positions and charges (32 B) never
   travel to every rank.
3. **Own bodies.**  The leaves are cut into Morton-contiguous body ranges
   (the rule of ``distributed.body_cuts``); each rank sends its input bodies
   to the rank owning their sorted position (one variable all-to-all) and
   keeps ``[lo, hi)`` of the Morton-ordered body arrays.
4. **Geometry.**  Centres and radii come from the keys; bmax (max body
   distance from the centre) is each rank's max over its own bodies
   (``fmm_cell_bmax_range``) MAX-all-reduced over the cells -- the same bits.
5. **Evaluation.**  ``evaluate_partitioned`` (owned upward, multipole
   all-gather, traversal and lists of the own targets) with one hook before
   P2P: the **halo** -- the body ranges of the own P2P rows' source runs
   outside ``[lo, hi)`` -- is requested from their owners and received
   (two variable all-to-alls).  Nothing else is resident.
6. **Results.**  The own rows' (phi, f), sent back to the ranks that hold
   the corresponding inputs (``results="input"``), or left in Morton order
   on the owner (``"local"``).

The body arrays keep their global length so every kernel and plan indexes
bodies as on one GPU; only the own range and the halo are ever written or
read.  Collectives go through ``torch.distributed`` (NCCL device tensors,
or host-staged under gloo).  Cubic cells with geometric centres only (the
rect/com geometries need every body of a cell).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .tree import Tree, _carve_tree

__all__ = ["shard_offsets", "owner_of", "halo_ranges", "build_tree_sharded", "evaluate_sharded",
           "RESULTS_SHARDED"]

RESULTS_SHARDED = ("input", "local")


# ---------------------------------------------------------------------------
# host logic (pure NumPy: tests/test_distributed.py)
# ---------------------------------------------------------------------------
def shard_offsets(sizes) -> np.ndarray:
    """Global input offsets of the ranks' contiguous shards."""
    return np.concatenate([[0], np.cumsum(np.asarray(sizes, np.int64))]).astype(np.int64)


def owner_of(idx, bounds) -> np.ndarray:
    """Rank owning each index under half-open ``bounds`` [b_r, b_{r+1})."""
    return np.searchsorted(np.asarray(bounds, np.int64), np.asarray(idx, np.int64), side="right") - 1


def halo_ranges(starts, ends, lo: int, hi: int, cuts) -> list:
    """Per owner rank, the sorted, merged body ranges [s, e) covered by the
    runs [starts[k], ends[k]) outside the own range [lo, hi), split at the
    cuts: ``out[r]`` is an (m, 2) int64 array (empty for the own rank)."""
    cuts = np.asarray(cuts, np.int64)
    world = len(cuts) - 1
    s = np.asarray(starts, np.int64)
    e = np.asarray(ends, np.int64)
    keep = e > s
    s, e = s[keep], e[keep]
    out = [np.zeros((0, 2), np.int64) for _ in range(world)]
    if s.size == 0:
        return out
    order = np.argsort(s, kind="stable")
    s, e = s[order], e[order]
    # merge overlapping / touching ranges
    run_end = np.maximum.accumulate(e)
    new = np.concatenate([[True], s[1:] > run_end[:-1]])
    gs = s[new]
    ge = np.maximum.reduceat(e, np.flatnonzero(new))
    pieces = []
    for a, b in zip(gs.tolist(), ge.tolist()):
        # cut out the own range, then split at the rank cuts
        for x, y in ((a, min(b, lo)), (max(a, hi), b)):
            if y <= x:
                continue
            r0, r1 = int(owner_of(x, cuts)), int(owner_of(y - 1, cuts))
            for r in range(r0, r1 + 1):
                u, v = max(x, int(cuts[r])), min(y, int(cuts[r + 1]))
                if v > u:
                    pieces.append((r, u, v))
    for r in range(world):
        rr = [(u, v) for q, u, v in pieces if q == r]
        if rr:
            out[r] = np.asarray(rr, np.int64)
    return out


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------
class _Comm:
    """Variable-size exchanges over ``torch.distributed``: device tensors
    under NCCL, host-staged under gloo."""

    def __init__(self, group, dev):
        self.group, self.dev = group, dev
        self.nccl = dist.get_backend(group) == "nccl"

    def _on(self, t):
        return t.to(self.dev) if self.nccl else t.cpu()

    def all_reduce(self, t: torch.Tensor, op) -> torch.Tensor:
        x = self._on(t).clone()
        dist.all_reduce(x, op=op, group=self.group)
        return x.to(self.dev)

    def all_gather_sizes(self, n: int, world: int) -> list:
        t = self._on(torch.tensor([n], dtype=torch.int64))
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=self.group)
        return [int(x.item()) for x in out]

    def all_gather_var(self, t: torch.Tensor, sizes: list) -> torch.Tensor:
        """Concatenation over ranks of each rank's rows (``sizes[r]`` rows)."""
        width = int(np.prod(t.shape[1:])) if t.dim() > 1 else 1
        rows = max(max(sizes), 1)
        send = torch.zeros((rows, width), dtype=t.dtype, device=t.device)
        if t.shape[0]:
            send[:t.shape[0]] = t.reshape(t.shape[0], width)
        send = self._on(send)
        recv = torch.empty((len(sizes) * rows, width), dtype=t.dtype, device=send.device)
        dist.all_gather_into_tensor(recv, send, group=self.group) if self.nccl else \
            dist.all_gather(list(recv.split(rows)), send, group=self.group)
        parts = [recv[r * rows:r * rows + sizes[r]] for r in range(len(sizes))]
        out = torch.cat(parts).to(self.dev)
        return out.reshape((-1,) + tuple(t.shape[1:])) if t.dim() > 1 else out.reshape(-1)

    def all_to_all_var(self, send: torch.Tensor, counts: list) -> tuple[torch.Tensor, list]:
        """Rows ``send`` grouped by destination (``counts[r]`` rows for rank
        r) -> the rows received, grouped by source, and their counts."""
        c = self._on(torch.tensor(counts, dtype=torch.int64))
        rc = torch.empty_like(c)
        dist.all_to_all_single(rc, c, group=self.group)
        rcounts = [int(x) for x in rc.tolist()]
        width = int(np.prod(send.shape[1:])) if send.dim() > 1 else 1
        s = self._on(send.reshape(-1, width).contiguous())
        r = torch.empty((sum(rcounts), width), dtype=send.dtype, device=s.device)
        dist.all_to_all_single(r, s, output_split_sizes=rcounts, input_split_sizes=list(counts), group=self.group)
        return r.to(self.dev), rcounts


# ---------------------------------------------------------------------------
# build
# ---------------------------------------------------------------------------
def _root_from_bounds(lo, hi) -> list:
    """The root record of csrc/tree_build.cu ``bounds_final`` from global
    min/max (same float64 operations, so the same bits)."""
    size = hi[0] - lo[0]
    e1, e2 = hi[1] - lo[1], hi[2] - lo[2]
    if e1 > size:
        size = e1
    if e2 > size:
        size = e2
    if size == 0.0:
        size = 1.0
    return [lo[0], lo[1], lo[2], size, float(1 << 21) / size, hi[0], hi[1], hi[2]]


def _pack32(xs, ys, zs, qs, idx, b32, b32lo):
    """The float4 copies of ``fmm_permute_bodies`` at positions ``idx``
    (round-to-nearest float32, then the float32 residual of x, y, z)."""
    x, y, z, q = xs[idx], ys[idx], zs[idx], qs[idx]
    h = torch.stack([x.float(), y.float(), z.float(), q.float()], 1)
    b32[idx] = h
    lo = torch.stack([(x - h[:, 0].double()).float(), (y - h[:, 1].double()).float(),
                      (z - h[:, 2].double()).float(), torch.zeros_like(h[:, 0])], 1)
    b32lo[idx] = lo
    return bool((lo[:, :3] != 0).any().item()) if idx.numel() else False


def build_tree_sharded(x, y, z, q, ncrit: int, rank: int, world: int, group=None, *, device=None,
                       allow_oversized_leaves: bool = False) -> Tree:
    """Collective build from this rank's shard (``x, y, z, q``: the rank-th
    contiguous block of the global input, host NumPy or device tensors).
    Returns a ``Tree`` whose cells, keys and permutation equal a single-GPU
    build of the whole input, with only the own bodies resident."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    comm = _Comm(group, dev)
    P = _lib.ptr
    with torch.cuda.device(dev):
        st = _lib.stream_handle()
        src = [torch.as_tensor(a).to(dev) for a in (x, y, z, q)]
        dt = src[0].dtype
        if dt not in (torch.float32, torch.float64):
            raise ValueError(f"positions must be float32 or float64, got {dt}")
        src = [a.to(dt).contiguous() for a in src]
        n_loc = src[0].numel()
        sizes = comm.all_gather_sizes(n_loc, world)
        offsets = shard_offsets(sizes)
        n = int(offsets[-1])
        if n == 0:
            raise ValueError("empty particle set")
        # 1. root cube
        l64 = [torch.empty(n_loc, dtype=torch.float64, device=dev) for _ in range(4)]
        root_l = torch.empty(8, dtype=torch.float64, device=dev)
        wsp, wsb = _lib.workspace(max(n, 1), dev)
        if n_loc:
            dcode = _lib.DTYPE_F64 if dt == torch.float64 else _lib.DTYPE_F32
            _lib.call("fmm_ingest_bounds", *(P(a) for a in src), dcode, n_loc, *(P(a) for a in l64), P(root_l),
                      wsp, wsb, st)
            ext = torch.cat([root_l[0:3], -root_l[5:8]])
        else:
            ext = torch.full((6,), float("inf"), dtype=torch.float64, device=dev)
        ext = comm.all_reduce(ext, dist.ReduceOp.MIN).tolist()
        root = torch.tensor(_root_from_bounds(ext[0:3], [-v for v in ext[3:6]]), dtype=torch.float64, device=dev)
        # 2. keys, all-gathered in input order; the replicated stable sort
        keys_l = torch.empty(n_loc, dtype=torch.int64, device=dev)
        iota_l = torch.empty(n_loc, dtype=torch.int32, device=dev)
        if n_loc:
            _lib.call("fmm_morton_keys", *(P(a) for a in l64[:3]), n_loc, P(root), P(keys_l), P(iota_l), st)
        keys = comm.all_gather_var(keys_l, sizes)
        iota = torch.arange(n, dtype=torch.int32, device=dev)
        skeys = torch.empty_like(keys)
        perm = torch.empty_like(iota)
        _lib.call("fmm_sort_pairs_u64", P(keys), P(iota), P(skeys), P(perm), n, 63, wsp, wsb, st)
        del keys, iota
        # full-length Morton-ordered body arrays, filled only where resident
        xs, ys, zs, qs = (torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(4))
        b32 = torch.zeros((n, 4), dtype=torch.float32, device=dev)
        b32lo = torch.zeros((n, 4), dtype=torch.float32, device=dev)
        inexact = torch.zeros(1, dtype=torch.int32, device=dev)
        tree = _carve_tree(dev, st, wsp, wsb, n, ncrit, "cubic", "geometric", allow_oversized_leaves, skeys, perm,
                           root, (xs, ys, zs, qs, b32, b32lo), inexact)
        # 3. cuts (distributed.body_cuts' rule) and the own bodies
        at = torch.tensor([r * n // world for r in range(1, world)], dtype=torch.int64, device=dev)
        inner = tree.d_start[tree.d_body_leaf[at].long()].tolist() if world > 1 else []
        cuts = [0]
        for c in inner:
            cuts.append(max(int(c), cuts[-1]))
        cuts.append(n)
        cuts = np.asarray(cuts, np.int64)
        lo, hi = int(cuts[rank]), int(cuts[rank + 1])
        pos_of = torch.empty(n, dtype=torch.int64, device=dev)
        pos_of[perm.long()] = torch.arange(n, dtype=torch.int64, device=dev)
        mine = pos_of[int(offsets[rank]):int(offsets[rank + 1])]  # sorted positions of the local inputs
        dest = torch.as_tensor(owner_of(mine.cpu().numpy(), cuts), device=dev)
        order = torch.argsort(dest, stable=True)
        rows = torch.stack([mine.double(), *l64], 1)[order]
        counts = torch.bincount(dest, minlength=world).tolist()
        recv, _ = comm.all_to_all_var(rows, counts)
        pos = recv[:, 0].long()
        for k, a in enumerate((xs, ys, zs, qs)):
            a[pos] = recv[:, 1 + k]
        flag = _pack32(xs, ys, zs, qs, pos, b32, b32lo)
        # 4. bmax over the own bodies, MAX over the ranks; float32 exactness over all ranks
        bm = torch.empty(tree.ncells, dtype=torch.float64, device=dev)
        _lib.call("fmm_cell_bmax_range", tree.ncells, P(tree.d_start), P(tree.d_end), P(tree.d_ctr), P(xs), P(ys),
                  P(zs), lo, hi, P(bm), wsp, wsb, st)
        tree.d_bmax.copy_(comm.all_reduce(bm, dist.ReduceOp.MAX))
        fl = comm.all_reduce(torch.tensor([int(flag)], dtype=torch.int32, device=dev), dist.ReduceOp.MAX)
        tree._fp32_exact = int(fl.item()) == 0
        tree.d_inexact.fill_(int(not tree._fp32_exact))
    tree._input_snapshot = None
    tree.build_time = 0.0
    tree.shard = dict(rank=rank, world=world, offsets=offsets, cuts=cuts, own=(lo, hi), n_local=n_loc,
                      halo_bodies=0)
    return tree


# ---------------------------------------------------------------------------
# evaluation
# ---------------------------------------------------------------------------
def _fetch_halo(tree: Tree, lists, comm: _Comm) -> int:
    """Bring the P2P source bodies outside the own range from their owners
    (before the rank's P2P); returns the number of halo bodies."""
    sh = tree.shard
    lo, hi, cuts, world = sh["own"][0], sh["own"][1], sh["cuts"], sh["world"]
    dev = tree.device
    nrows = int(lists.dev_nrows.item())
    run_off = lists.run_off[:2 * nrows].view(nrows, 2)
    runs = lists.runs
    # every run of every own row, as [bstart, bend) (row-local run storage)
    cnt = (run_off[:, 1] - run_off[:, 0]).clamp_min(0)
    if int(cnt.sum().item()):
        first = torch.repeat_interleave(run_off[:, 0], cnt)
        rel = torch.arange(first.numel(), device=dev) - torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt)
        rr = runs[(first + rel).long()]
        starts, ends = rr[:, 0].cpu().numpy(), rr[:, 1].cpu().numpy()
    else:
        starts = ends = np.zeros(0, np.int64)
    want = halo_ranges(starts, ends, lo, hi, cuts)
    # requests: (s, e) pairs to each owner; replies: the bodies in request order
    req = np.concatenate([w for w in want]) if world else np.zeros((0, 2), np.int64)
    got_req, rcounts = comm.all_to_all_var(torch.as_tensor(req.reshape(-1, 2), device=dev),
                                           [len(w) for w in want])
    gr = got_req.cpu().numpy().astype(np.int64).reshape(-1, 2)
    send_idx, send_counts, k = [], [], 0
    for r in range(world):
        seg = gr[k:k + rcounts[r]]
        k += rcounts[r]
        idx = np.concatenate([np.arange(s, e) for s, e in seg]) if len(seg) else np.zeros(0, np.int64)
        send_idx.append(idx)
        send_counts.append(len(idx))
    sidx = torch.as_tensor(np.concatenate(send_idx) if send_idx else np.zeros(0, np.int64), device=dev)
    body = torch.stack([tree.d_x[sidx], tree.d_y[sidx], tree.d_z[sidx], tree.d_q[sidx]], 1)
    recv, _ = comm.all_to_all_var(body, send_counts)
    pos = torch.as_tensor(np.concatenate([np.arange(s, e) for s, e in req]) if len(req) else np.zeros(0, np.int64),
                          device=dev)
    for j, a in enumerate((tree.d_x, tree.d_y, tree.d_z, tree.d_q)):
        a[pos] = recv[:, j]
    _pack32(tree.d_x, tree.d_y, tree.d_z, tree.d_q, pos, tree.d_b32, tree.d_b32lo)
    tree.__dict__.pop("d_b64", None)  # the FP64 P2P's packed copy is rebuilt from the filled arrays
    tree.shard["halo_bodies"] = int(pos.numel())
    return int(pos.numel())


def evaluate_sharded(tree: Tree, cfg, group=None, results: str = "input"):
    """Evaluate a ``build_tree_sharded`` tree.  ``results="input"`` returns
    (phi, fx, fy, fz) float64 tensors for this rank's input shard, in its
    order; ``"local"`` leaves the own rows in Morton order in the tree
    (``tree.owned_range``) and returns None.  Returns (report, results)."""
    from .distributed import evaluate_partitioned
    if results not in RESULTS_SHARDED:
        raise ValueError(f"results must be one of {RESULTS_SHARDED}, got {results!r}")
    sh = tree.shard
    rank, world = sh["rank"], sh["world"]
    comm = _Comm(group, tree.device)
    rep = evaluate_partitioned(tree, cfg, rank, world, group=group, results="local",
                               before_p2p=lambda lists: _fetch_halo(tree, lists, comm))
    if results == "local":
        return rep, None
    lo, hi = sh["own"]
    dev = tree.device
    offsets = sh["offsets"]
    g = tree.d_perm[lo:hi].long()  # global input index of each own row
    dest = torch.as_tensor(owner_of(g.cpu().numpy(), offsets), device=dev)
    order = torch.argsort(dest, stable=True)
    rows = torch.stack([(g - torch.as_tensor(offsets, device=dev)[dest]).double(), tree.d_phi[lo:hi],
                        tree.d_fx[lo:hi], tree.d_fy[lo:hi], tree.d_fz[lo:hi]], 1)[order]
    recv, _ = comm.all_to_all_var(rows, torch.bincount(dest, minlength=world).tolist())
    out = [torch.zeros(sh["n_local"], dtype=torch.float64, device=dev) for _ in range(4)]
    li = recv[:, 0].long()
    for k in range(4):
        out[k][li] = recv[:, 1 + k]
    return rep, tuple(out)
