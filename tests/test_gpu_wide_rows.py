"""Rows whose ids span several bitmap windows (16384 ids per pass; the
adaptive C3 trees) and rows longer than the plan's 512-source staging (the
per-pass gather path; theta = 0.3 at C4 density): the sparse row sort
(csrc/rowsort.cuh ``warp_bitmap_sort_sparse``, M2L/M2P CSR and
``Lists.p2p_src``) and the P2P plan rows (csrc/plan.cu ``plan_rows_kernel``:
``plan_row_staged`` and the gather passes) against independent torch /
numpy computations.  The golden cases are too small to reach these paths."""
import numpy as np
import pytest
import torch

import paper_1209_3516_b200 as fb
from paper_1209_3516_b200 import _lib, workloads
from paper_1209_3516_b200.traversal import _csr

pytestmark = pytest.mark.gpu


def test_sparse_row_sort_matches_torch():
    g = torch.Generator().manual_seed(7)
    ncells, nsrc = 3000, 400_000
    lens = torch.randint(1, 1025, (ncells,), generator=g)
    lens[::7] = torch.randint(1025, 3000, (len(lens[::7]),), generator=g)  # a few past the staged size
    t, s = [], []
    for r, ln in enumerate(lens.tolist()):
        # distinct ids in a few dense clusters far apart (several windows)
        centres = torch.randint(0, nsrc - 2000, (4,), generator=g)
        pool = torch.unique(torch.cat([c + torch.randint(0, 2000, (ln,), generator=g) for c in centres]))
        pick = pool[torch.randperm(len(pool), generator=g)[:ln]]
        t.append(torch.full((len(pick),), r, dtype=torch.int32))
        s.append(pick.to(torch.int32))
    t = torch.cat(t)
    s = torch.cat(s)
    perm = torch.randperm(len(t), generator=g)
    t, s = t[perm].cuda(), s[perm].cuda()
    n = len(t)
    wsp, wsb = _lib.workspace(max(n, ncells + 1), "cuda")
    src, rows = _csr(t, s, n, ncells, torch.device("cuda"), wsp, wsb, _lib.stream_handle(), nsrc=nsrc)
    torch.cuda.synchronize()
    key = t.long() * nsrc + s.long()
    want = (torch.sort(key).values % nsrc).to(torch.int32)
    assert torch.equal(src[:n], want)
    counts = torch.bincount(t.long(), minlength=ncells)
    assert torch.equal(rows[1:] - rows[:-1], counts)


@pytest.fixture(scope="module", params=["plummer_2e21", "uniform_2e18_theta0.3"])
def plummer_tree(request):
    if request.param == "plummer_2e21":
        gen, _, solver = workloads.CONFIGS["C3"]
        pos, q = gen(1 << 21, 0)
        theta = solver["theta"]
    else:
        gen, _, solver = workloads.CONFIGS["C4"]
        pos, q = gen(1 << 18, 0)
        theta = 0.3
    d = torch.as_tensor(pos, device="cuda")
    ps = fb.ParticleSet(d[:, 0].contiguous(), d[:, 1].contiguous(), d[:, 2].contiguous(),
                        torch.as_tensor(q, device="cuda"))
    tree = fb.build_tree(ps, ncrit=solver["ncrit"])
    return request.param, tree, fb.interaction_lists(tree, fb.MacConfig("fmm", theta))


def cnt_max(rows):
    return (rows[1:] - rows[:-1]).max()


def test_wide_plan_rows_match_numpy(plummer_tree):
    name, tree, lists = plummer_tree
    lists.settle()
    leaf = tree.d_leaf.cpu().numpy().astype(bool)
    start, end = tree.d_start.cpu().numpy(), tree.d_end.cpu().numpy()
    ordinal = np.cumsum(leaf) - 1
    # sorted P2P rows (the sparse sort, checked above) -> expected runs
    rows = lists.p2p_rows.cpu().numpy()
    src = lists.p2p_src[:rows[-1]].cpu().numpy()
    spans = [(ordinal[src[rows[c]:rows[c + 1]]].max() - ordinal[src[rows[c]:rows[c + 1]]].min())
             for c in np.nonzero(rows[1:] > rows[:-1])[0]]
    if name.startswith("plummer"):
        assert max(spans) >= 16384  # rows spanning several bitmap windows
    else:
        assert int(cnt_max(rows)) > 512  # rows past the staged size
    # expected runs, vectorised: an entry opens a run at a row start, at the
    # self leaf, right after it, or where the ordinals stop being consecutive
    cnt = rows[1:] - rows[:-1]
    row_of = np.repeat(np.arange(len(cnt)), cnt)
    o = ordinal[src]
    own = src == row_of
    first = np.zeros(len(src), dtype=bool)
    first[rows[:-1][cnt > 0]] = True
    prev_own = np.concatenate([[False], own[:-1]])
    prev_o = np.concatenate([[-2], o[:-1]])
    opens = first | own | prev_own | (o != prev_o + 1)
    rid = np.cumsum(opens) - 1
    nrun = np.bincount(rid)
    run_first = np.nonzero(opens)[0]
    run_last = run_first + nrun - 1
    want = np.stack([start[src[run_first]], end[src[run_last]], own[run_first].astype(np.int64)], axis=1)
    run_row = row_of[run_first]
    row_first_run = np.full(len(cnt), -1)
    row_first_run[run_row[::-1]] = np.arange(len(run_row))[::-1]
    slot = rows[:-1][run_row] + (np.arange(len(run_row)) - row_first_run[run_row])  # row-local at the CSR offset
    leaf_rows = lists.leaf_rows[:int(lists.dev_nrows.item())].cpu().numpy()
    run_off = lists.run_off.cpu().numpy().reshape(-1, 2)[:len(leaf_rows)]
    runs = lists.runs.cpu().numpy()
    nrun_row = np.bincount(run_row, minlength=len(cnt))
    assert np.array_equal(run_off[:, 0], rows[leaf_rows])
    assert np.array_equal(run_off[:, 1] - run_off[:, 0], nrun_row[leaf_rows])
    assert np.array_equal(runs[slot, :3], want)
    nt = (end - start)[row_of]
    pairs = int(np.sum(nt * (end - start)[src])) - int(np.sum(nt[own]))
    skipped = int(lists.dev_stats[1].item())
    assert int(lists.dev_stats[0].item()) == pairs - skipped
