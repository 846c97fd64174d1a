"""Sync-free (deferred-count) list construction: a traversal run from a
capacity hint chains its counting CSR and plan on the device and reads its
counters only at the end of the evaluation.  Its lists and results must be
bit-identical to the synchronising path, and an overflowing hint must be
detected and the evaluation redone."""

import numpy as np
import pytest

import paper_1209_3516_b200 as fb
from goldens import Case
from paper_1209_3516_b200 import traversal as tv

pytestmark = pytest.mark.gpu


def _tree(c):
    pos = np.asarray(c.pos, np.float64)
    return fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q), ncrit=c.ncrit)


def _hint_keys(t):
    return [k for k in tv._hint if isinstance(k[0], int) and k[0] == t.ncells]


@pytest.mark.parametrize("name", ["c1", "c2_32k", "plummer_32k"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_deferred_equals_synchronising(name, precision):
    c = Case(name)
    t = _tree(c)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", c.theta), p=c.p, precision=precision)
    for k in _hint_keys(t):
        del tv._hint[k]
    r1 = fb.evaluate_on_tree(t, cfg)  # no hint: synchronising path
    l1 = t.list_cache
    assert "_deferred" not in l1.__dict__ or l1.__dict__["_deferred"] is None
    want = [a.copy() for a in (t.bodies.phi, t.bodies.fx, t.bodies.fy, t.bodies.fz)]
    pairs1 = [np.asarray(x) for x in (*l1.host_pairs("m2l"), *l1.host_pairs("p2p"))]
    r2 = fb.evaluate_on_tree(t, cfg)  # hinted: deferred path
    l2 = t.list_cache
    pairs2 = [np.asarray(x) for x in (*l2.host_pairs("m2l"), *l2.host_pairs("p2p"))]
    for a, b in zip(pairs1, pairs2):
        assert np.array_equal(a, b)
    assert (r1.stats.p2p_pairs, r1.stats.m2l_calls, r1.stats.p2p_skipped) == \
        (r2.stats.p2p_pairs, r2.stats.m2l_calls, r2.stats.p2p_skipped)
    for w, g in zip(want, (t.bodies.phi, t.bodies.fx, t.bodies.fy, t.bodies.fz)):
        assert np.array_equal(w, g)


def test_overflowing_hint_is_redone():
    c = Case("c2_32k")
    t = _tree(c)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", c.theta), p=c.p)
    r0 = fb.evaluate_on_tree(t, cfg)
    want = t.bodies.phi.copy()
    keys = _hint_keys(t)
    assert keys
    for k in keys:  # far too small for every list and the frontier
        tv._hint[k] = (64, 64, 64)
    rep = fb.evaluate_on_tree(t, cfg)
    assert np.array_equal(t.bodies.phi, want)
    assert rep.stats.p2p_pairs == r0.stats.p2p_pairs and rep.stats.m2l_calls == r0.stats.m2l_calls
    assert all(tv._hint[k][0] > 64 for k in _hint_keys(t))


@pytest.mark.parametrize("method", ["bitmap", "radix"])
@pytest.mark.parametrize("nsrc", [70000, 3000000])
@pytest.mark.parametrize("shape", ["short", "long", "huge"])
def test_pairs_to_rows_matches_lexsort(shape, nsrc, method, monkeypatch):
    """The counting CSR (count, scatter, per-row block sort; long rows on the
    large tile, huge rows on the in-memory bitonic sort) against numpy."""
    import torch
    from paper_1209_3516_b200 import _lib
    rng = np.random.default_rng(5)
    if method == "radix":
        monkeypatch.setenv("FMM_B200_ROWSORT_RADIX", "1")
    ncells = 3000
    if shape == "short":
        t = rng.integers(0, ncells, 200000)
    elif shape == "long":  # a few rows of 1k..8k entries
        t = np.concatenate([rng.integers(0, ncells, 50000), np.repeat([7, 1234, 2999], [1500, 5000, 8000])])
    else:  # rows past the 8192-key tile
        t = np.concatenate([rng.integers(0, ncells, 20000), np.repeat([0, 42], [9000, 40000])])
    # distinct (t, s) pairs, as the traversals emit
    s = np.empty_like(t)
    for r in np.unique(t):
        m = t == r
        s[m] = rng.choice(nsrc, size=int(m.sum()), replace=False)
    perm = rng.permutation(t.size)
    t, s = t[perm], s[perm]
    dt = torch.as_tensor(t, dtype=torch.int32, device="cuda")
    ds = torch.as_tensor(s, dtype=torch.int32, device="cuda")
    cap = t.size + 100
    tt = torch.empty(cap, dtype=torch.int32, device="cuda")
    ss = torch.empty(cap, dtype=torch.int32, device="cuda")
    tt[:t.size] = dt
    ss[:t.size] = ds
    tt[t.size:] = 0  # past the device count: must be ignored
    ss[t.size:] = -5
    wsp, wsb = _lib.workspace(max(cap, ncells + 1), "cuda")
    dn = torch.full((1,), t.size, dtype=torch.int64, device="cuda")
    src = torch.empty(cap, dtype=torch.int32, device="cuda")
    rows = torch.empty(ncells + 1, dtype=torch.int64, device="cuda")
    _lib.call("fmm_pairs_to_rows", tt.data_ptr(), ss.data_ptr(), dn.data_ptr(), cap, ncells, nsrc, 1, src.data_ptr(),
              rows.data_ptr(), wsp, wsb, _lib.stream_handle())
    order = np.lexsort((s, t))
    want_rows = np.concatenate([[0], np.cumsum(np.bincount(t, minlength=ncells))])
    assert np.array_equal(rows.cpu().numpy(), want_rows)
    assert np.array_equal(src[:t.size].cpu().numpy(), s[order])


def test_plan_with_wide_rows_matches_oracle_p2p():
    """A tree with more than 32768 leaves: rows whose source-leaf ordinals
    span several bitmap windows take the register-sort plan path.  The P2P
    sums over the plan equal the oracle's over the same leaf pairs."""
    import torch
    from oracle import oracle as orc
    from paper_1209_3516_b200 import workloads as wl
    from paper_1209_3516_b200.traversal import run_p2p
    pos, q = wl.plummer(120000, 3)
    pos = np.asarray(pos, np.float64)
    q = np.asarray(q, np.float64)
    t = fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q), ncrit=3)
    assert t.nleaves > 40000
    lists = fb.interaction_lists(t, fb.MacConfig("fmm", 0.5))
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    run_p2p(t, lists, "fp64", flag=flag)
    got = t.d_phi.cpu().numpy()
    pt, ps = lists.host_pairs("p2p")
    ot = orc.build_tree(pos, q, 3)
    phi, fx, fy, fz, st = orc.exec_p2p(ot, pt, ps)
    assert np.linalg.norm(got - phi) <= 1e-12 * np.linalg.norm(phi)
    pairs, skipped = lists.dev_stats.tolist()
    assert (pairs, skipped) == (int(st[0]), int(st[1]))


def test_plan_short_runs_buffer_reports_capacity():
    """fmm_p2p_plan honours cap_runs: a short runs buffer leaves the
    overflowing rows empty, flags the required capacity in dev_stats[2] and
    (when the host asks for the run count) returns FMM_ERR_CAPACITY with the
    exact size -- the reference's grow-and-retry contract."""
    import ctypes as C

    import torch

    from paper_1209_3516_b200 import _lib
    c = Case("c1")
    t = _tree(c)
    lists = fb.interaction_lists(t, fb.MacConfig("fmm", c.theta), defer=False)
    P, dev = _lib.ptr, t.device
    wsp, wsb = _lib.workspace(max(lists.n_p2p, t.n, t.ncells + 1), dev)

    def plan(cap):
        leaf_rows = torch.empty(t.ncells, dtype=torch.int32, device=dev)
        run_off = torch.empty(2 * t.ncells, dtype=torch.int64, device=dev)
        runs = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=dev)
        stats = torch.empty(3, dtype=torch.int64, device=dev)
        nruns, nrows = C.c_int64(0), C.c_int32(0)
        _lib.call("fmm_p2p_plan", t.ncells, P(t.d_leaf), P(t.d_start), P(t.d_end), 0, t.n, None, P(lists.p2p_rows),
                  P(lists.p2p_grp), P(t.d_x), P(t.d_y), P(t.d_z), P(t.d_keys), None, 0, None, None, 0, P(leaf_rows),
                  P(run_off), P(runs), cap, C.byref(nruns), C.byref(nrows), None, P(stats), wsp, wsb,
                  _lib.stream_handle())
        return nruns.value, stats.tolist()

    n_ok, st_ok = plan(lists.n_p2p)
    assert st_ok[2] == 0 and st_ok[0] == c.meta["stats"]["p2p_pairs"] and 0 < n_ok <= lists.n_p2p
    short = lists.n_p2p // 3
    with pytest.raises(_lib.CapacityError):
        plan(short)
    # the exact requirement is the CSR end of the last row that did not fit
    rows = lists.p2p_rows.cpu().numpy()
    need = int(rows[1:][rows[1:] > short].max())
    nruns = C.c_int64(0)
    try:
        plan(short)
    except _lib.CapacityError as e:
        assert "needed" in str(e) and str(need) in str(e)
