"""Mutual dual traversal on the B200 vs the reference's
mutual goldens (tests/golden/make_golden_mutual.py) and the C oracle.

Bit-exact: the partition roots, the directed-expanded M2L / P2P event sets
(the reference's ``trace``) and the counters.  FP64 results within 1e-11
relative L2 of the reference's; FP32 near field within 2x the reference's
own error against direct summation.
"""

import numpy as np
import pytest
import torch

import paper_1209_3516_b200 as fb
from goldens import FP32_BAR_FLOOR, MU_CASES, MuCase, canon_pairs, rel_l2, sha
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
FP64_TOL = 1e-11
STAT_KEYS = ("p2p_pairs", "p2p_skipped", "p2p_flops", "m2l_calls", "p2m_calls", "m2m_calls", "l2l_calls",
             "l2p_calls")


def build(c: MuCase):
    pos = np.asarray(c.pos, np.float64)
    return fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q), ncrit=c.ncrit)


def cfg_of(c: MuCase, **kw):
    return fb.EvalConfig(mac=fb.MacConfig(c.mac, c.theta), p=c.p, mutual=True, task_grain=c.grain, **kw)


@pytest.fixture(scope="module", params=MU_CASES)
def case(request):
    return MuCase(request.param)


def test_partition_owner_matches_roots(case):
    from paper_1209_3516_b200.traversal import partition_owner
    t = build(case)
    owner = partition_owner(t, case.grain).cpu().numpy()
    roots = np.flatnonzero(owner == np.arange(t.ncells))
    assert np.array_equal(roots, case["roots"])


def test_mutual_lists_bit_exact(case):
    t = build(case)
    lists = fb.mutual_lists(t, fb.MacConfig(case.mac, case.theta), case.grain)
    assert lists.n_m2l == case.meta["n_m2l"] and lists.n_p2p == case.meta["n_p2p"]
    assert sha(canon_pairs(*lists.host_pairs("m2l"))) == case.meta["m2l_sha"]
    assert sha(canon_pairs(*lists.host_pairs("p2p"))) == case.meta["p2p_sha"]


def test_mutual_fp64_matches_reference(case):
    t = build(case)
    rep = fb.evaluate_on_tree(t, cfg_of(case), trace=True)
    assert rep.mutual and rep.task_grain == case.grain
    s = case.meta["stats"]
    for k in STAT_KEYS:
        assert getattr(rep.stats, k) == s[k], k
    ev_m = canon_pairs([a for k, a, _ in rep.trace if k == "m2l"], [b for k, _, b in rep.trace if k == "m2l"])
    assert sha(ev_m) == case.meta["m2l_sha"]
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(t.bodies, k), case[k]) <= FP64_TOL, k


def test_mutual_fp32_within_twice_reference_error(case):
    t = build(case)
    rep = fb.evaluate_on_tree(t, cfg_of(case, precision="fp32"))
    s = case.meta["stats"]
    assert rep.stats.p2p_pairs == s["p2p_pairs"] and rep.stats.p2p_skipped == s["p2p_skipped"]
    fref = np.stack([case["direct_fx"], case["direct_fy"], case["direct_fz"]], 1)

    def err(fx, fy, fz):
        f = np.stack([fx, fy, fz], 1)
        return float(np.sqrt(((f - fref) ** 2).sum() / (fref ** 2).sum()))

    ref = err(case["fx"], case["fy"], case["fz"])
    b = t.bodies
    got = err(b.fx, b.fy, b.fz)
    assert got <= 2.0 * ref + FP32_BAR_FLOOR, (got, ref)
    assert rel_l2(b.phi, case["direct_phi"]) <= 2.0 * rel_l2(case["phi"], case["direct_phi"]) + FP32_BAR_FLOOR


@pytest.mark.parametrize("grain", [1, 37, 250, 10 ** 9])
@pytest.mark.parametrize("mac", ["fmm", "bh"])
def test_mutual_lists_match_oracle_at_other_grains(grain, mac):
    c = MuCase("c1_4k_g700")
    t = build(c)
    ot = orc.build_tree(c.pos, c.q, c.ncrit)
    lists = fb.mutual_lists(t, fb.MacConfig(mac, 0.55), grain)
    mt, ms, mm, pt, ps, pm = orc.collect_mutual(ot, 0.55, grain, mac)
    assert np.array_equal(canon_pairs(*lists.host_pairs("m2l")), canon_pairs(*orc.expand_mutual(mt, ms, mm)))
    assert np.array_equal(canon_pairs(*lists.host_pairs("p2p")), canon_pairs(*orc.expand_mutual(pt, ps, pm)))


def test_mutual_body_range_partition():
    """Per-range mutual lists (a multi-GPU rank's share) partition the P2P
    list and cover the M2L list (shared top cells repeat on both ranks)."""
    c = MuCase("c1_4k_g700")
    t = build(c)
    mac = fb.MacConfig(c.mac, c.theta)
    full = fb.mutual_lists(t, mac, c.grain)
    full_p = canon_pairs(*full.host_pairs("p2p"))
    full_m = canon_pairs(*full.host_pairs("m2l"))
    leaf_starts = np.sort(t.cell_start[t.cell_leaf.astype(bool)])
    cut = int(leaf_starts[leaf_starts.size // 2])
    parts_p, parts_m = [], []
    for rng in ((0, cut), (cut, t.n)):
        lists = fb.mutual_lists(t, mac, c.grain, body_range=rng)
        parts_p.append(canon_pairs(*lists.host_pairs("p2p")))
        parts_m.append(canon_pairs(*lists.host_pairs("m2l")))
    assert np.array_equal(np.sort(np.concatenate(parts_p)), full_p)
    assert np.array_equal(np.unique(np.concatenate(parts_m)), full_m)


def test_mutual_as_accurate_as_directed():
    """tests/test_traversal.py:117-125 of the reference, on the GPU."""
    c = MuCase("c1_4k_g700")
    t = build(c)
    fb.evaluate_on_tree(t, fb.EvalConfig(mac=fb.MacConfig("fmm", 0.6), p=4))
    d = np.stack([t.bodies.fx, t.bodies.fy, t.bodies.fz], 1).copy()
    fb.evaluate_on_tree(t, fb.EvalConfig(mac=fb.MacConfig("fmm", 0.6), p=4, mutual=True, task_grain=700))
    m = np.stack([t.bodies.fx, t.bodies.fy, t.bodies.fz], 1)
    ref = np.stack([c["direct_fx"], c["direct_fy"], c["direct_fz"]], 1)
    e = lambda f: float(np.sqrt(((f - ref) ** 2).sum() / (ref ** 2).sum()))  # noqa: E731
    assert e(m) < 2.0 * e(d) + 1e-12
    assert torch.cuda.is_available()


# ---- symmetric executors (fmm_traverse_mutual_sym, fmm_p2p_sym) -------------
# The reference's _p2p_mutual (src/_taylor.py:410-449) evaluates an unordered
# leaf pair once and adds it to both leaves; here the unordered pairs run on
# the symmetric GPU kernel and must reproduce the reference's sets, counters
# and results.

def test_symmetric_lists_expand_to_reference_sets(case):
    t = build(case)
    lists = fb.mutual_lists(t, fb.MacConfig(case.mac, case.theta), case.grain, symmetric=True)
    assert lists.n_m2l == case.meta["n_m2l"] and lists.n_p2p == case.meta["n_p2p"]
    assert sha(canon_pairs(*lists.host_pairs("m2l"))) == case.meta["m2l_sha"]
    assert sha(canon_pairs(*lists.host_pairs("p2p"))) == case.meta["p2p_sha"]
    sym = lists.sym_p2p
    a, b = sym.pairs()
    assert sym.n == a.numel() and bool((a < b).all())
    leaf = t.cell_leaf.astype(bool)
    assert leaf[a.numpy()].all() and leaf[b.numpy()].all()


def test_symmetric_unordered_pairs_match_oracle():
    """The unordered list is the oracle's mutual P2P entries of two distinct
    leaves (both members kept)."""
    c = MuCase("c1_4k_g700")
    t = build(c)
    ot = orc.build_tree(c.pos, c.q, c.ncrit)
    for grain in (37, 700, 10 ** 9):
        lists = fb.mutual_lists(t, fb.MacConfig("fmm", 0.55), grain, symmetric=True)
        _, _, _, pt, ps, pm = orc.collect_mutual(ot, 0.55, grain, "fmm")
        keep = (pm != 0) & (pt != ps)
        want = np.unique(np.stack([np.minimum(pt[keep], ps[keep]), np.maximum(pt[keep], ps[keep])], 1), axis=0)
        a, b = lists.sym_p2p.pairs()
        got = np.unique(np.stack([a.numpy(), b.numpy()], 1), axis=0)
        assert lists.sym_p2p.n == len(want) and np.array_equal(got, want)
        assert grain < 10 ** 9 or lists.sym_p2p.n > 0


def test_symmetric_fp64_matches_reference(case):
    t = build(case)
    rep = fb.evaluate_on_tree(t, cfg_of(case, symmetric=True), trace=True)
    s = case.meta["stats"]
    for k in STAT_KEYS:
        assert getattr(rep.stats, k) == s[k], k
    ev_p = canon_pairs([a for k, a, _ in rep.trace if k == "p2p"], [b for k, _, b in rep.trace if k == "p2p"])
    assert sha(ev_p) == case.meta["p2p_sha"]
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(t.bodies, k), case[k]) <= FP64_TOL, k


def test_symmetric_fp32_within_twice_reference_error(case):
    t = build(case)
    rep = fb.evaluate_on_tree(t, cfg_of(case, precision="fp32", symmetric=True))
    s = case.meta["stats"]
    assert rep.stats.p2p_pairs == s["p2p_pairs"] and rep.stats.p2p_skipped == s["p2p_skipped"]
    fref = np.stack([case["direct_fx"], case["direct_fy"], case["direct_fz"]], 1)

    def err(fx, fy, fz):
        f = np.stack([fx, fy, fz], 1)
        return float(np.sqrt(((f - fref) ** 2).sum() / (fref ** 2).sum()))

    ref = err(case["fx"], case["fy"], case["fz"])
    b = t.bodies
    assert err(b.fx, b.fy, b.fz) <= 2.0 * ref + FP32_BAR_FLOOR
    assert rel_l2(b.phi, case["direct_phi"]) <= 2.0 * rel_l2(case["phi"], case["direct_phi"]) + FP32_BAR_FLOOR


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_symmetric_is_deterministic_and_equals_directed(precision):
    """Two symmetric runs agree bit for bit (no atomics); the symmetric and
    the directed executors agree to rounding."""
    c = MuCase("c1_4k_g700")
    t = build(c)
    cfg = lambda sym: fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=4, mutual=True, task_grain=10 ** 9,  # noqa: E731
                                    precision=precision, symmetric=sym)
    runs = []
    for sym in (True, True, False):
        rep = fb.evaluate_on_tree(t, cfg(sym))
        b = t.bodies
        runs.append((rep.stats.p2p_pairs, np.stack([b.phi, b.fx, b.fy, b.fz]).copy()))
    assert runs[0][0] == runs[1][0] == runs[2][0]
    assert np.array_equal(runs[0][1], runs[1][1])
    tol = 1e-12 if precision == "fp64" else 2e-5
    for k in range(4):
        assert rel_l2(runs[0][1][k], runs[2][1][k]) <= tol, k


@pytest.mark.parametrize("ncrit", [8, 100, 300])
def test_symmetric_other_leaf_sizes_match_oracle(ncrit):
    """Leaves beyond one 64-target sweep (ncrit 100, 300) and tiny leaves."""
    from paper_1209_3516_b200 import workloads
    pos, q = workloads.config1(3000, 5)
    t = fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q), ncrit=ncrit)
    ot = orc.build_tree(pos, q, ncrit)
    want = orc.evaluate_mutual(ot, 3, 0.5, 10 ** 9)
    rep = fb.evaluate_on_tree(t, fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=3, mutual=True, task_grain=10 ** 9,
                                               symmetric=True))
    assert rep.stats.p2p_pairs == want["p2p_pairs"]
    assert t.list_cache.sym_p2p.n > 0
    b = t.bodies
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(b, k), want[k]) <= FP64_TOL, k


def test_symmetric_chunked_reaction_buffer(monkeypatch):
    """A reaction buffer smaller than the list sweeps the first leaves in
    chunks: same results to rounding, same counters."""
    from paper_1209_3516_b200 import traversal
    c = MuCase("c1_4k_g700")
    t = build(c)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=4, mutual=True, task_grain=10 ** 9, symmetric=True)
    rep0 = fb.evaluate_on_tree(t, cfg)
    whole = np.stack([t.bodies.phi, t.bodies.fx, t.bodies.fy, t.bodies.fz]).copy()
    assert len(t.list_cache.sym_p2p.chunks[1]) == 2
    monkeypatch.setattr(traversal, "SYM_BUFFER_BYTES", 64 << 10)
    rep1 = fb.evaluate_on_tree(t, cfg)
    assert len(t.list_cache.sym_p2p.chunks[1]) > 3
    assert rep1.stats.p2p_pairs == rep0.stats.p2p_pairs
    got = np.stack([t.bodies.phi, t.bodies.fx, t.bodies.fy, t.bodies.fz])
    for k in range(4):
        assert rel_l2(got[k], whole[k]) <= 1e-13, k


def test_symmetric_multirank_ranges_sum_to_whole():
    """Per-range symmetric lists (both members kept stay unordered, the rest
    directed) expand to the same directed set as the whole."""
    c = MuCase("c1_4k_g700")
    t = build(c)
    mac = fb.MacConfig(c.mac, c.theta)
    full = canon_pairs(*fb.mutual_lists(t, mac, c.grain).host_pairs("p2p"))
    leaf_starts = np.sort(t.cell_start[t.cell_leaf.astype(bool)])
    cut = int(leaf_starts[leaf_starts.size // 2])
    parts = [canon_pairs(*fb.mutual_lists(t, mac, c.grain, body_range=rng, symmetric=True).host_pairs("p2p"))
             for rng in ((0, cut), (cut, t.n))]
    assert np.array_equal(np.sort(np.concatenate(parts)), full)


# ---- symmetric M2L (fmm_m2l_sym, the reference's _m2l_mutual) ---------------

def test_symmetric_m2l_lists_expand_to_reference_sets(case):
    t = build(case)
    lists = fb.mutual_lists(t, fb.MacConfig(case.mac, case.theta), case.grain, symmetric=True, symmetric_m2l=True)
    assert lists.n_m2l == case.meta["n_m2l"] and lists.n_p2p == case.meta["n_p2p"]
    assert sha(canon_pairs(*lists.host_pairs("m2l"))) == case.meta["m2l_sha"]
    assert sha(canon_pairs(*lists.host_pairs("p2p"))) == case.meta["p2p_sha"]
    a, b = lists.sym_m2l.pairs()
    assert lists.sym_m2l.n == a.numel() and bool((a < b).all())


def test_symmetric_m2l_unordered_pairs_match_oracle():
    """The unordered M2L list is the oracle's mutual M2L entries."""
    c = MuCase("c1_4k_g700")
    t = build(c)
    ot = orc.build_tree(c.pos, c.q, c.ncrit)
    for grain in (37, 700, 10 ** 9):
        lists = fb.mutual_lists(t, fb.MacConfig("fmm", 0.55), grain, symmetric=True, symmetric_m2l=True)
        mt, ms, mm, _, _, _ = orc.collect_mutual(ot, 0.55, grain, "fmm")
        keep = (mm != 0) & (mt != ms)
        want = np.unique(np.stack([np.minimum(mt[keep], ms[keep]), np.maximum(mt[keep], ms[keep])], 1), axis=0)
        a, b = lists.sym_m2l.pairs()
        got = np.unique(np.stack([a.numpy(), b.numpy()], 1), axis=0)
        assert lists.sym_m2l.n == len(want) and np.array_equal(got, want)
        assert grain < 10 ** 9 or lists.sym_m2l.n > 0


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_symmetric_m2l_orders_match_oracle(p):
    """Every order of the symmetric M2L kernel (1..7) against the oracle's
    _m2l_mutual; p = 8 keeps the M2L pairs directed (grouped tensor kernel)."""
    from paper_1209_3516_b200 import workloads
    pos, q = workloads.config1(3000, 9)
    t = fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q), ncrit=16)
    ot = orc.build_tree(pos, q, 16)
    want = orc.evaluate_mutual(ot, p, 0.5, 10 ** 9)
    rep = fb.evaluate_on_tree(t, fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=p, mutual=True, task_grain=10 ** 9,
                                               symmetric=True))
    assert rep.stats.m2l_calls == want["m2l_calls"] and rep.stats.p2p_pairs == want["p2p_pairs"]
    sym = t.list_cache.__dict__.get("sym_m2l")
    assert (sym is not None and sym.n > 0) if p <= 7 else sym is None
    b = t.bodies
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(b, k), want[k]) <= FP64_TOL, k


def test_symmetric_m2l_locals_deterministic_and_equal_directed():
    """The locals after M2L: two symmetric runs agree bit for bit; against
    the directed M2L of the same pairs they agree to rounding."""
    from paper_1209_3516_b200.traversal import run_m2l, run_m2l_sym
    from paper_1209_3516_b200.tree import upward_pass
    c = MuCase("c1_4k_g700")
    t = build(c)
    p, mac = 5, fb.MacConfig("fmm", 0.5)
    upward_pass(t, p)
    out = []
    for sym in (True, True, False):
        lists = fb.mutual_lists(t, mac, 10 ** 9, symmetric=True, symmetric_m2l=sym)
        t._L = torch.zeros_like(t._M)
        run_m2l(t, lists, p)
        run_m2l_sym(t, lists, p)
        torch.cuda.synchronize()
        out.append(t._L.cpu().numpy().copy())
    assert np.array_equal(out[0], out[1])
    assert np.abs(out[0]).max() > 0
    assert np.abs(out[0] - out[2]).max() <= 1e-12 * np.abs(out[2]).max()


def test_symmetric_m2l_chunked_reaction_buffer(monkeypatch):
    from paper_1209_3516_b200 import traversal
    c = MuCase("c1_4k_g700")
    t = build(c)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=4, mutual=True, task_grain=10 ** 9, symmetric=True)
    rep0 = fb.evaluate_on_tree(t, cfg)
    whole = np.stack([t.bodies.phi, t.bodies.fx, t.bodies.fy, t.bodies.fz]).copy()
    nsym = t.list_cache.sym_m2l.n
    assert nsym * 35 * 8 > 8 * (16 << 10)
    monkeypatch.setattr(traversal, "SYM_BUFFER_BYTES", 16 << 10)
    rep1 = fb.evaluate_on_tree(t, cfg)
    assert rep1.stats.m2l_calls == rep0.stats.m2l_calls
    got = np.stack([t.bodies.phi, t.bodies.fx, t.bodies.fy, t.bodies.fz])
    for k in range(4):
        assert rel_l2(got[k], whole[k]) <= 1e-13, k
