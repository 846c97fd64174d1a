"""Cross-tree evaluation on the B200 (targets of one tree, sources of
another) vs the reference's cross-tree goldens
(tests/golden/make_golden_cross.py, src/traversal.py:864-932 and
:1002-1046 with ``source_tree``).

Bit-exact: the M2L / M2P / P2P pair sets and the reference's counters
(coincident target/source bodies skipped and counted).  FP64 results within
1e-11 relative L2 of the reference's; FP32 near field within 2x the
reference's own error against direct summation.
"""

import numpy as np
import pytest
import torch

import paper_1209_3516_b200 as fb
from goldens import FP32_BAR_FLOOR, CX_CASES, CxCase, canon_pairs, rel_l2, sha

pytestmark = pytest.mark.gpu
FP64_TOL = 1e-11
STAT_KEYS = ("p2p_pairs", "p2p_skipped", "p2p_flops", "m2l_calls", "m2p_calls", "p2m_calls", "m2m_calls",
             "l2l_calls", "l2p_calls")


def _tree(pos, q, ncrit):
    pos = np.asarray(pos, np.float64)
    return fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q), ncrit=ncrit)


def trees(c: CxCase):
    return _tree(c.pa, c.qa, c.ncrit_a), _tree(c.pb, c.qb, c.ncrit_b)


@pytest.fixture(scope="module", params=CX_CASES)
def case(request):
    return CxCase(request.param)


def test_cross_dual_lists_bit_exact(case):
    A, B = trees(case)
    lists = fb.interaction_lists(A, fb.MacConfig("fmm", case.theta), src=B)
    assert lists.n_m2l == case.meta["n_m2l"] and lists.n_p2p == case.meta["n_p2p"]
    assert sha(canon_pairs(*lists.host_pairs("m2l"))) == case.meta["m2l_sha"]
    assert sha(canon_pairs(*lists.host_pairs("p2p"))) == case.meta["p2p_sha"]


def test_cross_treecode_lists_bit_exact(case):
    A, B = trees(case)
    lists = fb.treecode_lists(A, fb.MacConfig("fmm", case.theta), src=B)
    assert lists.n_m2p == case.meta["n_m2p"] and lists.n_p2p == case.meta["tc_p2p_n"]
    assert sha(canon_pairs(*lists.host_pairs("m2p"))) == case.meta["m2p_sha"]
    assert sha(canon_pairs(*lists.host_pairs("p2p"))) == case.meta["tc_p2p_sha"]


@pytest.mark.parametrize("strategy", ["dualtree", "treecode"])
def test_cross_fp64_matches_reference(case, strategy):
    A, B = trees(case)
    cfg = fb.EvalConfig(strategy=strategy, mac=fb.MacConfig("fmm", case.theta), p=case.p)
    rep = fb.evaluate_on_tree(A, cfg, source_tree=B)
    assert rep.n == A.n and rep.n_sources == B.n
    assert rep.build_time == pytest.approx(A.build_time + B.build_time)
    s = case.meta["stats_" + strategy]
    for k in STAT_KEYS:
        assert getattr(rep.stats, k) == s[k], k
    b = A.bodies
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(b, k), case[f"{strategy}_{k}"]) <= FP64_TOL, k
    # the source tree's own accumulators are untouched
    sb = B.bodies
    assert not np.any(sb.phi) and not np.any(sb.fx)


@pytest.mark.parametrize("strategy", ["dualtree", "treecode"])
def test_cross_fp32_within_twice_reference_error(case, strategy):
    A, B = trees(case)
    cfg = fb.EvalConfig(strategy=strategy, mac=fb.MacConfig("fmm", case.theta), p=case.p, precision="fp32")
    rep = fb.evaluate_on_tree(A, cfg, source_tree=B)
    s = case.meta["stats_" + strategy]
    assert rep.stats.p2p_pairs == s["p2p_pairs"] and rep.stats.p2p_skipped == s["p2p_skipped"]
    b = A.bodies
    fref = np.stack([case["direct_fx"], case["direct_fy"], case["direct_fz"]], 1)

    def errs(fx, fy, fz, phi):
        f = np.stack([fx, fy, fz], 1)
        return float(np.sqrt(((f - fref) ** 2).sum() / (fref ** 2).sum())), rel_l2(phi, case["direct_phi"])

    ref_f, ref_p = errs(*(case[f"{strategy}_{k}"] for k in ("fx", "fy", "fz", "phi")))
    got_f, got_p = errs(b.fx, b.fy, b.fz, b.phi)
    assert got_f <= 2.0 * ref_f + FP32_BAR_FLOOR, (got_f, ref_f)
    assert got_p <= 2.0 * ref_p + FP32_BAR_FLOOR, (got_p, ref_p)


def test_cross_chunked_matches_one_pass(monkeypatch):
    """Target chunks (FMM_B200_CHUNKS) partition the cross lists exactly."""
    c = CxCase("uniform_vs_clustered")
    A, B = trees(c)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", c.theta), p=c.p)
    monkeypatch.setenv("FMM_B200_CHUNKS", "3")
    rep = fb.evaluate_on_tree(A, cfg, source_tree=B)
    for k in STAT_KEYS:
        assert getattr(rep.stats, k) == c.meta["stats_dualtree"][k], k
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(A.bodies, k), c["dualtree_" + k]) <= FP64_TOL, k


def test_cross_then_self_keeps_expansions_consistent():
    """A cross evaluation at order p leaves the target tree usable for a
    self evaluation at another order (no stale multipoles of the wrong p)."""
    c = CxCase("inside_bigger")
    A, B = trees(c)
    fb.evaluate_on_tree(A, fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=6), source_tree=B)
    fb.evaluate_on_tree(A, fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=3))
    got = [getattr(A.bodies, k).copy() for k in ("phi", "fx", "fy", "fz")]
    A2, _ = trees(c)
    fb.evaluate_on_tree(A2, fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=3))
    for g, k in zip(got, ("phi", "fx", "fy", "fz")):
        assert np.array_equal(g, getattr(A2.bodies, k)), k
    # and the source tree's cached order-6 multipoles are reused as-is
    rep = fb.evaluate_on_tree(A, fb.EvalConfig(mac=fb.MacConfig("fmm", c.theta), p=6), source_tree=B)
    assert rep.stats.p2m_calls == 0 and rep.stats.m2m_calls == 0


def test_cross_mutual_rejected_like_reference():
    c = CxCase("coincident")
    A, B = trees(c)
    with pytest.raises(ValueError, match="share one tree"):
        fb.evaluate_dual_tree(A, fb.EvalConfig(mutual=True), source_tree=B)


def test_cross_source_tree_of_itself_is_self_evaluation():
    c = CxCase("coincident")
    A, _ = trees(c)
    rep = fb.evaluate_on_tree(A, fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=4), source_tree=A)
    A2, _ = trees(c)
    rep2 = fb.evaluate_on_tree(A2, fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=4))
    assert rep.stats.p2p_pairs == rep2.stats.p2p_pairs
    assert np.array_equal(A.bodies.phi, A2.bodies.phi)
    assert torch.cuda.is_available()
