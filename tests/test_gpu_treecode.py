"""Treecode strategy on the B200 vs the reference's
treecode goldens (tests/golden/make_golden_treecode.py) and the C oracle.

Bit-exact: the M2P and P2P pair sets and the reference's counters.  FP64
numerics (M2P alone, and the full evaluate_treecode output) within 1e-11
relative L2; FP32 near field within 2x the reference's own error against
direct summation.
"""

import numpy as np
import pytest
import torch

import paper_1209_3516_b200 as fb
from goldens import FP32_BAR_FLOOR, TC_CASES, TcCase, canon_pairs, rel_l2, sha
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
FP64_TOL = 1e-11


def build(c: TcCase):
    pos = np.asarray(c.pos, np.float64)
    return fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q), ncrit=c.ncrit)


@pytest.fixture(scope="module", params=TC_CASES)
def case(request):
    return TcCase(request.param)


def test_treecode_lists_bit_exact(case):
    t = build(case)
    lists = fb.treecode_lists(t, fb.MacConfig("fmm", case.theta))
    mt, ms = lists.host_pairs("m2p")
    pt, ps = lists.host_pairs("p2p")
    assert lists.n_m2p == case.meta["n_m2p"] and lists.n_p2p == case.meta["n_p2p"]
    assert sha(canon_pairs(mt, ms)) == case.meta["m2p_sha"]
    assert sha(canon_pairs(pt, ps)) == case.meta["p2p_sha"]
    pairs, skipped = lists.dev_stats.tolist()
    assert pairs == case.meta["stats"]["p2p_pairs"] and skipped == case.meta["stats"]["p2p_skipped"]


def test_m2p_fp64_only(case):
    """M2P alone on zeroed accumulators vs the reference's _exec_m2p."""
    t = build(case)
    fb.upward_pass(t, case.p)
    from paper_1209_3516_b200.traversal import run_m2p
    lists = fb.treecode_lists(t, fb.MacConfig("fmm", case.theta))
    out = torch.zeros((4, t.n), dtype=torch.float64, device="cuda")
    run_m2p(t, lists, case.p, tuple(out))
    got = out.cpu().numpy()  # tree (Morton) order, like the golden
    if case.has("m2p_phi"):
        for k, g in zip(("phi", "fx", "fy", "fz"), got):
            assert rel_l2(g, case["m2p_" + k]) <= FP64_TOL, k
    else:
        for g, want in zip(got, case.meta["m2p_norm"]):
            assert abs(np.linalg.norm(g) - want) <= FP64_TOL * max(want, 1e-300)


def test_m2p_fp32(case):
    """precision="fp32" M2P (float32 terms for p <= 6, float64 above) against
    the reference's _exec_m2p: float32 rounding of D and the moments, far
    below the expansion's truncation error."""
    if not case.has("m2p_phi"):
        pytest.skip("no stored M2P-only sums for this case")
    t = build(case)
    fb.upward_pass(t, case.p)
    from paper_1209_3516_b200.traversal import run_m2p
    lists = fb.treecode_lists(t, fb.MacConfig("fmm", case.theta))
    out = torch.zeros((4, t.n), dtype=torch.float64, device="cuda")
    run_m2p(t, lists, case.p, tuple(out), precision="fp32")
    got = out.cpu().numpy()
    tol = 2e-5 if case.p <= 6 else FP64_TOL
    for k, g in zip(("phi", "fx", "fy", "fz"), got):
        assert rel_l2(g, case["m2p_" + k]) <= tol, k


def test_treecode_fp64_matches_reference(case):
    t = build(case)
    cfg = fb.EvalConfig(strategy="treecode", mac=fb.MacConfig("fmm", case.theta), p=case.p)
    rep = fb.evaluate_on_tree(t, cfg)
    assert rep.strategy == "treecode" and rep.downward_time == 0.0
    s = case.meta["stats"]
    for k in ("p2p_pairs", "p2p_skipped", "p2p_flops", "m2p_calls", "m2l_calls", "p2m_calls", "m2m_calls"):
        assert getattr(rep.stats, k) == s[k], k
    b = t.bodies
    if case.has("phi"):
        for k in ("phi", "fx", "fy", "fz"):
            assert rel_l2(getattr(b, k), case[k]) <= FP64_TOL, k
    else:
        idx = case["direct_idx"]
        for k in ("phi", "fx", "fy", "fz"):
            assert rel_l2(getattr(b, k)[idx], case["sample_" + k]) <= FP64_TOL, k


def test_treecode_fp32_within_twice_reference_error(case):
    t = build(case)
    fb.evaluate_on_tree(t, fb.EvalConfig(strategy="treecode", mac=fb.MacConfig("fmm", case.theta), p=case.p,
                                         precision="fp32"))
    idx = case["direct_idx"]
    b = t.bodies
    fref = np.stack([case["direct_fx"], case["direct_fy"], case["direct_fz"]], 1)
    fgot = np.stack([b.fx[idx], b.fy[idx], b.fz[idx]], 1)
    ferr = float(np.sqrt(((fgot - fref) ** 2).sum() / (fref ** 2).sum()))
    perr = rel_l2(b.phi[idx], case["direct_phi"])
    assert ferr <= 2.0 * case.meta["force_err"] + FP32_BAR_FLOOR, (ferr, case.meta["force_err"])
    assert perr <= 2.0 * case.meta["pot_err"] + FP32_BAR_FLOOR, (perr, case.meta["pot_err"])


def test_treecode_matches_oracle_at_other_mac_inputs():
    """A second theta on the C1 tree, checked against the oracle's walk."""
    c = TcCase("c1")
    t = build(c)
    ot = orc.build_tree(c.pos, c.q, c.ncrit, False)
    for theta in (0.3, 0.8):
        lists = fb.treecode_lists(t, fb.MacConfig("fmm", theta))
        mt, ms, pt, ps = orc.collect_treecode(ot, theta)
        assert np.array_equal(canon_pairs(*lists.host_pairs("m2p")), canon_pairs(mt, ms))
        assert np.array_equal(canon_pairs(*lists.host_pairs("p2p")), canon_pairs(pt, ps))


def test_treecode_body_range_partition():
    """Per-range walks (a multi-GPU rank's share) union to the full lists."""
    c = TcCase("c1")
    t = build(c)
    mac = fb.MacConfig("fmm", c.theta)
    full_m = canon_pairs(*fb.treecode_lists(t, mac).host_pairs("m2p"))
    full_p = canon_pairs(*fb.treecode_lists(t, mac).host_pairs("p2p"))
    start = t.cell_start
    leaf_starts = np.sort(start[t.cell_leaf.astype(bool)])
    cut = int(leaf_starts[leaf_starts.size // 2])
    parts_m, parts_p = [], []
    for rng in ((0, cut), (cut, t.n)):
        lists = fb.treecode_lists(t, mac, body_range=rng)
        parts_m.append(canon_pairs(*lists.host_pairs("m2p")))
        parts_p.append(canon_pairs(*lists.host_pairs("p2p")))
    assert np.array_equal(np.sort(np.concatenate(parts_m)), full_m)
    assert np.array_equal(np.sort(np.concatenate(parts_p)), full_p)
