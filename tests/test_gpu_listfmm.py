"""listfmm strategy on the B200 vs the reference's
listfmm goldens (tests/golden/make_golden_listfmm.py) and the C oracle.

Bit-exact: the V (M2L) and U (P2P) pair sets and the reference's counters.
FP64 results within 1e-11 relative L2; FP32 near field within 2x the
reference's own error against direct summation."""

import numpy as np
import pytest

import paper_1209_3516_b200 as fb
from goldens import FP32_BAR_FLOOR, LF_CASES, LfCase, canon_pairs, rel_l2, sha

pytestmark = pytest.mark.gpu
FP64_TOL = 1e-11


def build(c):
    pos = np.asarray(c.pos, np.float64)
    return fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q), ncrit=c.ncrit)


@pytest.fixture(scope="module", params=LF_CASES)
def case(request):
    return LfCase(request.param)


def test_listfmm_lists_bit_exact(case):
    t = build(case)
    lists = fb.listfmm_lists(t)
    assert lists.n_m2l == case.meta["n_m2l"] and lists.n_p2p == case.meta["n_p2p"]
    assert sha(canon_pairs(*lists.host_pairs("m2l"))) == case.meta["m2l_sha"]
    assert sha(canon_pairs(*lists.host_pairs("p2p"))) == case.meta["p2p_sha"]
    pairs, skipped = lists.dev_stats.tolist()
    assert pairs == case.meta["stats"]["p2p_pairs"] and skipped == case.meta["stats"]["p2p_skipped"]


def test_listfmm_fp64_matches_reference(case):
    t = build(case)
    rep = fb.evaluate_on_tree(t, fb.EvalConfig(strategy="listfmm", p=case.p))
    assert rep.strategy == "listfmm"
    for k in ("p2p_pairs", "p2p_skipped", "p2p_flops", "m2l_calls", "p2m_calls", "m2m_calls", "l2l_calls",
              "l2p_calls"):
        assert getattr(rep.stats, k) == case.meta["stats"][k], k
    b = t.bodies
    idx = case["direct_idx"]
    for k in ("phi", "fx", "fy", "fz"):
        if case.has(k):
            assert rel_l2(getattr(b, k), case[k]) <= FP64_TOL, k
        else:
            assert rel_l2(getattr(b, k)[idx], case["sample_" + k]) <= FP64_TOL, k


def test_listfmm_fp32_within_twice_reference_error(case):
    t = build(case)
    fb.evaluate_on_tree(t, fb.EvalConfig(strategy="listfmm", p=case.p, precision="fp32"))
    idx = case["direct_idx"]
    b = t.bodies
    fref = np.stack([case["direct_fx"], case["direct_fy"], case["direct_fz"]], 1)
    fgot = np.stack([b.fx[idx], b.fy[idx], b.fz[idx]], 1)
    ferr = float(np.sqrt(((fgot - fref) ** 2).sum() / (fref ** 2).sum()))
    perr = rel_l2(b.phi[idx], case["direct_phi"])
    assert ferr <= 2.0 * case.meta["force_err"] + FP32_BAR_FLOOR, (ferr, case.meta["force_err"])
    assert perr <= 2.0 * case.meta["pot_err"] + FP32_BAR_FLOOR, (perr, case.meta["pot_err"])
