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
