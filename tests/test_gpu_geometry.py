"""rect / center-of-mass trees on the B200 vs the
reference's fixtures (tests/golden/make_golden_geometry.py): every cell
array bit-exact, the dual-tree pair sets and counters bit-exact, and the
dual-tree and treecode FP64 results within 1e-11."""

import numpy as np
import pytest

import paper_1209_3516_b200 as fb
from goldens import GEO_CASES, GeoCase, canon_pairs, rel_l2, sha

pytestmark = pytest.mark.gpu
FIELDS = ("children", "parent", "level", "key", "start", "end", "sub_end", "lo", "hi", "center", "bmax", "rmax",
          "leaf")
DT = dict(children=np.int32, parent=np.int32, level=np.int8, key=np.uint64, start=np.int32, end=np.int32,
          sub_end=np.int32, leaf=np.uint8)


@pytest.fixture(scope="module", params=GEO_CASES)
def case(request):
    return GeoCase(request.param)


def build(c):
    pos = np.asarray(c.pos, np.float64)
    return fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q), ncrit=c.ncrit, shape=c.shape,
                         center_mode=c.center_mode)


def test_geometry_bit_exact(case):
    t = build(case)
    assert t.shape == case.shape and t.center_mode == case.center_mode
    for f in FIELDS:
        got = np.ascontiguousarray(getattr(t, "cell_" + f)).astype(DT.get(f, np.float64))
        assert sha(got) == case.meta["cells_sha"][f], f


def test_lists_and_results(case):
    t = build(case)
    lists = fb.interaction_lists(t, fb.MacConfig("fmm", case.theta))
    assert sha(canon_pairs(*lists.host_pairs("m2l"))) == case.meta["m2l_sha"]
    assert sha(canon_pairs(*lists.host_pairs("p2p"))) == case.meta["p2p_sha"]
    for strategy in ("dualtree", "treecode"):
        rep = fb.evaluate_on_tree(t, fb.EvalConfig(strategy=strategy, mac=fb.MacConfig("fmm", case.theta),
                                                   p=case.p))
        s = case.meta["stats_" + strategy]
        for k in ("p2p_pairs", "p2p_skipped", "m2l_calls", "m2p_calls"):
            assert getattr(rep.stats, k) == s[k], (strategy, k)
        b = t.bodies
        for k in ("phi", "fx", "fy", "fz"):
            want = case[f"{strategy}_{k}"]
            got = getattr(b, k)
            if np.any(want):
                assert rel_l2(got, want) <= 1e-11, (strategy, k)
            else:
                assert not np.any(got), (strategy, k)


def test_listfmm_needs_cubic():
    c = GeoCase(next(k for k in GEO_CASES if GeoCase(k).shape == "rect"))
    t = build(c)
    with pytest.raises(ValueError, match="cubic"):
        fb.evaluate_on_tree(t, fb.EvalConfig(strategy="listfmm"))


def test_lists_exact_after_a_capacity_hint_from_another_tree():
    """A tree with the same cell and leaf counts but other centres (geometric
    instead of centre-of-mass) leaves a capacity hint behind its evaluation;
    the public list builder must not take it on trust (it sizes exactly), and
    an evaluation that does take it must notice the overflow and redo."""
    c = GeoCase("clustered3k_cubic_com")
    pos = np.asarray(c.pos, np.float64)
    mac = fb.MacConfig("fmm", c.theta)
    other = fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q), ncrit=c.ncrit, shape=c.shape,
                          center_mode="geometric")
    for _ in range(2):  # the second evaluation runs from (and refreshes) the hint
        fb.evaluate_on_tree(other, fb.EvalConfig(mac=mac, p=c.p))
    t = build(c)
    assert (t.ncells, t.nleaves) == (other.ncells, other.nleaves)
    lists = fb.interaction_lists(t, mac)
    assert sha(canon_pairs(*lists.host_pairs("m2l"))) == c.meta["m2l_sha"]
    assert sha(canon_pairs(*lists.host_pairs("p2p"))) == c.meta["p2p_sha"]
    rep = fb.evaluate_on_tree(t, fb.EvalConfig(mac=mac, p=c.p))
    for k in ("p2p_pairs", "m2l_calls"):
        assert getattr(rep.stats, k) == c.meta["stats_dualtree"][k], k
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(t.bodies, k), c[f"dualtree_{k}"]) <= 1e-11, k
