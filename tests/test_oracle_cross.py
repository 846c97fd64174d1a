"""Pin the oracle's cross-tree restatement (two-tree dual traversal and
treecode walk, cross M2L, _p2p_cross) to the reference's cross-tree goldens
(tests/golden/make_golden_cross.py)."""

import numpy as np
import pytest

from goldens import CX_CASES, CxCase, canon_pairs, rel_l2, sha
from oracle import oracle as orc


@pytest.fixture(scope="module", params=CX_CASES)
def trees(request):
    c = CxCase(request.param)
    return c, orc.build_tree(c.pa, c.qa, c.ncrit_a), orc.build_tree(c.pb, c.qb, c.ncrit_b)


def test_cross_dual_lists_and_result(trees):
    c, A, B = trees
    r = orc.evaluate_cross(A, B, c.p, c.theta)
    assert sha(canon_pairs(*r["m2l"])) == c.meta["m2l_sha"] and sha(canon_pairs(*r["p2p"])) == c.meta["p2p_sha"]
    s = c.meta["stats_dualtree"]
    assert r["p2p_pairs"] == s["p2p_pairs"] and r["p2p_skipped"] == s["p2p_skipped"]
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(r[k], c["dualtree_" + k]) <= 1e-12, k


def test_cross_treecode_lists_and_result(trees):
    c, A, B = trees
    r = orc.evaluate_treecode_cross(A, B, c.p, c.theta)
    assert sha(canon_pairs(*r["m2p"])) == c.meta["m2p_sha"] and sha(canon_pairs(*r["p2p"])) == c.meta["tc_p2p_sha"]
    s = c.meta["stats_treecode"]
    assert r["p2p_pairs"] == s["p2p_pairs"] and r["p2p_skipped"] == s["p2p_skipped"]
    assert len(r["m2p"][0]) == s["m2p_calls"]
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(r[k], c["treecode_" + k]) <= 1e-12, k
