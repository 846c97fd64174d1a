"""Pin the oracle's treecode restatement (oracle/fmm_oracle.c:
orc_collect_treecode, orc_exec_m2p) to the reference's treecode goldens
(tests/golden/make_golden_treecode.py): bit-exact M2P/P2P pair sets and
counters, and -- same DFS order, no FMA contraction -- bitwise M2P sums and
final evaluate_treecode output."""

import numpy as np
import pytest

from goldens import TC_CASES, TcCase, canon_pairs, rel_l2, sha
from oracle import oracle as orc


@pytest.fixture(scope="module", params=TC_CASES)
def case_and_tree(request):
    c = TcCase(request.param)
    return c, orc.build_tree(c.pos, c.q, c.ncrit, False)


def test_treecode_lists_bit_exact(case_and_tree):
    c, t = case_and_tree
    mt, ms, pt, ps = orc.collect_treecode(t, c.theta)
    m2p, p2p = canon_pairs(mt, ms), canon_pairs(pt, ps)
    assert m2p.size == c.meta["n_m2p"] and p2p.size == c.meta["n_p2p"]
    assert sha(m2p) == c.meta["m2p_sha"] and sha(p2p) == c.meta["p2p_sha"]
    assert mt.size == c.meta["stats"]["m2p_calls"]


def test_treecode_m2p_and_result(case_and_tree):
    c, t = case_and_tree
    r = orc.evaluate_treecode(t, c.p, c.theta)
    assert r["p2p_pairs"] == c.meta["stats"]["p2p_pairs"]
    assert r["p2p_skipped"] == c.meta["stats"]["p2p_skipped"]
    if c.full:
        mt, ms = r["m2p"]
        acc = orc.exec_m2p(t, mt, ms, r["M"], c.p)
        # same DFS list order and operation order as the reference: bitwise
        for k, a in zip(("phi", "fx", "fy", "fz"), acc):
            assert np.array_equal(a, c["m2p_" + k]), k
        for k in ("phi", "fx", "fy", "fz"):
            assert np.array_equal(r[k], c[k]), k
    else:
        idx = c["direct_idx"]
        for k in ("phi", "fx", "fy", "fz"):
            assert rel_l2(r[k][idx], c["sample_" + k]) <= 1e-12, k
