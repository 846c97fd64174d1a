"""Pin the oracle's listfmm restatement (oracle/fmm_oracle.c:
orc_collect_vlist, orc_collect_ulist) to the reference's listfmm goldens
(tests/golden/make_golden_listfmm.py): bit-exact V/U pair sets and counters,
and the final evaluate_list_fmm output."""

import numpy as np
import pytest

from goldens import LF_CASES, LfCase, canon_pairs, rel_l2, sha
from oracle import oracle as orc


@pytest.fixture(scope="module", params=LF_CASES)
def case_and_tree(request):
    c = LfCase(request.param)
    return c, orc.build_tree(c.pos, c.q, c.ncrit, False)


def test_listfmm_lists_bit_exact(case_and_tree):
    c, t = case_and_tree
    mt, ms, pt, ps = orc.collect_listfmm(t)
    m2l, p2p = canon_pairs(mt, ms), canon_pairs(pt, ps)
    assert m2l.size == c.meta["n_m2l"] and p2p.size == c.meta["n_p2p"]
    assert sha(m2l) == c.meta["m2l_sha"] and sha(p2p) == c.meta["p2p_sha"]
    assert mt.size == c.meta["stats"]["m2l_calls"]


def test_listfmm_result(case_and_tree):
    c, t = case_and_tree
    r = orc.evaluate_listfmm(t, c.p)
    assert r["p2p_pairs"] == c.meta["stats"]["p2p_pairs"]
    assert r["p2p_skipped"] == c.meta["stats"]["p2p_skipped"]
    idx = c["direct_idx"]
    for k in ("phi", "fx", "fy", "fz"):
        want = c[k] if c.full else c["sample_" + k]
        got = r[k] if c.full else r[k][idx]
        assert rel_l2(got, want) <= 1e-12, k
