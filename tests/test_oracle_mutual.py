"""Pin the oracle's mutual dual traversal (partition roots, driver demotion,
mutual units, symmetric M2L/P2P) to the reference's mutual goldens
(tests/golden/make_golden_mutual.py)."""

import numpy as np
import pytest

from goldens import MU_CASES, MuCase, canon_pairs, rel_l2, sha
from oracle import oracle as orc


@pytest.fixture(scope="module", params=MU_CASES)
def case(request):
    c = MuCase(request.param)
    return c, orc.build_tree(c.pos, c.q, c.ncrit)


def test_partition_roots(case):
    c, t = case
    roots, owner = orc.partition_roots(t, c.grain)
    assert np.array_equal(roots, c["roots"])
    assert roots.size == c.meta["n_roots"]
    # every leaf is owned; an unowned cell is internal with >= grain bodies
    assert (owner[t.cell_leaf.astype(bool)] >= 0).all()
    up = owner < 0
    assert (t.cell_end[up] - t.cell_start[up] >= c.grain).all()


def test_mutual_lists_and_result(case):
    c, t = case
    r = orc.evaluate_mutual(t, c.p, c.theta, c.grain, c.mac)
    assert sha(canon_pairs(*r["m2l"])) == c.meta["m2l_sha"]
    assert sha(canon_pairs(*r["p2p"])) == c.meta["p2p_sha"]
    s = c.meta["stats"]
    assert r["p2p_pairs"] == s["p2p_pairs"] and r["p2p_skipped"] == s["p2p_skipped"]
    assert r["m2l_calls"] == s["m2l_calls"]
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(r[k], c[k]) <= 1e-12, k


def test_mutual_differs_from_directed(case):
    """The goldens pin lists the directed traversal does not produce."""
    c, _ = case
    assert c.meta["differs_from_directed"]
