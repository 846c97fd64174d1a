"""Pin the oracle's rect / center-of-mass geometry (oracle/fmm_oracle.c:
orc_fill_geometry with rect/com, restating src/tree.py:80-160) to the
reference's fixtures (tests/golden/make_golden_geometry.py): every cell
array and the dual-tree pair sets bit-exact, final dual-tree phi/f."""

import numpy as np
import pytest

from goldens import GEO_CASES, GeoCase, canon_pairs, rel_l2, sha
from oracle import oracle as orc

FIELDS = ("children", "parent", "level", "key", "start", "end", "sub_end", "lo", "hi", "center", "bmax", "rmax",
          "leaf")
DT = dict(children=np.int32, parent=np.int32, level=np.int8, key=np.uint64, start=np.int32, end=np.int32,
          sub_end=np.int32, leaf=np.uint8)


@pytest.fixture(scope="module", params=GEO_CASES)
def case_and_tree(request):
    c = GeoCase(request.param)
    return c, orc.build_tree(c.pos, c.q, c.ncrit, False, c.shape, c.center_mode)


def test_geometry_bit_exact(case_and_tree):
    c, t = case_and_tree
    for f in FIELDS:
        got = np.ascontiguousarray(getattr(t, "cell_" + f)).astype(DT.get(f, np.float64))
        assert sha(got) == c.meta["cells_sha"][f], f


def test_lists_and_result(case_and_tree):
    c, t = case_and_tree
    r = orc.evaluate(t, c.p, c.theta)
    assert sha(canon_pairs(*r["m2l"])) == c.meta["m2l_sha"]
    assert sha(canon_pairs(*r["p2p"])) == c.meta["p2p_sha"]
    assert r["p2p_pairs"] == c.meta["stats_dualtree"]["p2p_pairs"]
    for k in ("phi", "fx", "fy", "fz"):
        want = c["dualtree_" + k]
        if np.any(want):
            assert rel_l2(r[k], want) <= 1e-12, k
        else:
            assert not np.any(r[k]), k
