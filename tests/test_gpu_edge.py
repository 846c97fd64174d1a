"""Edge cases on the B200 path against the C oracle: tiny clouds (N = 1, 2,
3, 17), a root that is a single leaf, ncrit = 1, a degenerate (flat) cloud,
and float64 inputs that are not float32-exact (anchored FP32 mode)."""

import numpy as np
import pytest

import paper_1209_3516_b200 as fb
from goldens import canon_pairs, rel_l2
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _run(pos, q, ncrit, p=4, theta=0.5, precision="fp64", strategy="dualtree"):
    ps = fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q)
    t = fb.build_tree(ps, ncrit=ncrit)
    rep = fb.evaluate_on_tree(t, fb.EvalConfig(strategy=strategy, mac=fb.MacConfig("fmm", theta), p=p,
                                               precision=precision))
    return t, rep


@pytest.mark.parametrize("n,ncrit", [(1, 4), (2, 1), (3, 1), (17, 64), (17, 2), (300, 1)])
def test_tiny_clouds_match_oracle(n, ncrit):
    rng = np.random.default_rng(n * 7 + ncrit)
    pos = rng.random((n, 3))
    q = rng.uniform(-1, 1, n)
    t, rep = _run(pos, q, ncrit)
    ot = orc.build_tree(pos, q, ncrit)
    assert t.ncells == ot.ncells
    r = orc.evaluate(ot, 4, 0.5)
    lists = t.list_cache
    assert np.array_equal(canon_pairs(*lists.host_pairs("p2p")), canon_pairs(*r["p2p"]))
    assert np.array_equal(canon_pairs(*lists.host_pairs("m2l")), canon_pairs(*r["m2l"]))
    assert rep.stats.p2p_pairs == r["p2p_pairs"]
    b = t.bodies
    for k in ("phi", "fx", "fy", "fz"):
        want = r[k]
        if n == 1:
            assert np.all(getattr(b, k) == 0.0)  # a lone body feels nothing
        else:
            assert rel_l2(getattr(b, k), want) <= 1e-11, k


def test_flat_cloud_all_strategies():
    """All bodies in the plane z = 0.5 (a degenerate extent)."""
    rng = np.random.default_rng(3)
    pos = rng.random((2000, 3))
    pos[:, 2] = 0.5
    q = rng.uniform(-1, 1, 2000)
    ot = orc.build_tree(pos, q, 16)
    want = orc.evaluate(ot, 4, 0.5)
    t, _ = _run(pos, q, 16)
    for k in ("phi", "fx", "fy", "fz"):  # (fz != 0: truncation error, as in the reference)
        assert rel_l2(getattr(t.bodies, k), want[k]) <= 1e-11, k
    for strategy in ("treecode", "listfmm"):
        t2, rep = _run(pos, q, 16, strategy=strategy)
        assert rep.strategy == strategy and np.all(np.isfinite(t2.bodies.phi))


def test_anchored_fp32_for_float64_inputs():
    """Offsets far from the origin: float64 positions that float32 cannot
    hold; the FP32 path switches to anchored sources and keeps its accuracy."""
    rng = np.random.default_rng(11)
    pos = 1000.0 + rng.random((4000, 3)) * 1e-3
    q = rng.uniform(-1, 1, 4000)
    t64, _ = _run(pos, q, 32, precision="fp64")
    t32, _ = _run(pos, q, 32, precision="fp32")
    assert not t32.fp32_exact
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(t32.bodies, k), getattr(t64.bodies, k)) <= 1e-5, k


def test_pinned_host_inputs_build_the_same_tree():
    """Host arrays in page-locked memory are copied from where they are (no
    staging pass); the tree and the results equal the pageable build's, and
    the caller may overwrite the arrays once build_tree has returned."""
    import torch
    from paper_1209_3516_b200 import workloads
    pos, q = workloads.config2(20000, 3)
    cols = [np.ascontiguousarray(pos[:, k]) for k in range(3)] + [np.ascontiguousarray(q)]
    pinned = []
    for a in cols:
        h = torch.empty(a.shape, dtype=torch.from_numpy(a).dtype, pin_memory=True).numpy()
        h[...] = a
        pinned.append(h)
    assert all(torch.from_numpy(h).is_pinned() for h in pinned)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", 0.4), p=4, precision="fp32")
    t0 = fb.build_tree(fb.ParticleSet(*cols), ncrit=64)
    fb.evaluate_on_tree(t0, cfg)
    want = t0.results_in_input_order()
    t1 = fb.build_tree(fb.ParticleSet(*pinned), ncrit=64)
    t1._input_snapshot.result()  # (the tree's own copy of the inputs is taken on a worker thread)
    for h in pinned:
        h[...] = 0  # the device copy was complete when build_tree returned
    fb.evaluate_on_tree(t1, cfg)
    got = t1.results_in_input_order()
    assert np.array_equal(t0.permutation, t1.permutation) and np.array_equal(t0.cell_bmax, t1.cell_bmax)
    for k in ("phi", "fx", "fy", "fz"):
        assert np.array_equal(getattr(got, k), getattr(want, k)), k
    assert np.array_equal(np.asarray(got.x), np.asarray(want.x))  # the snapshot of the inputs, not the zeros
