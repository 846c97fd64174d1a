"""The (p, θ) tuner on the GPU path vs the reference's
own ``max_theta_for_error`` answers (tests/golden/make_golden_tuner.py).

The bisection takes the same branches as the reference when the GPU's FP64
errors agree with the reference's (they do to ~1e-11), so the tuned angles
must be EQUAL; the winner of ``select_p_theta`` depends on timings and is
only checked for consistency."""

import json
import os

import numpy as np
import pytest

import paper_1209_3516_b200 as fb
from goldens import GOLDEN, sha
from paper_1209_3516_b200 import workloads as wl

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "index_tuner.json")) as fh:
    TUNE = json.load(fh)


@pytest.fixture(scope="module")
def tree():
    pos, q = wl.uniform_unit(2000, 11)
    got = sha(np.concatenate([pos[:, 0], pos[:, 1], pos[:, 2], q]).astype(np.float64))
    assert got == TUNE["input_sha"]
    return fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q), ncrit=TUNE["ncrit"])


@pytest.mark.parametrize("k", range(len(TUNE["cases"])))
def test_max_theta_matches_reference(tree, k):
    c = TUNE["cases"][k]
    oracle = fb.error_sample(tree, 1000, 0)
    if c["theta"] is None:
        with pytest.raises(ValueError, match="unreachable"):
            fb.max_theta_for_error(tree, c["p"], c["target"], oracle=oracle)
        return
    theta = fb.max_theta_for_error(tree, c["p"], c["target"], oracle=oracle)
    assert theta == c["theta"]
    fb.evaluate_dual_tree(tree, fb.EvalConfig(mac=fb.MacConfig("fmm", theta), p=c["p"]))
    err = fb.sampled_force_error(tree, *oracle)
    # relative 1e-9, with an absolute floor for near-direct configurations
    # whose error is FP64 rounding (~1e-15, order-dependent)
    assert abs(err - c["tuned_error"]) <= 1e-9 * c["tuned_error"] + 1e-13


def test_select_p_theta_consistent(tree):
    res = fb.select_p_theta(tree, 1e-4, p_candidates=(3, 4, 5), reps=2)
    want = {c["p"]: c["theta"] for c in TUNE["cases"] if c["target"] == 1e-4}
    assert [e.p for e in res.entries] == [3, 4, 5]
    for e in res.entries:
        assert e.theta == want[e.p] and e.error <= 1e-4 and e.traversal_time > 0
    assert res.best in res.entries
    assert res.best.traversal_time == min(e.traversal_time for e in res.entries)
    with pytest.raises(ValueError, match="unreachable"):
        fb.select_p_theta(tree, 1e-20, p_candidates=(2,), reps=1)


@pytest.mark.parametrize("name,precision", [("c2_32k", "fp64"), ("plummer_32k", "fp32"), ("c1", "fp64")])
def test_sampled_evaluation_is_exact_at_the_sample(name, precision):
    """A sampled evaluation (target mask = the cells holding the sample
    bodies) gives the full evaluation's values at the sample bodies,
    bit for bit, with a small fraction of the P2P work."""
    from goldens import Case
    from paper_1209_3516_b200.tuner import ErrorProbe
    c = Case(name)
    pos = np.asarray(c.pos, np.float64)
    t = fb.build_tree(fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], c.q), ncrit=c.ncrit)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", c.theta), p=c.p, precision=precision)
    full = fb.evaluate_on_tree(t, cfg)
    probe = ErrorProbe(t, 200, 3)
    b = t.bodies
    want = np.stack([b.phi[probe.idx], b.fx[probe.idx], b.fy[probe.idx], b.fz[probe.idx]])
    ferr = probe.force_error()
    t._results_changed()
    for a in (t.d_phi, t.d_fx, t.d_fy, t.d_fz):
        a.fill_(float("nan"))
    part = probe.evaluate(cfg)
    t._results_changed()
    b = t.bodies
    got = np.stack([b.phi[probe.idx], b.fx[probe.idx], b.fy[probe.idx], b.fz[probe.idx]])
    assert np.array_equal(got, want)
    assert probe.force_error() == ferr
    assert 0 < part.stats.p2p_pairs < full.stats.p2p_pairs
    if t.nleaves > 1000:
        assert part.stats.p2p_pairs < 0.5 * full.stats.p2p_pairs
