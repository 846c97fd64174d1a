"""BASELINE configurations at full size against the REAL reference
(tests/golden/make_golden_full.py): C2 (2^20), C3 (Plummer 2^22), C5 (2^24,
ncrit 128), the C4 high-order corner at 2^20 and the whole C4 grid at 2^16.

Bit-exact (SHA-256 of the reference's arrays): sorted Morton keys, the
permutation, all 13 cell arrays, the single-root M2L and P2P pair sets and
the reference's KernelStats counters.  FP64 results on the 1000-body error
sample (src/tuner.py:30-39) within 1e-10 relative L2 of the reference FMM's
own output (the north-star bar is 1e-5).  FP32 mode: force and potential
error against direct summation within 2x the reference's error.
"""

import json
import os

import numpy as np
import pytest
import torch

import paper_1209_3516_b200 as fb
from goldens import FP32_BAR_FLOOR, GOLDEN, rel_l2, sha
from paper_1209_3516_b200 import workloads as wl

pytestmark = pytest.mark.gpu

FULL = os.path.join(GOLDEN, "full")
FP64_TOL = 1e-10
CELL_DT = dict(children=np.int32, parent=np.int32, level=np.int8, key=np.uint64, start=np.int32, end=np.int32,
               sub_end=np.int32, leaf=np.uint8)
BIG = ["c2_full", "c3_full", "c5_full"]
CORNER = [f"c4_full_p{p}_t{t}" for p in (8, 10) for t in (0.3, 0.4)]
GRID = [f"c4_64k_p{p}_t{t}" for p in (3, 4, 6, 8, 10) for t in (0.3, 0.4, 0.5, 0.6)]


def _gen(name):
    if name == "c2_full":
        return wl.config2(1 << 20, 0)
    if name == "c3_full":
        return wl.plummer(1 << 22, 0)
    if name == "c5_full":
        return wl.config5(1 << 24, 0)
    if name.startswith("c4_full"):
        return wl.config4(1 << 20, 0)
    return wl.config4(1 << 16, 0)


def load(name):
    with open(os.path.join(FULL, name + ".json")) as fh:
        meta = json.load(fh)
    return meta, np.load(os.path.join(FULL, name + ".npz"))


def test_every_full_size_golden_present():
    for name in BIG + CORNER + GRID:
        assert os.path.exists(os.path.join(FULL, name + ".json")), name


_trees = {}


def tree_for(name, meta):
    key = (name.split("_p")[0] if name.startswith("c4") else name, meta["ncrit"])
    if key not in _trees:
        _trees.clear()
        pos, q = _gen(name)
        d = torch.as_tensor(pos, device="cuda")
        ps = fb.ParticleSet(d[:, 0].contiguous(), d[:, 1].contiguous(), d[:, 2].contiguous(),
                            torch.as_tensor(q, device="cuda"))
        _trees[key] = (fb.build_tree(ps, ncrit=meta["ncrit"]), pos, q)
    return _trees[key]


def device_canon_sha(lists, which):
    """SHA of the canonical pair encoding (sorted int64 t << 32 | s), built
    and sorted on the device."""
    rows = getattr(lists, which + "_rows")
    src = getattr(lists, which + "_src")
    cnt = rows[1:] - rows[:-1]
    t = torch.repeat_interleave(torch.arange(cnt.numel(), device=rows.device, dtype=torch.int64), cnt)
    code = (t << 32) | src[:t.numel()].long()
    return sha(torch.sort(code).values.cpu().numpy())


def sample_errors(tree, arrs):
    idx = arrs["idx"]
    b = tree.bodies
    fref = np.stack([arrs["direct_fx"], arrs["direct_fy"], arrs["direct_fz"]], 1)
    fgot = np.stack([b.fx[idx], b.fy[idx], b.fz[idx]], 1)
    ferr = float(np.sqrt(((fgot - fref) ** 2).sum() / (fref ** 2).sum()))
    return ferr, rel_l2(b.phi[idx], arrs["direct_phi"])


@pytest.mark.parametrize("name", BIG)
def test_full_size_tree_lists_and_counters(name):
    meta, _ = load(name)
    t, pos, q = tree_for(name, meta)
    p64 = np.asarray(pos, np.float64)
    got_in = sha(np.concatenate([p64[:, 0], p64[:, 1], p64[:, 2], np.asarray(q, np.float64)]))
    assert got_in == meta["input_sha"]
    assert (t.ncells, t.nleaves, t.depth) == (meta["ncells"], meta["nleaves"], meta["depth"])
    assert sha(t.keys.astype(np.uint64)) == meta["keys_sha"]
    assert sha(t.permutation.astype(np.int64)) == meta["perm_sha"]
    for f, want in meta["cells_sha"].items():
        got = np.ascontiguousarray(getattr(t, "cell_" + f)).astype(CELL_DT.get(f, np.float64))
        assert sha(got) == want, f
    lists = fb.interaction_lists(t, fb.MacConfig("fmm", meta["theta"]), defer=False)
    assert (lists.n_m2l, lists.n_p2p) == (meta["n_m2l"], meta["n_p2p"])
    assert device_canon_sha(lists, "m2l") == meta["m2l_sha"]
    lists.p2p_src  # noqa: B018  (sorted rows, built on demand)
    assert device_canon_sha(lists, "p2p") == meta["p2p_sha"]
    pairs, skipped = lists.dev_stats.tolist()
    assert (pairs, skipped) == (meta["stats"]["p2p_pairs"], meta["stats"]["p2p_skipped"])


@pytest.mark.parametrize("name", BIG + CORNER)
def test_full_size_fp64_matches_reference_fmm(name):
    meta, arrs = load(name)
    t, _, _ = tree_for(name, meta)
    t._M = None  # the reference ran upward on a fresh tree (p2m/m2m counted)
    rep = fb.evaluate_on_tree(t, fb.EvalConfig(mac=fb.MacConfig("fmm", meta["theta"]), p=meta["p"]))
    for k in ("p2p_pairs", "p2p_skipped", "p2p_flops", "m2l_calls", "p2m_calls", "m2m_calls", "l2l_calls",
              "l2p_calls"):
        assert getattr(rep.stats, k) == meta["stats"][k], k
    idx = arrs["idx"]
    b = t.bodies
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(b, k)[idx], arrs[k]) <= FP64_TOL, k
    ferr, perr = sample_errors(t, arrs)
    assert abs(ferr - meta["force_err"]) <= 1e-6 * meta["force_err"]
    assert abs(perr - meta["pot_err"]) <= 1e-6 * meta["pot_err"]


@pytest.mark.parametrize("name", BIG + CORNER)
def test_full_size_fp32_within_twice_reference_error(name):
    meta, arrs = load(name)
    t, _, _ = tree_for(name, meta)
    fb.evaluate_on_tree(t, fb.EvalConfig(mac=fb.MacConfig("fmm", meta["theta"]), p=meta["p"], precision="fp32"))
    ferr, perr = sample_errors(t, arrs)
    assert ferr <= 2.0 * meta["force_err"] + FP32_BAR_FLOOR, (ferr, meta["force_err"])
    assert perr <= 2.0 * meta["pot_err"] + FP32_BAR_FLOOR, (perr, meta["pot_err"])


@pytest.mark.parametrize("name", GRID)
def test_c4_grid_reduced_n(name):
    """The whole C4 accuracy grid at N=2^16: counters exact, FP64 within
    1e-10 of the reference FMM, FP32 within 2x the reference's error."""
    meta, arrs = load(name)
    t, _, _ = tree_for(name, meta)
    cfg = fb.EvalConfig(mac=fb.MacConfig("fmm", meta["theta"]), p=meta["p"])
    rep = fb.evaluate_on_tree(t, cfg)
    assert (rep.stats.p2p_pairs, rep.stats.m2l_calls) == (meta["stats"]["p2p_pairs"], meta["stats"]["m2l_calls"])
    idx = arrs["idx"]
    for k in ("phi", "fx", "fy", "fz"):
        assert rel_l2(getattr(t.bodies, k)[idx], arrs[k]) <= FP64_TOL, k
    cfg.precision = "fp32"
    fb.evaluate_on_tree(t, cfg)
    ferr, perr = sample_errors(t, arrs)
    assert ferr <= 2.0 * meta["force_err"] + FP32_BAR_FLOOR, (ferr, meta["force_err"])
    assert perr <= 2.0 * meta["pot_err"] + FP32_BAR_FLOOR, (perr, meta["pot_err"])

