"""CPU-only checks: the C ABI library loads and exports what include/*.h
declares (no compute calls), and the host-side API mirrors the reference's
validation and error behaviour."""

import ctypes
import glob
import os
import re

import numpy as np
import pytest

import paper_1209_3516_b200 as fb
from paper_1209_3516_b200 import _lib, workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_decls():
    decls = {}
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"FMM_API\s+[\w\s\*]+?\b(fmm_\w+)\s*\(([^;]*?)\)\s*;", txt, flags=re.S):
            args = m.group(2).strip()
            nargs = 0 if args in ("", "void") else len(args.split(","))
            decls[m.group(1)] = nargs
    return decls


def test_library_exports_every_declared_symbol():
    decls = header_decls()
    assert len(decls) >= 20
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name, nargs in decls.items():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
        assert len(_lib.SIGNATURES[name]) == nargs, (name, nargs, len(_lib.SIGNATURES[name]))
    assert set(_lib.SIGNATURES) == set(decls)


def test_library_loads_without_gpu():
    lib = _lib.load()
    assert lib.fmm_abi_version() == 1
    assert lib.fmm_last_error() == b""


def test_workspace_query_is_host_only():
    n = ctypes.c_size_t(0)
    _lib.call("fmm_workspace_bytes", 1 << 20, ctypes.byref(n))
    assert n.value > (1 << 20) * 16


def test_sm100a_cubin_in_library():
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_build_validation_matches_reference():
    pos, q = workloads.uniform_unit(10, 0)
    ps = fb.ParticleSet(pos[:, 0], pos[:, 1], pos[:, 2], q)
    with pytest.raises(ValueError):
        fb.build_tree(ps, ncrit=0)
    with pytest.raises(ValueError, match="shape"):
        fb.build_tree(ps, shape="spherical")
    with pytest.raises(ValueError, match="center"):
        fb.build_tree(ps, center_mode="origin")
    with pytest.raises(ValueError):
        fb.build_tree(fb.ParticleSet(np.empty(0), np.empty(0), np.empty(0), np.empty(0)))


def test_config_validation():
    with pytest.raises(ValueError, match="MAC kind"):
        fb.MacConfig("nope", 0.5)
    with pytest.raises(ValueError, match="theta"):
        fb.MacConfig("fmm", 0.0)
    with pytest.raises(ValueError, match="theta"):
        fb.MacConfig("fmm", 2.5)
    with pytest.raises(ValueError, match="expansion order"):
        fb.EvalConfig(p=13)
    with pytest.raises(ValueError, match="strategy"):
        fb.EvalConfig(strategy="fast")
    with pytest.raises(ValueError, match="precision"):
        fb.EvalConfig(precision="fp16")
    with pytest.raises(TypeError):
        fb.EvalConfig(mac=0.5)
    assert fb.EvalConfig().precision == "fp64"


def test_particle_set_contract():
    ps = fb.ParticleSet([0, 1], [0, 0], [0, 0], [1, 1])
    assert ps.x.dtype == np.float64 and ps.phi.shape == (2,)
    with pytest.raises(ValueError, match="disagree"):
        fb.ParticleSet([0, 1], [0], [0, 0], [1, 1])
    v = ps.view(0, 1)
    v.phi[:] = 3.0
    assert ps.phi[0] == 3.0


def test_mac_accept_matches_reference_formula():
    class Cell:
        def __init__(self, c, b, r):
            self.center, self.bmax, self.rmax = np.array(c, float), b, r
    a, b = Cell([0, 0, 0], 0.1, 0.2), Cell([1, 0, 0], 0.1, 0.2)
    assert fb.accept(fb.MacConfig("fmm", 0.3), a, b)        # 0.2 < 0.3
    assert not fb.accept(fb.MacConfig("fmm", 0.2), a, b)    # strict <
    assert not fb.accept(fb.MacConfig("fmm", 2.0), a, a)    # r == 0 rejects
    assert fb.accept(fb.MacConfig("bh", 0.5), a, b) and not fb.accept(fb.MacConfig("bh", 0.4), a, b)


def test_ncoef():
    assert [fb.ncoef(p) for p in (1, 4, 5, 10, 12)] == [1, 20, 35, 220, 364]


def test_report_schema():
    st = fb.KernelStats(p2p_pairs=10, p2p_flops=200)
    st.add_time("p2p", 0.5)
    rep = fb.EvalReport("dualtree", 4, 4, 4, "fmm", 0.4, False, 1, 5000, st, 0.1, 0.2, 0.3, 0.4)
    d = rep.to_dict()
    assert d["schema"] == "fmmkit-report-v1"
    assert d["times_ms"]["total"] == 1000 and d["kernel_times_ms"]["p2p"] == 500
    assert d["counts"]["p2p_flops"] == 200


def test_workload_generators_are_seeded():
    a, qa = workloads.plummer(4096, 0)
    b, qb = workloads.plummer(4096, 0)
    assert np.array_equal(a, b) and a.dtype == np.float32
    r = np.linalg.norm(a.astype(np.float64), axis=1)
    assert r.max() <= 10.0 + 1e-4 and np.all(qa == np.float32(1.0 / 4096))
    p2, q2 = workloads.config2(1000, 0)
    assert p2.dtype == np.float32 and q2.min() >= 0.0 and q2.max() < 1.0
    p1, q1 = workloads.config1(1000, 0)
    assert abs(q1.mean()) < 1e-15


def test_reference_argument_errors():
    with pytest.raises(ValueError, match="share one tree"):  # the reference's error
        fb.evaluate_dual_tree(object(), fb.EvalConfig(mutual=True), source_tree=object())
    with pytest.raises(ValueError, match="one tree onto itself"):  # the reference's error
        fb.evaluate_list_fmm(object(), fb.EvalConfig(strategy="listfmm"), source_tree=object())


def _static_len(node, env):
    """Length of a starred argument when it is statically knowable."""
    import ast
    if isinstance(node, (ast.Tuple, ast.List)):
        return len(node.elts)
    if isinstance(node, ast.GeneratorExp) and len(node.generators) == 1:
        it = node.generators[0].iter
        if isinstance(it, (ast.Tuple, ast.List)):
            return len(it.elts)
        if isinstance(it, ast.Name) and it.id in env:
            return env[it.id]
    return None


def test_call_sites_match_abi_arity():
    """Every _lib.call("fmm_*", ...) in the package passes exactly the
    arguments the C ABI declares (catches host/ABI drift without a GPU)."""
    import ast
    pkg = os.path.join(ROOT, "paper_1209_3516_b200")
    checked = 0
    for fn in glob.glob(os.path.join(pkg, "*.py")) + [os.path.join(ROOT, "bench.py")]:
        tree = ast.parse(open(fn).read())
        seen = {}
        for node in ast.walk(tree):
            if isinstance(node, ast.Assign) and len(node.targets) == 1 and isinstance(node.targets[0], ast.Name):
                k = None
                if isinstance(node.value, (ast.Tuple, ast.List)):
                    k = len(node.value.elts)
                elif isinstance(node.value, ast.ListComp) and isinstance(node.value.generators[0].iter, ast.Call):
                    c = node.value.generators[0].iter
                    if getattr(c.func, "id", "") == "range" and c.args and isinstance(c.args[0], ast.Constant):
                        k = c.args[0].value
                seen.setdefault(node.targets[0].id, set()).add(k)
        # names bound more than one way are ambiguous: those call sites are skipped
        env = {n: next(iter(v)) for n, v in seen.items() if len(v) == 1 and None not in v}
        for node in ast.walk(tree):
            if not (isinstance(node, ast.Call) and node.args and isinstance(node.args[0], ast.Constant)
                    and isinstance(node.args[0].value, str) and node.args[0].value.startswith("fmm_")):
                continue
            name = node.args[0].value
            n = 0
            for a in node.args[1:]:
                if isinstance(a, ast.Starred):
                    k = _static_len(a.value, env)
                    if k is None:
                        n = None
                        break
                    n += k
                else:
                    n += 1
            if n is None:
                continue
            assert n == len(_lib.SIGNATURES[name]), (fn, node.lineno, name, n, len(_lib.SIGNATURES[name]))
            checked += 1
    assert checked >= 15


def test_integration_binding_matches_header():
    """INTEGRATION.md's reference-side ctypes stub declares argtypes with the
    arity the header declares (the doc cannot drift from the ABI)."""
    decls = header_decls()
    txt = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    found = re.findall(r"_lib\.(fmm_\w+)\.argtypes\s*=\s*\[([^\]]*)\]", txt)
    assert found
    for name, args in found:
        n = len([a for a in args.split(",") if a.strip()])
        assert decls[name] == n, (name, decls[name], n)


def test_fp32_promotion_rule(monkeypatch):
    """precision="fp32" keeps FP32 near fields except where the expansion is
    more accurate than float32 sums (theta^p < 5e-4): there float32 terms
    summed in float64 ("fp32acc") down to theta^p = 5e-5, float64 below.
    On the C4 grid: (8, 0.3) and (10, 0.4) fp32acc, (10, 0.3) fp64."""
    import paper_1209_3516_b200 as fb
    from paper_1209_3516_b200.traversal import near_field_precision
    monkeypatch.delenv("FMM_B200_NEAR_FIELD", raising=False)
    nf = {(p, t): near_field_precision(fb.EvalConfig(mac=fb.MacConfig("fmm", t), p=p, precision="fp32"))
          for p in (3, 4, 6, 8, 10) for t in (0.3, 0.4, 0.5, 0.6)}
    assert sorted(k for k, v in nf.items() if v == "fp32acc") == [(8, 0.3), (10, 0.4)]
    assert sorted(k for k, v in nf.items() if v == "fp64") == [(10, 0.3)]
    assert near_field_precision(fb.EvalConfig(mac=fb.MacConfig("fmm", 0.3), p=10, precision="fp64")) == "fp64"
    assert near_field_precision(fb.EvalConfig(mac=fb.MacConfig("fmm", 0.4), p=4, precision="fp32acc")) == "fp32acc"
    monkeypatch.setenv("FMM_B200_NEAR_FIELD", "fp32acc")
    assert near_field_precision(fb.EvalConfig(mac=fb.MacConfig("fmm", 0.5), p=4, precision="fp64")) == "fp32acc"
    monkeypatch.setenv("FMM_B200_NEAR_FIELD", "bf16")
    with pytest.raises(ValueError):
        near_field_precision(fb.EvalConfig(p=4))


def test_deferred_report_fills_times_once_on_first_use():
    """DeferredReport: counters are readable without resolving; the first
    touch of a timed field (or total_time / to_dict) runs the thunk once."""
    from paper_1209_3516_b200 import traversal as tv
    rep = tv.DeferredReport(strategy="dualtree", n=8, n_sources=8, p=4, mac_kind="fmm", theta=0.4, mutual=False,
                            threads=1, task_grain=5000, stats=tv.KernelStats(), build_time=0.0, upward_time=0.0,
                            traversal_time=0.0, downward_time=0.0)
    calls = []

    def thunk(r):
        calls.append(1)
        r.__dict__["stats"].add_time("p2p", 0.25)
        r.__dict__.update(build_time=1.0, upward_time=2.0, traversal_time=3.0, downward_time=4.0,
                          spans={"wall": 9.0})

    rep.__dict__["_thunk"] = thunk
    assert rep.n == 8 and rep.strategy == "dualtree" and not calls
    assert rep.total_time == 10.0 and calls == [1]
    assert rep.stats.times["p2p"] == 0.25 and rep.spans == {"wall": 9.0}
    rep.resolve_times()
    assert calls == [1] and rep.to_dict()["times_ms"]["total"] == 10000
