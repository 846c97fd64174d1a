"""paper_1209_3516_b200: B200-native (sm_100a) Laplace FMM hot path.

A drop-in for the dual-tree path of the reference package ``fmmkit``
(arXiv 1209.3516): ``ParticleSet`` -> ``build_tree`` ->
``evaluate_on_tree(EvalConfig(p, MacConfig("fmm", theta)))`` -> potentials
and forces, computed by hand-written CUDA kernels in ``libfmm_b200.so``
(see include/fmm_b200.h and DESIGN.md).  No CPU fallback.
"""

from .geometry import MAX_LEVEL, Aabb, ParticleSet, compute_bounds
from .kernels import P2P_FLOPS_PER_PAIR, TMAX, KernelStats, direct, ncoef
from .mac import MacConfig, accept, error_bound
from .traversal import (EvalConfig, EvalReport, evaluate_dual_tree, evaluate_list_fmm, evaluate_on_tree,
                        evaluate_treecode, interaction_lists, listfmm_lists, mutual_lists, treecode_lists)
from .tree import Tree, build_tree, check_invariants, downward_pass, upward_pass
from .tuner import (TuneEntry, TuneResult, error_sample, max_theta_for_error, sampled_force_error, select_p_theta,
                    verify_against_direct)

__version__ = "0.1.0"

__all__ = [
    "MAX_LEVEL", "TMAX", "P2P_FLOPS_PER_PAIR", "Aabb", "ParticleSet", "compute_bounds",
    "KernelStats", "direct", "ncoef", "MacConfig", "accept", "error_bound",
    "EvalConfig", "EvalReport", "evaluate_dual_tree", "evaluate_on_tree", "evaluate_treecode", "interaction_lists",
    "mutual_lists", "treecode_lists", "evaluate_list_fmm", "listfmm_lists",
    "Tree", "build_tree", "check_invariants", "downward_pass", "upward_pass",
    "error_sample", "sampled_force_error", "verify_against_direct", "max_theta_for_error", "select_p_theta",
    "TuneEntry", "TuneResult", "__version__",
]
