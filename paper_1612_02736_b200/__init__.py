"""B200-native HPS (hierarchical Poincare-Steklov) multidomain spectral direct solver.

Drop-in for the build/solve hot path of the reference package ``specdtn``
(arXiv 1612.02736): same tree / plan / problem description in, same solution values on
the Chebyshev collocation nodes out. Host code mirrors the reference API; the numerics run
in hand-written sm_100a CUDA kernels behind the C ABI in include/hps_b200.h.
"""

from .geometry import (BoxNode, DomainTree, MeshConformityError, MergePlan, MeshSpec, NodePlan, Rect,
                       RefinementSpec, build_balanced_refined_tree, build_forest, build_mesh, build_uniform_tree,
                       count_chebyshev_dofs, enumerate_gauss_nodes, refine_near_point)
from .model import CoefficientField, ProblemSpec, catalog, manufactured_spec
from .solver import (FactorizedSolver, LeafSingularError, MergeSingularError, SolveState,
                     build_stage, downward_pass, solve, upward_pass)
from .reference import ReferenceSolution, linf_error
from .timestepping import ParabolicProblem, TimeStepConfig, be_run, cn_elliptic_spec, cn_run
from .archive import ArchiveError, load_operators, persist_operators

__version__ = "0.1.0"

__all__ = [
    "BoxNode", "DomainTree", "MeshConformityError", "MergePlan", "MeshSpec", "NodePlan", "Rect", "RefinementSpec",
    "build_balanced_refined_tree", "build_forest", "build_mesh", "build_uniform_tree", "count_chebyshev_dofs",
    "enumerate_gauss_nodes", "refine_near_point", "CoefficientField", "ProblemSpec", "catalog",
    "manufactured_spec", "FactorizedSolver", "LeafSingularError", "MergeSingularError",
    "SolveState", "build_stage", "downward_pass", "solve", "upward_pass", "ReferenceSolution", "linf_error",
    "ParabolicProblem", "TimeStepConfig", "be_run", "cn_elliptic_spec", "cn_run", "ArchiveError",
    "load_operators", "persist_operators",
]
