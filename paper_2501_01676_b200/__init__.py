"""B200-native adaptive BDDC-preconditioned GMRES for 3D SUPG
advection-diffusion (the data-parallel hot path of arXiv 2501.01676).

Drop-in for the reference package's hot-path API (adbddc: substructuring,
scaling, adaptive, solver); the numerics run in hand-written sm_100a CUDA
kernels behind the C-ABI in include/bddc_b200.h.  Host preprocessing
(mesh, element blocks, partitions, globs) lives in mesh / discretization /
decomposition / configs.
"""

__version__ = "0.1.0"

from .engine import NumericalError  # noqa: F401


def __getattr__(name):
    # lazy API exports so that importing the package never touches CUDA
    import importlib

    table = {
        "PrimalBasis": "adaptive", "GevpReport": "adaptive", "adaptive_primal_space": "adaptive",
        "build_scaling": "scaling", "ScalingSet": "scaling",
        "build_subdomain_operator": "substructuring", "build_subdomain_operators": "substructuring",
        "SubdomainOperator": "substructuring",
        "SolveReport": "solver", "BddcPreconditioner": "solver", "build_preconditioner": "solver",
        "gmres_solve": "solver", "interface_operator": "solver", "interface_rhs": "solver",
        "recover_interior": "solver", "averaging_and_jump": "solver",
        "assemble_dense_schur": "solver", "direct_schur_solve": "solver",
        "EigenPairList": "linalg", "pseudo_inverse": "linalg", "parallel_sum": "linalg",
        "parallel_sum_chain": "linalg", "sym_pencil_gevp": "linalg",
        "build_change_of_basis": "adaptive", "reduce_edge_constraints": "adaptive",
        "assemble_primal_space": "adaptive",
    }
    if name in table:
        return getattr(importlib.import_module(f".{table[name]}", __name__), name)
    raise AttributeError(name)
