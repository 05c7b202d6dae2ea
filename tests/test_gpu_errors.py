"""Error paths of the device hot path with the reference's NumericalError
messages (reference substructuring.py:64-75, :160-171; scaling.py:19-24;
adaptive.py:50-54; solver.py:91-98).  Each failure is provoked at the data
the failing factorisation reads, then the drop-in API must raise the
reference's error instead of returning garbage."""

import dataclasses
import math

import numpy as np
import pytest

from tests.cases import inputs

pytestmark = pytest.mark.gpu

THETA_F = 1.0 + math.log(4.0)


def _api():
    import paper_2501_01676_b200 as P

    return P


def _fresh_ops(system=None):
    P = _api()
    sys0, part, globs = inputs("jump")
    system = system if system is not None else dataclasses.replace(sys0)
    ops = [P.build_subdomain_operator(system, part, globs, i) for i in range(part.n_subdomains)]
    return system, part, globs, ops


def test_bsym_not_positive_definite():
    """Element blocks of subdomain 0 negated: its Schur complement, and Bsym,
    are negative definite -> the Cholesky-criterion check fails."""
    P = _api()
    sys0, part, globs = inputs("jump")
    K = sys0.elem_matrices.copy()
    F = sys0.elem_rhs.copy()
    mask = np.asarray(part.subdomain_of) == 0
    K[mask] *= -1.0
    F[mask] *= -1.0
    system = dataclasses.replace(sys0, elem_matrices=K, elem_rhs=F)
    _, _, _, ops = _fresh_ops(system)
    with pytest.raises(P.NumericalError, match="Bsym of subdomain 0 is not positive definite"):
        ops[0].bsym_inverse()


def test_singular_glob_schur_block():
    """A zeroed (Bsym^-1)[F, F] slot block: ((Bsym^-1)[F,F])^-1 does not exist."""
    P = _api()
    system, part, globs, ops = _fresh_ops()
    scaling = P.build_scaling(globs, ops)
    ls = ops[0].ls
    p = ls.plan
    BiC = ls.slot_binv()
    k = int(np.flatnonzero(p.kind == 0)[0])
    slot = int(p.sh_start[k])
    n = int(p.gsize[k])
    BiC[int(p.sh_doff[slot]):int(p.sh_doff[slot]) + n * n] = 0.0
    with pytest.raises(P.NumericalError, match=f"glob Schur block on subdomain {int(p.sh_sub[slot])} is singular"):
        P.adaptive_primal_space(globs, ops, scaling, THETA_F, 10.0, "old")


def test_singular_deluxe_sum():
    """Zeroed Bsym[g, g] blocks of every sharer of glob 0: sum_k B_k = 0."""
    P = _api()
    system, part, globs, ops = _fresh_ops()
    ls = ops[0].ls
    p = ls.plan
    BsC = ls.slot_bsym()
    n = int(p.gsize[0])
    for slot in range(int(p.sh_start[0]), int(p.sh_start[1])):
        BsC[int(p.sh_doff[slot]):int(p.sh_doff[slot]) + n * n] = 0.0
    with pytest.raises(P.NumericalError, match="deluxe block sum is singular"):
        P.build_scaling(globs, ops)


def test_pencil_failure_message():
    """A pencil right-hand side that is not PSD is reported as the reference's
    wrapped error (adaptive.py:50-54) by the status decoder of the glob phase,
    and as ValueError by the device pencil itself (linalg.py:151-152)."""
    import torch

    P = _api()
    from paper_2501_01676_b200 import linalg
    from paper_2501_01676_b200.engine import DevicePrimalSpace

    with pytest.raises(ValueError, match="not positive semidefinite"):
        linalg.sym_pencil_gevp(np.eye(3), np.diag([1.0, 2.0, -1.0]))
    system, part, globs, ops = _fresh_ops()
    scaling = P.build_scaling(globs, ops)
    basis, _ = P.adaptive_primal_space(globs, ops, scaling, THETA_F, 10.0, "old", detail=False)
    space = basis.device
    status = torch.zeros(space.ls.plan.G, dtype=torch.int32, device="cuda")
    status[3] = 203
    gid = globs.glob_id(globs.globs[3])
    with pytest.raises(P.NumericalError,
                       match=f"eigenproblem on glob {gid} failed: Btil is not positive semidefinite"):
        DevicePrimalSpace._raise(space, status, "face")


def test_dual_block_lost_positive_definiteness(monkeypatch):
    """S of subdomain 0 negated after Bsym^-1 (the certificate's premise
    Bsym = sym(S) broken), certificate forced off: the LDL^T check of
    sym(Sbar_dd) (the reference's cho_factor) must fail."""
    P = _api()
    from paper_2501_01676_b200.engine import DevicePreconditioner

    system, part, globs, ops = _fresh_ops()
    scaling = P.build_scaling(globs, ops)
    basis, _ = P.adaptive_primal_space(globs, ops, scaling, THETA_F, 10.0, "old", detail=False)
    ls = ops[0].ls
    n0 = int(ls.plan.nB[0])
    ls.S[:n0 * n0] *= -1.0
    monkeypatch.setattr(DevicePreconditioner, "_dual_pd_certified", staticmethod(lambda ls: False))
    with pytest.raises(P.NumericalError, match="dual block of subdomain 0 lost positive definiteness"):
        P.build_preconditioner(ops, basis, scaling)
