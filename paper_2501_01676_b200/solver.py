"""BDDC preconditioner, interface system and GMRES (reference solver.py),
on the device (csrc/precond.cu, csrc/krylov.cu)."""

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import lib, stream
from .coupled import CoupledMixin, averaging_and_jump
from .engine import (PANEL, DeviceInterfaceOperator, DevicePreconditioner, NumericalError, dev_f64,
                     dev_i32, dev_i64, gmres_device, gmres_right_device, recover_device)

F64 = torch.float64


@dataclass
class SolveReport:
    """solver.py:31-43"""

    iterations: int
    converged: bool
    solution: np.ndarray
    residual_history: list
    preconditioned_history: list
    setup_time: float = 0.0
    solve_time: float = 0.0
    gevp_time: float = 0.0
    pnumF: int = 0
    pnumE: int = 0
    extra: dict = field(default_factory=dict)


class BddcPreconditioner(CoupledMixin, DevicePreconditioner):
    """Reference class name (solver.py:46); ``apply`` takes numpy or device vectors.

    The reference's internals (dual_loc, primal_loc, gprimal, gdual_pos,
    primal_pos, Dbar, wt_size, transform, inject, inject_t, scale) are
    available through coupled.PartiallyCoupledSpace, built on first access."""

    def __init__(self, ops, primal, scaling):
        ls = ops[0].ls
        self.ops = sorted(ops, key=lambda o: o.sub_id)
        self.primal = primal
        self.scaling = scaling
        if primal.device is not None:
            Q, q_off = primal.device.Q, primal.device.d_q_off
        else:
            Q, q_off = _upload_transforms(ls, primal)
        super().__init__(ls, scaling.device, primal.r, Q, q_off,
                         householder=primal.device is not None)


def _upload_transforms(ls, primal):
    sizes = ls.plan.gsize.astype(np.int64)
    off = np.concatenate([[0], np.cumsum(sizes * sizes)])
    flat = np.zeros(max(int(off[-1]), 1))
    for k, (Q, _) in enumerate(primal.transforms):
        flat[off[k]:off[k + 1]] = np.asarray(Q, dtype=float).ravel()
    return dev_f64(flat), dev_i64(off[:-1])


def build_preconditioner(ops, primal, scaling):
    """solver.py:212-213"""
    return BddcPreconditioner(ops, primal, scaling)


class InterfaceOperator(DeviceInterfaceOperator):
    """Callable S_hat (solver.py:226-235) on numpy or device vectors."""


def interface_operator(ops, n):
    op = InterfaceOperator(ops[0].ls)
    if n != op.n:
        raise ValueError(f"interface size {n} does not match the operators ({op.n})")
    return op


def interface_rhs(ops, n):
    """g_hat = sum R_i^T g_i (solver.py:238-242)."""
    return InterfaceOperator(ops[0].ls).rhs_device().cpu().numpy()


def gmres_solve(operator, rhs, pc, rel_tol=1e-8, max_iter=300, side="left", restart=None):
    """Full left-preconditioned GMRES (solver.py:262-315) on the device.

    side="right" (with restart, default 200): right-preconditioned restarted
    GMRES, the variant BASELINE.json names (not in the reference);
    its histories are the true relative residuals."""
    if not isinstance(operator, DeviceInterfaceOperator) or not isinstance(pc, DevicePreconditioner):
        raise TypeError("gmres_solve runs on the device: pass interface_operator(...) and "
                        "build_preconditioner(...) objects from this package")
    t0 = time.perf_counter()
    rhs_d = rhs if isinstance(rhs, torch.Tensor) else dev_f64(rhs)
    lay = operator.layout
    b = lay.to_local(rhs_d.to(dtype=F64, device="cuda")).contiguous()
    if side == "left":
        it, conv, x, th, ph = gmres_device(operator, b, pc, rel_tol, max_iter)
    elif side == "right":
        it, conv, x, th, ph = gmres_right_device(operator, b, pc, rel_tol, max_iter,
                                                 200 if restart is None else restart)
    else:
        raise ValueError(f"unknown preconditioning side {side!r}")
    x = lay.to_global(x)
    return SolveReport(it, conv, x.cpu().numpy(), th, ph, solve_time=time.perf_counter() - t0)


def assemble_dense_schur(ops, n):
    """Dense S_hat = sum_i R_i^T S_i R_i (solver.py:245-249), assembled on the
    device in a fixed summation order (one warp per row)."""
    return _dense_schur_device(ops[0].ls, n).view(n, n).cpu().numpy()


def _dense_schur_device(ls, n, ld=None):
    p, d = ls.plan, ls.d
    if n != p.n_hat:
        raise ValueError(f"interface size {n} does not match the operators ({p.n_hat})")
    ld = n if ld is None else ld
    S = torch.empty(n * ld, dtype=F64, device="cuda")
    lib.bddc_coarse_scatter(dev_i32(p.voff), d.iface_perm, ls.S, d.soff, d.tstart, d.tsrc, S, ld,
                            n, p.N, stream())
    return S


def direct_schur_solve(ops, globs, rhs):
    """Dense assembled interface solve (solver.py:252-259), the oracle of the
    iterative path: [S_hat | rhs] eliminated on the device by the blocked
    no-pivot LU of the subdomain kernels (S_hat has a positive-definite
    symmetric part), then back-substituted."""
    ls = ops[0].ls
    n = globs.interface_nodes.shape[0]
    if (n + 2) * 8 > 220 * 1024:
        raise ValueError(f"direct_schur_solve: dense interface system of size {n} is beyond the "
                         "back-substitution kernel (n <= 28,000)")
    ld = (n + 2) // 2 * 2
    M = _dense_schur_device(ls, n, ld).view(n, ld)
    # the kernel wrote columns [0, n); column n carries the right-hand side
    M[:, n] = torch.as_tensor(np.asarray(rhs, dtype=np.float64)).cuda()
    if ld > n + 1:
        M[:, n + 1:] = 0.0
    M = M.reshape(-1)
    one = lambda v: dev_i32(np.array([v]))
    off, ldv, nv = dev_i64(np.array([0])), one(ld), one(n)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    pinv = torch.empty(4096, dtype=F64, device="cuda")
    st = stream()
    lib.bddc_schur_eliminate(M, off, ldv, nv, nv, one(n + 1), 1, n, n, n + 1, PANEL, pinv, 4096, 0,
                             status, 0, None, 0, None, None, st)
    if int(status.item()):
        raise NumericalError("assembled interface operator is singular")
    x = torch.empty(n, dtype=F64, device="cuda")
    lib.bddc_recover_interior(M, off, ldv, nv, one(0), dev_i64(np.array([0, 0])), one(0),
                              dev_i64(np.array([0, n])), torch.arange(n, device="cuda"), x, x, 1,
                              n, 64, None, st)
    return x.cpu().numpy()


def recover_interior(ops, globs, system, u_hat):
    """solver.py:318-326"""
    ls = ops[0].ls
    u_d = u_hat if isinstance(u_hat, torch.Tensor) else dev_f64(u_hat)
    u_l = ls.layout.to_local(u_d.to(dtype=F64, device="cuda")).contiguous()
    return recover_device(ls, u_l).cpu().numpy()


__all__ = ["BddcPreconditioner", "InterfaceOperator", "NumericalError", "SolveReport",
           "assemble_dense_schur", "averaging_and_jump", "build_preconditioner",
           "direct_schur_solve", "gmres_solve", "interface_operator", "interface_rhs",
           "recover_interior"]
