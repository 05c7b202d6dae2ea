"""Dense symmetric kernels of the reference's linalg.py on the device.

``pseudo_inverse``, ``parallel_sum``, ``parallel_sum_chain`` and
``sym_pencil_gevp`` keep the reference signatures (linalg.py:23-214) and
return host arrays / an ``EigenPairList``; the ``*_batched`` forms take a
stack of matrices (numpy or CUDA tensors, shape (b, n, n)) and run one CTA
per member (``bddc_linalg_batched``, csrc/globs.cu).  The per-glob kernels of
the adaptive primal space call the same device functions.

Argument checks (shapes, symmetry to the reference's relative tolerances)
raise ``ValueError`` with the reference's messages; a pencil whose
right-hand side is indefinite raises ``ValueError("Btil is not positive
semidefinite")`` like linalg.py:151-152.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import lib, require_cuda, stream
from .engine import NumericalError

F64 = torch.float64


@dataclass
class EigenPairList:
    """Eigenpairs of B v = lambda Btil v (reference linalg.py:81-113): values
    non-increasing with +inf first, degenerate (common-nullspace) directions
    flagged, eigenvalue 0, last, never selected."""

    values: np.ndarray
    vectors: np.ndarray
    degenerate: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.degenerate is None:
            self.degenerate = np.zeros(len(self.values), dtype=bool)

    @property
    def n_infinite(self):
        return int(np.count_nonzero(np.isinf(self.values)))

    def selection_mask(self, theta):
        return (self.values >= theta) & ~self.degenerate

    def n_selected(self, theta):
        return int(np.count_nonzero(self.selection_mask(theta)))

    def selected_vectors(self, theta):
        return self.vectors[:, self.selection_mask(theta)]


def _stack(M, name):
    """(b, n, n) float64 CUDA tensor from one matrix or a stack."""
    require_cuda()
    t = M if isinstance(M, torch.Tensor) else torch.from_numpy(np.asarray(M, dtype=np.float64))
    t = t.to(device="cuda", dtype=F64).contiguous()
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if t.dim() != 3 or t.shape[1] != t.shape[2]:
        raise ValueError(f"{name} must be square, got shape {tuple(M.shape)}")
    return t


def _check_symmetric(t, rel_tol, name):
    """reference _check_symmetric (linalg.py:15-20), per stack member, on the device."""
    if t.shape[1] == 0:
        return
    scale = torch.linalg.matrix_norm(t)
    asym = torch.linalg.matrix_norm(t - t.transpose(1, 2))
    bad = (scale > 0) & (asym > rel_tol * scale)
    if bool(bad.any()):
        raise ValueError(f"{name} is not symmetric to within {rel_tol:g} relative")


def _run(mode, A, B, rel_tol):
    b, n = A.shape[0], A.shape[1]
    out = torch.empty_like(A)
    nvec = torch.full((b,), n, dtype=torch.int32, device="cuda")
    off = torch.arange(b, dtype=torch.int64, device="cuda") * (n * n)
    wsz = int(lib.bddc_ws_linalg(n))
    ws = torch.empty(max(b * wsz, 1), dtype=F64, device="cuda")
    ws_off = torch.arange(b, dtype=torch.int64, device="cuda") * wsz
    vals = torch.empty((b, max(n, 1)), dtype=F64, device="cuda")
    voff = torch.arange(b, dtype=torch.int64, device="cuda") * max(n, 1)
    degen = torch.zeros((b, max(n, 1)), dtype=torch.int32, device="cuda")
    status = torch.zeros(b, dtype=torch.int32, device="cuda")
    lib.bddc_linalg_batched(mode, A, B if B is not None else A, off, nvec, b, float(rel_tol), out,
                            vals, voff, degen, status, ws, ws_off, n, stream())
    return out, vals[:, :n], degen[:, :n], status


def pseudo_inverse_batched(M, rel_tol=1e-12):
    """pinv of each symmetric member (eigen-based, cut rel_tol * max|w|); CUDA tensor."""
    A = _stack(M, "M")
    _check_symmetric(A, 1e-12, "M")
    if A.shape[1] == 0:
        return A.clone()
    return _run(0, A, None, rel_tol)[0]


def pseudo_inverse(M, rel_tol=1e-12):
    """reference linalg.py:23-50 (host array in, host array out)."""
    return pseudo_inverse_batched(M, rel_tol)[0].cpu().numpy()


def parallel_sum_batched(A, B, rel_tol=1e-12):
    """A_k : B_k = sym(A_k (A_k + B_k)^+ B_k) for each member; CUDA tensor."""
    a, b = _stack(A, "A"), _stack(B, "B")
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {tuple(np.shape(A))} vs {tuple(np.shape(B))}")
    _check_symmetric(a, 1e-12, "A")
    _check_symmetric(b, 1e-12, "B")
    if a.shape[1] == 0:
        return a.clone()
    return _run(1, a, b, rel_tol)[0]


def parallel_sum(A, B, rel_tol=1e-12):
    """reference linalg.py:53-67."""
    if np.shape(A) != np.shape(B):
        raise ValueError(f"shape mismatch: {np.shape(A)} vs {np.shape(B)}")
    return parallel_sum_batched(A, B, rel_tol)[0].cpu().numpy()


def parallel_sum_chain(mats, rel_tol=1e-12):
    """Left-associative chain (reference linalg.py:70-78), accumulated on the device."""
    mats = list(mats)
    if not mats:
        raise ValueError("empty chain")
    acc = _stack(mats[0], "A")
    for M in mats[1:]:
        acc = parallel_sum_batched(acc, M, rel_tol)
    return acc[0].cpu().numpy()


def sym_pencil_gevp_batched(B, Btil, rel_tol=1e-12):
    """Device pencils of a stack: (values (b, n), vectors (b, n, n), degenerate
    (b, n) bool) as CUDA tensors."""
    a, t = _stack(B, "B"), _stack(Btil, "Btil")
    if a.shape != t.shape:
        raise ValueError(f"shape mismatch: {tuple(np.shape(B))} vs {tuple(np.shape(Btil))}")
    _check_symmetric(a, 1e-10, "B")
    _check_symmetric(t, 1e-10, "Btil")
    n = a.shape[1]
    if n == 0:
        z = torch.zeros((a.shape[0], 0), dtype=F64, device="cuda")
        return z, torch.zeros((a.shape[0], 0, 0), dtype=F64, device="cuda"), z.bool()
    vecs, vals, degen, status = _run(2, a, t, rel_tol)
    if bool((status != 0).any()):
        raise ValueError("Btil is not positive semidefinite")
    return vals, vecs, degen.bool()


def sym_pencil_gevp(B, Btil, rel_tol=1e-12):
    """reference linalg.py:116-214: EigenPairList of B v = lambda Btil v."""
    vals, vecs, degen = sym_pencil_gevp_batched(B, Btil, rel_tol)
    return EigenPairList(vals[0].cpu().numpy(), vecs[0].cpu().numpy(), degen[0].cpu().numpy())


__all__ = ["EigenPairList", "NumericalError", "parallel_sum", "parallel_sum_batched",
           "parallel_sum_chain", "pseudo_inverse", "pseudo_inverse_batched", "sym_pencil_gevp",
           "sym_pencil_gevp_batched"]
