"""Subdomain operators (reference substructuring.py).

``build_subdomain_operator(system, partition, globs, i)`` keeps the
reference signature; the first call for a (system, partition, globs) triple
factorises *all* subdomains in one batched device pass (csrc/local.cu) and
later calls return views into it.  Views expose the reference attributes in
the reference's nodal B order (sorted by global node id); device buffers are
in glob-major order (plan.py).
"""

import weakref

import numpy as np

from .engine import LocalSystem, NumericalError

_CACHE = {}


def local_system(system, partition, globs, **kw):
    key = (id(system), id(partition), id(globs))
    hit = _CACHE.get(key)
    if hit is not None:
        refs, ls = hit
        if all(r() is o for r, o in zip(refs, (system, partition, globs))):
            return ls
    ls = LocalSystem(system, partition, globs, **kw)
    _CACHE.clear()  # one resident problem at a time keeps device memory bounded
    _CACHE[key] = ((weakref.ref(system), weakref.ref(partition), weakref.ref(globs)), ls)
    return ls


class SubdomainOperator:
    """View of subdomain ``sub_id`` (reference substructuring.py:23-75)."""

    def __init__(self, ls, sub_id):
        self.ls = ls
        self.sub_id = sub_id
        p = ls.plan
        self._perm = p.nodal_order(sub_id)  # glob-major -> nodal
        gm_nodes = p.B_nodes[p.voff[sub_id]:p.voff[sub_id + 1]]
        self.interface_nodes = gm_nodes[self._perm]
        self.interior_nodes = ls.interior_nodes_host[p.ioff[sub_id]:p.ioff[sub_id + 1]]
        self.iface_index = ls.globs.interface_index(self.interface_nodes)
        self._pos = {int(n): k for k, n in enumerate(self.interface_nodes)}

    @property
    def n_B(self):
        return self.interface_nodes.shape[0]

    def _nodal(self, buf):
        M = self.ls.matrix(buf, self.sub_id)
        return M[np.ix_(self._perm, self._perm)]

    @property
    def S(self):
        return self._nodal(self.ls.S)

    @property
    def Bsym(self):
        S = self.S
        return 0.5 * (S + S.T)

    @property
    def Zskew(self):
        S = self.S
        return 0.5 * (S - S.T)

    @property
    def g(self):
        return self.ls.vector(self.ls.g, self.sub_id)[self._perm]

    def glob_index(self, glob):
        try:
            return np.array([self._pos[int(n)] for n in glob.nodes], dtype=int)
        except KeyError:
            raise ValueError(f"glob with sharers {glob.sharers} is not on subdomain "
                             f"{self.sub_id}") from None

    def bsym_inverse(self):
        return self._nodal(self.ls.bsym_inverse())


def build_subdomain_operator(system, partition, globs, i):
    """Reference signature (substructuring.py:78); batched underneath."""
    ls = local_system(system, partition, globs)
    if not 0 <= i < ls.N:
        raise ValueError(f"subdomain {i} has no elements")
    return SubdomainOperator(ls, i)


def build_subdomain_operators(system, partition, globs):
    """All subdomain operators at once (one batched device pass)."""
    ls = local_system(system, partition, globs)
    return [SubdomainOperator(ls, i) for i in range(ls.N)]


def glob_principal_block(op, glob):
    """Bsym[X, X] (reference substructuring.py:146-149), from the device copy."""
    idx = op.glob_index(glob)
    return op.Bsym[np.ix_(idx, idx)]


def glob_schur_block(op, glob):
    """((Bsym^-1)[X,X])^-1, symmetrised (reference substructuring.py:152-171),
    by the device Gauss-Jordan with the Cholesky criterion (positive pivots)."""
    import torch

    from ._lib import lib, stream
    from .engine import dev_i32, dev_i64

    idx = op.glob_index(glob)
    n = idx.size
    block = op.bsym_inverse()[np.ix_(idx, idx)]
    M = torch.from_numpy(np.ascontiguousarray(block)).cuda().reshape(-1)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    pinv = torch.empty(4096, dtype=torch.float64, device="cuda")
    one = dev_i32(np.array([n]))
    lib.bddc_gj_inverse(M, dev_i64(np.array([0])), one, one, 1, n, pinv, 4096, status, 1, 0, stream())
    if int(status.item()):
        raise NumericalError(f"glob Schur block on subdomain {op.sub_id} is singular "
                             f"(cond ~ {np.linalg.cond(block):.2e})")
    out = M.view(n, n)
    return (0.5 * (out + out.T)).cpu().numpy()


__all__ = ["NumericalError", "SubdomainOperator", "build_subdomain_operator",
           "build_subdomain_operators", "glob_principal_block", "glob_schur_block", "local_system"]
