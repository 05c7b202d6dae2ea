"""SUPG-stabilised P1 element blocks and Dirichlet data (host preprocessing,
input side of the hot path).

Restates the reference discretisation (reference:
pkg/src/adbddc/discretization.py:101-206): diffusion + least-squares
stabilisation (Peclet-switched weight, tau = 0.7) + shifted reaction
ctil = c - div(a)/2 + skew-symmetric advection, 4-point degree-2 quadrature.
The hot path consumes only ``elem_matrices``, ``elem_rhs``, ``node_to_free``
and ``dirichlet_values``; the assembled global CSR matrices are built lazily
on first access (they are used by direct-solve checks only).

Element blocks are computed in chunks so the 12.6M-element config-5 mesh
fits in host memory; the per-element arithmetic is evaluation-order identical
to the reference (np.einsum without BLAS paths), so blocks agree bitwise.
"""

import os
from dataclasses import dataclass, field
from typing import Callable, Optional, Union

import numpy as np

from .mesh import Mesh, element_diameters

_QA = 0.5854101966249685
_QB = 0.13819660112501053
QBARY = np.full((4, 4), _QB)
np.fill_diagonal(QBARY, _QA)


def peclet(h, anorm, nu):
    """Element Peclet number h |a| / (2 nu) (reference discretization.py:34-36)."""
    return h * anorm / (2.0 * np.asarray(nu))


def stabilization(h, anorm, nu, tau=0.7):
    """Peclet-switched least-squares weight (reference discretization.py:39-49)."""
    h = np.asarray(h, dtype=float)
    anorm = np.asarray(anorm, dtype=float)
    nu = np.asarray(nu, dtype=float)
    adv = peclet(h, anorm, nu) >= 1.0
    safe = np.where(adv, anorm, 1.0)
    return np.where(adv, tau * h / (2.0 * safe), tau * h * h / (4.0 * nu))


@dataclass
class DeviceFields:
    """Coefficient fields the device can evaluate (csrc/elements.cu): velocity
    a(x) = velocity_matrix @ x + velocity_offset, constant reaction and source,
    viscosity nu[e] = viscosity_table[e % viscosity_period].  Optional: a
    Coefficients carrying one lets the element blocks be built on the GPU
    inside every solve; the callables stay authoritative for the host."""

    velocity_matrix: np.ndarray
    velocity_offset: np.ndarray
    reaction: float
    source: float
    viscosity_table: np.ndarray
    viscosity_period: int

    def packed(self, tau, with_div):
        """The 16 doubles of bddc_supg_elements: A, a0, c, f, c - div(a)/2, tau."""
        A = np.asarray(self.velocity_matrix, dtype=float).reshape(3, 3)
        cdiv = self.reaction - 0.5 * float(np.trace(A)) if with_div else self.reaction
        return np.concatenate([A.ravel(), np.asarray(self.velocity_offset, dtype=float).ravel(),
                               [self.reaction, self.source, cdiv, tau]])


@dataclass
class Coefficients:
    """Problem data, same fields as the reference (discretization.py:52-67)."""

    viscosity: Union[np.ndarray, Callable]
    velocity: Callable
    reaction: Callable
    source: Callable
    dirichlet: Callable
    velocity_div: Optional[Callable] = None
    tau: float = 0.7
    device_fields: Optional[DeviceFields] = None


@dataclass
class AssembledSystem:
    """Element-level problem data plus the free/Dirichlet split
    (reference discretization.py:70-88)."""

    mesh: Mesh
    free_nodes: np.ndarray
    node_to_free: np.ndarray
    dirichlet_values: np.ndarray
    elem_matrices: np.ndarray = field(repr=False)
    elem_rhs: np.ndarray = field(repr=False)
    viscosity: np.ndarray = field(repr=False)
    device_fields: Optional[np.ndarray] = field(default=None, repr=False)  # packed fields
    device_viscosity: Optional[tuple] = field(default=None, repr=False)    # (table, period)
    _full: object = field(default=None, repr=False)
    _load: object = field(default=None, repr=False)

    @property
    def n_free(self):
        return self.free_nodes.shape[0]

    def _assemble(self):
        import scipy.sparse

        if self._full is None:
            el = self.mesh.elements
            n = self.mesh.n_nodes
            rows = np.repeat(el, 4, axis=1).ravel()
            cols = np.tile(el, (1, 4)).ravel()
            self._full = scipy.sparse.coo_matrix(
                (self.elem_matrices.ravel(), (rows, cols)), shape=(n, n)).tocsr()
            load = np.zeros(n)
            np.add.at(load, el.ravel(), self.elem_rhs.ravel())
            self._load = load
        return self._full, self._load

    @property
    def full_matrix(self):
        return self._assemble()[0]

    @property
    def matrix(self):
        full = self._assemble()[0]
        return full[self.free_nodes][:, self.free_nodes].tocsr()

    @property
    def rhs(self):
        full, load = self._assemble()
        dn = np.flatnonzero(self.node_to_free < 0)
        return load[self.free_nodes] - full[self.free_nodes][:, dn] @ self.dirichlet_values[dn]


def p1_gradients(verts):
    """Constant P1 basis gradients and volumes (reference discretization.py:91-98)."""
    E = verts[:, 1:] - verts[:, :1]
    Einv = np.linalg.inv(E)
    G = np.empty((verts.shape[0], 4, 3))
    G[:, 1:] = np.transpose(Einv, (0, 2, 1))
    G[:, 0] = -G[:, 1:].sum(axis=1)
    return G, np.linalg.det(E) / 6.0


def _chunk_blocks(verts, nu, coeffs):
    m = verts.shape[0]
    G, vol = p1_gradients(verts)
    if np.any(vol <= 0.0):
        raise ValueError("mesh contains degenerate or inverted elements")
    cent = verts.mean(axis=1)
    qpts = np.einsum("qi,mid->mqd", QBARY, verts).reshape(-1, 3)
    a_q = np.asarray(coeffs.velocity(qpts), dtype=float).reshape(m, 4, 3)
    c_q = np.asarray(coeffs.reaction(qpts), dtype=float).reshape(m, 4)
    f_q = np.asarray(coeffs.source(qpts), dtype=float).reshape(m, 4)
    if coeffs.velocity_div is None:
        ctil = c_q.copy()
    else:
        ctil = c_q - 0.5 * np.asarray(coeffs.velocity_div(qpts), dtype=float).reshape(m, 4)
    bad = np.any(ctil <= 0.0, axis=1)
    if bad.any():
        return None, None, int(np.flatnonzero(bad)[0])

    h = np.zeros(m)
    for a in range(4):
        for b in range(a + 1, 4):
            d = verts[:, a] - verts[:, b]
            h = np.maximum(h, np.sqrt((d * d).sum(-1)))
    samples = np.concatenate([verts, cent[:, None, :]], axis=1).reshape(-1, 3)
    a_s = np.asarray(coeffs.velocity(samples), dtype=float).reshape(m, 5, 3)
    anorm = np.sqrt((a_s * a_s).sum(-1)).max(axis=1)
    C = stabilization(h, anorm, nu, coeffs.tau)

    w = vol[:, None] / 4.0
    adv = np.einsum("mqd,mjd->mqj", a_q, G)
    t1 = np.einsum("mq,qi,mqj->mij", w, QBARY, adv)
    Lq = adv + c_q[:, :, None] * QBARY[None, :, :]
    K = np.einsum("mid,mjd->mij", G, G) * (nu * vol)[:, None, None]
    K = K + np.einsum("mq,qi,qj->mij", w * ctil, QBARY, QBARY)
    K = K + 0.5 * (t1 - np.transpose(t1, (0, 2, 1)))
    K = K + C[:, None, None] * np.einsum("mq,mqi,mqj->mij", w, Lq, Lq)
    wf = w * f_q
    F = np.einsum("mq,qi->mi", wf, QBARY)
    F += C[:, None] * np.einsum("mq,mqi->mi", wf, Lq)
    return K, F, -1


def element_contributions(mesh, coeffs, chunk=1 << 18):
    """Per-element 4x4 blocks and 4-vectors (reference discretization.py:101-158)."""
    el = mesh.elements
    m = el.shape[0]
    nu = coeffs.viscosity
    if callable(nu):
        cent = np.empty((m, 3))
        for s in range(0, m, chunk):
            cent[s:s + chunk] = mesh.nodes[el[s:s + chunk]].mean(axis=1)
        nu = np.asarray(nu(cent), dtype=float)
    else:
        nu = np.asarray(nu, dtype=float)
    if nu.shape != (m,):
        raise ValueError(f"viscosity must give one value per element, got {nu.shape}")
    if np.any(nu <= 0.0):
        raise ValueError("viscosity must be positive")
    K = np.empty((m, 4, 4))
    F = np.empty((m, 4))

    def work(s):
        Kc, Fc, bad = _chunk_blocks(mesh.nodes[el[s:s + chunk]], nu[s:s + chunk], coeffs)
        if bad < 0:
            K[s:s + chunk] = Kc
            F[s:s + chunk] = Fc
        return s + bad if bad >= 0 else -1

    starts = list(range(0, m, chunk))
    if len(starts) > 1:
        # numpy releases the GIL in these loops: chunks run on a thread pool
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(len(starts), os.cpu_count() or 1)) as ex:
            bads = list(ex.map(work, starts))
    else:
        bads = [work(s) for s in starts]
    bads = [b for b in bads if b >= 0]
    if bads:
        raise ValueError(
            f"shifted reaction c - div(a)/2 is not positive on element {min(bads)}; "
            "the symmetric part of the form would lose definiteness")
    return K, F, nu


def assemble_system(mesh, coeffs, dirichlet_nodes=None):
    """Element blocks + Dirichlet split (reference discretization.py:161-206).

    The global CSR matrix and right-hand side are available lazily as
    ``matrix`` / ``rhs`` / ``full_matrix``."""
    K, F, nu = element_contributions(mesh, coeffs)
    n = mesh.n_nodes
    if dirichlet_nodes is None:
        dirichlet_nodes = mesh.boundary_nodes
    dirichlet_nodes = np.asarray(dirichlet_nodes, dtype=np.int64)
    is_dir = np.zeros(n, dtype=bool)
    is_dir[dirichlet_nodes] = True
    free = np.flatnonzero(~is_dir)
    node_to_free = np.full(n, -1, dtype=np.int64)
    node_to_free[free] = np.arange(free.size)
    g = np.zeros(n)
    if dirichlet_nodes.size:
        g[dirichlet_nodes] = np.asarray(coeffs.dirichlet(mesh.nodes[dirichlet_nodes]), dtype=float)
    dev = None
    dvisc = None
    if coeffs.device_fields is not None:
        df = coeffs.device_fields
        dev = df.packed(coeffs.tau, coeffs.velocity_div is not None)
        dvisc = (np.asarray(df.viscosity_table, dtype=float), int(df.viscosity_period))
    return AssembledSystem(mesh=mesh, free_nodes=free, node_to_free=node_to_free,
                           dirichlet_values=g, elem_matrices=K, elem_rhs=F, viscosity=nu,
                           device_fields=dev, device_viscosity=dvisc)


def solve_direct(system):
    """Sparse direct solve of the assembled system (reference discretization.py:209-215)."""
    import scipy.sparse.linalg

    u = scipy.sparse.linalg.spsolve(system.matrix.tocsc(), system.rhs)
    out = system.dirichlet_values.copy()
    out[system.free_nodes] = u
    return out
