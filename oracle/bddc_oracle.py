"""CPU oracle for the adaptive-BDDC hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module; the product (``paper_2501_01676_b200``) never
does and has no CPU fallback.

This is a numpy/scipy restatement of the reference package's per-subdomain
setup and solve (reference: /root/reference/pkg/src/adbddc, cited per
function as ``file:line``).  It calls the same LAPACK / SuperLU routines as
the reference (splu, cho_factor, eigh, svd, lu_factor, lstsq/gelsd), so its
timing is a faithful stand-in for the reference's CPU path on a machine
without ``/root/reference``.

Pinning: ``tests/golden/make_golden.py`` runs the unmodified reference in
the build container and records per-glob eigenvalues and primal counts,
pnumF/pnumE/n_c, GMRES iteration counts, residual histories and solutions;
``tests/test_oracle_golden.py`` checks this module against those fixtures.
"""

import logging
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

log = logging.getLogger(__name__)

SVD_CUT = 1e-10  # adaptive.py:33


class NumericalError(RuntimeError):
    """linalg.py:11"""


# --------------------------------------------------------------------------
# dense kernels (linalg.py)
# --------------------------------------------------------------------------

def _require_symmetric(M, tol, name):
    # linalg.py:15-20
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError(f"{name} must be square, got shape {M.shape}")
    nrm = np.linalg.norm(M)
    if nrm > 0.0 and np.linalg.norm(M - M.T) > tol * nrm:
        raise ValueError(f"{name} is not symmetric to within {tol:g} relative")


def pinv_sym(M, rel_tol=1e-12):
    """Eigen-based pseudo-inverse, cut |w| <= rel_tol*max|w| (linalg.py:23-50)."""
    M = np.asarray(M, dtype=float)
    _require_symmetric(M, 1e-12, "M")
    if M.shape[0] == 0:
        return M.copy()
    w, U = scipy.linalg.eigh(0.5 * (M + M.T))
    keep = np.abs(w) > rel_tol * np.abs(w).max(initial=0.0)
    winv = np.where(keep, 1.0 / np.where(keep, w, 1.0), 0.0)
    P = (U * winv) @ U.T
    return 0.5 * (P + P.T)


def psum(A, B, rel_tol=1e-12):
    """Parallel sum sym(A (A+B)^+ B) (linalg.py:53-67)."""
    A = np.asarray(A, dtype=float)
    B = np.asarray(B, dtype=float)
    if A.shape != B.shape:
        raise ValueError(f"shape mismatch: {A.shape} vs {B.shape}")
    _require_symmetric(A, 1e-12, "A")
    _require_symmetric(B, 1e-12, "B")
    R = A @ pinv_sym(A + B, rel_tol) @ B
    return 0.5 * (R + R.T)


def psum_chain(mats, rel_tol=1e-12):
    """Left-associative parallel-sum chain (linalg.py:70-78)."""
    mats = list(mats)
    if not mats:
        raise ValueError("empty chain")
    acc = np.asarray(mats[0], dtype=float)
    for M in mats[1:]:
        acc = psum(acc, M, rel_tol)
    return acc


@dataclass
class Pencil:
    """Eigenpairs of B v = lambda Btil v (linalg.py:81-113)."""

    values: np.ndarray
    vectors: np.ndarray
    degenerate: np.ndarray

    def mask(self, theta):
        # linalg.py:104-107: ties selected, +inf always, degenerate never
        return (self.values >= theta) & ~self.degenerate


def pencil(B, Bt, rel_tol=1e-12):
    """Symmetric pencil with PSD, possibly singular right side (linalg.py:116-214).

    Output order: +inf modes (by decreasing |beta|), finite modes by
    decreasing lambda, degenerate modes last."""
    B = np.asarray(B, dtype=float)
    Bt = np.asarray(Bt, dtype=float)
    if B.shape != Bt.shape:
        raise ValueError(f"shape mismatch: {B.shape} vs {Bt.shape}")
    _require_symmetric(B, 1e-10, "B")
    _require_symmetric(Bt, 1e-10, "Btil")
    n = B.shape[0]
    if n == 0:
        return Pencil(np.zeros(0), np.zeros((0, 0)), np.zeros(0, dtype=bool))
    B = 0.5 * (B + B.T)
    Bt = 0.5 * (Bt + Bt.T)
    mu, U = scipy.linalg.eigh(Bt)
    mu_max = mu.max(initial=0.0)
    if mu.min(initial=0.0) < -1e-10 * max(mu_max, 1.0):
        raise ValueError("Btil is not positive semidefinite")
    rng = (mu > rel_tol * mu_max) if mu_max > 0.0 else np.zeros(n, dtype=bool)
    V1, V0, mu1 = U[:, rng], U[:, ~rng], mu[rng]
    bscale = np.abs(scipy.linalg.eigvalsh(B)).max(initial=0.0)
    tiny = max(bscale, 1e-300)

    inf_vals, inf_vecs = [], []
    deg = np.zeros((n, 0))
    B00p = None
    if V0.shape[1]:
        beta, P = scipy.linalg.eigh(V0.T @ B @ V0)
        acts = np.abs(beta) > rel_tol * tiny
        for j in np.argsort(-np.abs(beta)):
            if acts[j]:
                inf_vecs.append(V0 @ P[:, j] / np.sqrt(np.abs(beta[j])))
                inf_vals.append(np.inf)
        deg = V0 @ P[:, ~acts]
        B00p = (P[:, acts] / beta[acts]) @ P[:, acts].T

    fin_vals, fin_vecs = [], []
    if V1.shape[1]:
        W1 = V1 / np.sqrt(mu1)
        BW = B @ W1
        Bh = W1.T @ BW
        if B00p is not None:
            C = V0.T @ BW
            Bh = Bh - C.T @ B00p @ C
        lam, Y = scipy.linalg.eigh(0.5 * (Bh + Bh.T))
        Vf = W1 @ Y
        if B00p is not None:
            Vf = Vf - V0 @ (B00p @ (C @ Y))
        floor = 1e-14 * tiny
        for j in np.argsort(-lam):
            v = Vf[:, j]
            if abs(lam[j]) > floor:
                v = v / np.sqrt(abs(lam[j]))
            fin_vals.append(float(lam[j]))
            fin_vecs.append(v)

    deg_vecs = []
    for j in range(deg.shape[1]):
        v = deg[:, j]
        nv = np.linalg.norm(v)
        deg_vecs.append(v / nv if nv > 0.0 else v)
    vals = np.array(inf_vals + fin_vals + [0.0] * len(deg_vecs))
    vecs = inf_vecs + fin_vecs + deg_vecs
    flags = np.array([False] * (len(inf_vals) + len(fin_vals)) + [True] * len(deg_vecs), dtype=bool)
    return Pencil(vals, np.column_stack(vecs) if vecs else np.zeros((n, 0)), flags)


# --------------------------------------------------------------------------
# subdomain operators (substructuring.py)
# --------------------------------------------------------------------------

class LocalOp:
    """Condensed subdomain operator (substructuring.py:23-75)."""

    def __init__(self, sub_id, S, g, lu, f_I, A_IB, interior_nodes, interface_nodes, iface_index):
        self.sub_id = sub_id
        self.S = S
        self.Bsym = 0.5 * (S + S.T)
        self.g = g
        self.lu_II = lu
        self.f_I = f_I
        self.A_IB = A_IB
        self.interior_nodes = interior_nodes
        self.interface_nodes = interface_nodes
        self.iface_index = iface_index
        self._inv = None

    @property
    def n_B(self):
        return self.interface_nodes.size

    def positions(self, nodes):
        p = np.searchsorted(self.interface_nodes, nodes)
        p = np.minimum(p, self.interface_nodes.size - 1)
        if np.any(self.interface_nodes[p] != nodes):
            raise ValueError(f"glob is not on subdomain {self.sub_id}")
        return p

    def bsym_inverse(self):
        # substructuring.py:64-75
        if self._inv is None:
            try:
                c = scipy.linalg.cho_factor(self.Bsym)
            except scipy.linalg.LinAlgError as exc:
                raise NumericalError(
                    f"Bsym of subdomain {self.sub_id} is not positive definite "
                    f"(cond ~ {np.linalg.cond(self.Bsym):.2e})") from exc
            self._inv = scipy.linalg.cho_solve(c, np.eye(self.n_B))
        return self._inv


def local_operator(system, part, globs, i, elems=None):
    """Local assembly, lifting, splu(A_II), dense S and g (substructuring.py:78-143)."""
    el_all = system.mesh.elements
    if elems is None:
        elems = np.flatnonzero(part.subdomain_of == i)
    if elems.size == 0:
        raise ValueError(f"subdomain {i} has no elements")
    conn = el_all[elems]
    nodes = np.unique(conn)
    free = system.node_to_free[nodes] >= 0
    iface = np.isin(nodes, globs.interface_nodes)
    B_nodes = nodes[free & iface]
    I_nodes = nodes[free & ~iface]
    D_nodes = nodes[~free]
    if B_nodes.size == 0:
        raise ValueError(f"subdomain {i} has no interface unknowns")
    if I_nodes.size == 0:
        raise ValueError(f"subdomain {i} has no interior unknowns")
    nI, nB = I_nodes.size, B_nodes.size
    order = np.concatenate([I_nodes, B_nodes, D_nodes])
    perm = np.argsort(order)
    loc = perm[np.searchsorted(order[perm], conn)]
    nl = order.size
    A = scipy.sparse.coo_matrix(
        (system.elem_matrices[elems].ravel(),
         (np.repeat(loc, 4, axis=1).ravel(), np.tile(loc, (1, 4)).ravel())),
        shape=(nl, nl)).tocsr()
    load = np.zeros(nl)
    np.add.at(load, loc.ravel(), system.elem_rhs[elems].ravel())
    f = load[:nI + nB] - A[:nI + nB, nI + nB:] @ system.dirichlet_values[D_nodes]
    A_II = A[:nI, :nI].tocsc()
    A_IB = A[:nI, nI:nI + nB].tocsr()
    A_BI = A[nI:nI + nB, :nI].tocsr()
    A_BB = A[nI:nI + nB, nI:nI + nB]
    try:
        lu = scipy.sparse.linalg.splu(A_II)
    except RuntimeError as exc:
        raise NumericalError(f"interior block of subdomain {i} is singular") from exc
    S = A_BB.toarray() - A_BI @ lu.solve(A_IB.toarray())
    g = f[nI:] - A_BI @ lu.solve(f[:nI])
    return LocalOp(i, S, g, lu, f[:nI], A_IB, I_nodes, B_nodes, globs.interface_index(B_nodes))


def all_local_operators(system, part, globs):
    order = np.argsort(part.subdomain_of, kind="stable")
    cuts = np.searchsorted(part.subdomain_of[order], np.arange(part.n_subdomains + 1))
    return [local_operator(system, part, globs, i, order[cuts[i]:cuts[i + 1]])
            for i in range(part.n_subdomains)]


def schur_block(Minv, idx, sub_id):
    """((Minv)[X,X])^-1 by Cholesky, symmetrised (substructuring.py:161-171)."""
    blk = Minv[np.ix_(idx, idx)]
    try:
        c = scipy.linalg.cho_factor(blk)
        out = scipy.linalg.cho_solve(c, np.eye(len(idx)))
    except scipy.linalg.LinAlgError as exc:
        raise NumericalError(
            f"glob Schur block on subdomain {sub_id} is singular "
            f"(cond ~ {np.linalg.cond(blk):.2e})") from exc
    return 0.5 * (out + out.T)


def principal(op, g):
    idx = op.positions(g.nodes)
    return op.Bsym[np.ix_(idx, idx)]


# --------------------------------------------------------------------------
# deluxe scaling (scaling.py)
# --------------------------------------------------------------------------

def deluxe_family(blocks):
    """D_s = (sum_k B_k)^-1 B_s (scaling.py:10-25)."""
    sh = sorted(blocks)
    T = sum(blocks[s] for s in sh)
    try:
        c = scipy.linalg.cho_factor(T)
    except scipy.linalg.LinAlgError as exc:
        raise NumericalError(
            f"deluxe block sum is singular (cond ~ {np.linalg.cond(T):.2e})") from exc
    return {s: scipy.linalg.cho_solve(c, blocks[s]) for s in sh}


def scaling_families(globs, ops):
    """Per-glob family: deluxe for faces/edges, 1/|n(V)| for vertices (scaling.py:28-57)."""
    by = {op.sub_id: op for op in ops}
    fam = []
    for g in globs.globs:
        if g.kind == "vertex" and g.size == 1:
            fam.append({s: np.array([[1.0 / len(g.sharers)]]) for s in g.sharers})
        else:
            fam.append(deluxe_family({s: principal(by[s], g) for s in g.sharers}))
    return fam


# --------------------------------------------------------------------------
# adaptive primal space (adaptive.py)
# --------------------------------------------------------------------------

@dataclass
class GlobReport:
    """adaptive.py:36-47 (subset used for parity)."""

    glob_id: str
    variant: str
    eigenvalues: np.ndarray
    n_primal: int
    rows: np.ndarray
    n_dofs: int
    vectors: np.ndarray = None
    degenerate: np.ndarray = None
    left: np.ndarray = None
    right: np.ndarray = None


def _pencil_or_raise(B, Bt, gid):
    # adaptive.py:50-54
    try:
        return pencil(B, Bt)
    except (ValueError, NumericalError) as exc:
        raise NumericalError(f"eigenproblem on glob {gid} failed: {exc}") from exc


def face_report(gid, F, ops, D, theta):
    """adaptive.py:57-72"""
    i, j = F.sharers
    Bi, Bj = principal(ops[i], F), principal(ops[j], F)
    BF = D[j].T @ Bi @ D[j] + D[i].T @ Bj @ D[i]
    BF = 0.5 * (BF + BF.T)
    ti = schur_block(ops[i].bsym_inverse(), ops[i].positions(F.nodes), i)
    tj = schur_block(ops[j].bsym_inverse(), ops[j].positions(F.nodes), j)
    Bt = psum(ti, tj)
    p = _pencil_or_raise(BF, Bt, gid)
    m = p.mask(theta)
    return GlobReport(gid, "face", p.values, int(m.sum()), (BF @ p.vectors[:, m]).T, F.size,
                      p.vectors, p.degenerate, BF, Bt)


def edge_report_old(gid, E, ops, D, theta):
    """adaptive.py:75-91"""
    sh = list(E.sharers)
    BE = np.zeros((E.size, E.size))
    for i in sh:
        Bi = principal(ops[i], E)
        for k in sh:
            if k != i:
                BE += D[k].T @ Bi @ D[k]
    BE = 0.5 * (BE + BE.T)
    Bt = psum_chain([schur_block(ops[s].bsym_inverse(), ops[s].positions(E.nodes), s) for s in sh])
    p = _pencil_or_raise(BE, Bt, gid)
    m = p.mask(theta)
    return GlobReport(gid, "edge_old", p.values, int(m.sum()), (BE @ p.vectors[:, m]).T, E.size,
                      p.vectors, p.degenerate, BE, Bt)


def edge_report_new(gid, E, ops, D, theta, blocks):
    """adaptive.py:94-156; blocks[s] = (EE, EH, HE, HH)."""
    sh = list(E.sharers)
    n, ne = len(sh), E.size
    Ds = [D[s] for s in sh]
    nC = (n - 1) * ne
    eye = np.eye(ne)
    J = [np.hstack([(eye if i == k else 0.0) - Ds[k] for k in range(1, n)]) for i in range(n)]
    M = np.zeros((nC, nC))
    for i, s in enumerate(sh):
        M += J[i].T @ principal(ops[s], E) @ J[i]
    M = 0.5 * (M + M.T)
    nH = [blocks[s][3].shape[0] for s in sh]
    W = nC + ne + sum(nH)
    Bt = np.zeros((W, W))
    off = nC + ne
    for i, s in enumerate(sh):
        EE, EH, HE, HH = blocks[s]
        T = np.hstack([J[i], eye])
        h = slice(off, off + nH[i])
        Bt[:nC + ne, :nC + ne] += T.T @ EE @ T
        Bt[:nC + ne, h] += T.T @ EH
        Bt[h, :nC + ne] += HE @ T
        Bt[h, h] += HH
        off += nH[i]
    Bt = 0.5 * (Bt + Bt.T)
    KK, KR, RR = Bt[:nC, :nC], Bt[:nC, nC:], Bt[nC:, nC:]
    try:
        c = scipy.linalg.cho_factor(RR)
        Btt = KK - KR @ scipy.linalg.cho_solve(c, KR.T)
    except scipy.linalg.LinAlgError:
        log.info("edge %s: singular elimination block, pseudo-inverse used", gid)
        Btt = KK - KR @ pinv_sym(RR) @ KR.T
    Btt = 0.5 * (Btt + Btt.T)
    p = _pencil_or_raise(M, Btt, gid)
    m = p.mask(theta)
    return GlobReport(gid, "edge_new", p.values, int(m.sum()), (M @ p.vectors[:, m]).T, ne,
                      p.vectors, p.degenerate, M, Btt)


def reduce_rows(rows, ne):
    """SVD compression of stacked difference rows (adaptive.py:172-187)."""
    if rows.size == 0:
        return np.zeros((0, ne))
    _, s, Vt = scipy.linalg.svd(rows.reshape(-1, ne), full_matrices=False)
    return Vt[s >= SVD_CUT * s[0]] if s.size else np.zeros((0, ne))


def change_of_basis(n, rows):
    """(Q, r): full SVD, Q = V^T, r = #{s >= 1e-10 s0} (adaptive.py:190-206)."""
    rows = np.asarray(rows, dtype=float)
    if rows.size == 0:
        return np.eye(n), 0
    if rows.shape[1] != n:
        raise ValueError(f"constraint rows have width {rows.shape[1]}, expected {n}")
    _, s, Vt = scipy.linalg.svd(rows, full_matrices=True)
    return Vt, int(np.count_nonzero(s >= SVD_CUT * s[0]))


def primal_space(globs, ops_list, fam, theta_f, theta_e, variant):
    """Faces first, then edges ("old" or prior-aware "new"); returns
    (transforms [(Q, r) per glob], reports dict) (adaptive.py:267-342)."""
    ops = {op.sub_id: op for op in ops_list}
    gidx = {id(g): k for k, g in enumerate(globs.globs)}
    reports = {}
    for F in globs.faces:
        k = gidx[id(F)]
        reports[k] = face_report(f"F{k}", F, ops, fam[k], theta_f)
    if variant == "old":
        for E in globs.edges:
            k = gidx[id(E)]
            reports[k] = edge_report_old(f"E{k}", E, ops, fam[k], theta_e)
    elif variant == "new":
        fq = {gidx[id(F)]: change_of_basis(F.size, reports[gidx[id(F)]].rows) for F in globs.faces}
        tinv, prior = {}, {}
        for op in ops_list:
            Minv = op.bsym_inverse().copy()
            pidx = []
            for g in globs.globs:
                if op.sub_id not in g.sharers:
                    continue
                idx = op.positions(g.nodes)
                if g.kind == "vertex":
                    pidx.extend(idx)
                elif g.kind == "face":
                    Q, r = fq[gidx[id(g)]]
                    Minv[idx, :] = Q @ Minv[idx, :]
                    Minv[:, idx] = Minv[:, idx] @ Q.T
                    pidx.extend(idx[:r])
            tinv[op.sub_id] = Minv
            prior[op.sub_id] = np.asarray(pidx, dtype=np.int64)
        for E in globs.edges:
            k = gidx[id(E)]
            blocks = {}
            for s in E.sharers:
                op = ops[s]
                e_idx = op.positions(E.nodes)
                full = schur_block(tinv[s], np.concatenate([e_idx, prior[s]]), s)
                ne = e_idx.size
                blocks[s] = (full[:ne, :ne], full[:ne, ne:], full[ne:, :ne], full[ne:, ne:])
            reports[k] = edge_report_new(f"E{k}", E, ops, fam[k], theta_e, blocks)
    else:
        raise ValueError(f"unknown variant {variant!r}")
    transforms = []
    for k, g in enumerate(globs.globs):
        if g.kind == "vertex":
            transforms.append((np.eye(g.size), g.size))
            continue
        rep = reports[k]
        rows = reduce_rows(rep.rows, g.size) if rep.variant == "edge_new" else rep.rows
        transforms.append(change_of_basis(g.size, rows))
    return transforms, reports


def primal_counts(globs, transforms):
    pf = sum(r for g, (_, r) in zip(globs.globs, transforms) if g.kind == "face")
    pe = sum(r for g, (_, r) in zip(globs.globs, transforms) if g.kind == "edge")
    pv = sum(r for g, (_, r) in zip(globs.globs, transforms) if g.kind == "vertex")
    return pf, pe, pv


# --------------------------------------------------------------------------
# preconditioner and Krylov driver (solver.py)
# --------------------------------------------------------------------------

class Preconditioner:
    """M^-1 = Qhat^T Rtil^T Dtil Stil^-1 Dtil^T Rtil Qhat (solver.py:46-209)."""

    def __init__(self, ops, globs, transforms, fam):
        self.ops = sorted(ops, key=lambda o: o.sub_id)
        self.n_hat = globs.interface_nodes.size
        offs = np.concatenate([[0], np.cumsum([r for _, r in transforms])]).astype(np.int64)
        self.n_primal = int(offs[-1])
        if self.n_primal == 0:
            raise NumericalError("empty primal space: no coarse problem to anchor the solver")
        self.transforms = transforms
        self.gpos = [globs.interface_index(g.nodes) for g in globs.globs]
        self.primal_pos = np.concatenate(
            [p[:r] for p, (_, r) in zip(self.gpos, transforms)]).astype(np.int64)
        sub_globs = {op.sub_id: [] for op in self.ops}
        for k, g in enumerate(globs.globs):
            for s in g.sharers:
                if s in sub_globs:
                    sub_globs[s].append(k)
        coarse = np.zeros((self.n_primal, self.n_primal))
        self.dual, self.ploc, self.gprim, self.gdual = [], [], [], []
        self.lu, self.SdP, self.SPd, self.Dbar = [], [], [], []
        for op in self.ops:
            Qi = np.eye(op.n_B)
            Db = np.zeros((op.n_B, op.n_B))
            ploc, gids = [], []
            for k in sub_globs[op.sub_id]:
                g = globs.globs[k]
                Q, r = transforms[k]
                idx = op.positions(g.nodes)
                Qi[np.ix_(idx, idx)] = Q
                Db[np.ix_(idx, idx)] = Q @ fam[k][op.sub_id] @ Q.T
                ploc.extend(idx[:r])
                gids.extend(range(offs[k], offs[k] + r))
            ploc = np.asarray(ploc, dtype=np.int64)
            gids = np.asarray(gids, dtype=np.int64)
            dual = np.setdiff1d(np.arange(op.n_B), ploc)
            Sb = Qi @ op.S @ Qi.T
            Sdd = Sb[np.ix_(dual, dual)]
            if dual.size:
                try:
                    scipy.linalg.cho_factor(0.5 * (Sdd + Sdd.T))
                except scipy.linalg.LinAlgError as exc:
                    raise NumericalError(
                        f"dual block of subdomain {op.sub_id} lost positive definiteness") from exc
                lu = scipy.linalg.lu_factor(Sdd)
            else:
                lu = None
            SdP = Sb[np.ix_(dual, ploc)]
            SPd = Sb[np.ix_(ploc, dual)]
            SPP = Sb[np.ix_(ploc, ploc)]
            coarse[np.ix_(gids, gids)] += (SPP - SPd @ scipy.linalg.lu_solve(lu, SdP)) if dual.size else SPP
            self.dual.append(dual)
            self.ploc.append(ploc)
            self.gprim.append(gids)
            self.gdual.append(op.iface_index[dual])
            self.lu.append(lu)
            self.SdP.append(SdP)
            self.SPd.append(SPd)
            self.Dbar.append(Db)
        self.doff = np.concatenate([[0], np.cumsum([d.size for d in self.dual])]).astype(np.int64)
        self.n_dual = int(self.doff[-1])
        self.coarse = coarse
        self.coarse_lu = scipy.linalg.lu_factor(coarse)
        dg = np.abs(np.diag(self.coarse_lu[0]))
        if dg.size and dg.min() <= 1e-14 * max(dg.max(), 1.0):
            bad = int(np.argmin(dg))
            gk = int(np.searchsorted(offs[:-1], bad, side="right")) - 1
            g = globs.globs[gk]
            raise NumericalError(
                f"coarse matrix is singular at primal dof {bad} "
                f"(glob {g.kind[0].upper()}{gk}, constraint {bad - offs[gk]})")

    def _Q(self, u, transpose):
        out = u.copy()
        for (Q, _), p in zip(self.transforms, self.gpos):
            out[p] = (Q.T if transpose else Q) @ u[p]
        return out

    def apply(self, r):
        """solver.py:201-209 with transform/inject/scale/tilde_solve/inject_t inlined."""
        v = self._Q(r, False)
        nd = self.n_dual
        wp = v[self.primal_pos]
        ys, rp = [], np.zeros(self.n_primal)
        for i, op in enumerate(self.ops):  # scale(transpose=True) then dual solve
            x = np.zeros(op.n_B)
            x[self.dual[i]] = v[self.gdual[i]]
            x[self.ploc[i]] = wp[self.gprim[i]]
            y = self.Dbar[i].T @ x
            rp[self.gprim[i]] += y[self.ploc[i]]
            ys.append(y[self.dual[i]])
        zs = []
        for i in range(len(self.ops)):
            if self.dual[i].size:
                z = scipy.linalg.lu_solve(self.lu[i], ys[i])
                rp[self.gprim[i]] -= self.SPd[i] @ z
            else:
                z = np.zeros(0)
            zs.append(z)
        up = scipy.linalg.lu_solve(self.coarse_lu, rp)
        out = np.zeros(self.n_hat)
        acc = np.zeros(self.n_primal)
        for i, op in enumerate(self.ops):
            x = np.zeros(op.n_B)
            if self.dual[i].size:
                x[self.dual[i]] = zs[i] - scipy.linalg.lu_solve(self.lu[i], self.SdP[i] @ up[self.gprim[i]])
            x[self.ploc[i]] = up[self.gprim[i]]
            y = self.Dbar[i] @ x
            out[self.gdual[i]] += y[self.dual[i]]
            acc[self.gprim[i]] += y[self.ploc[i]]
        out[self.primal_pos] += acc
        return self._Q(out, True)


def interface_apply(ops, n):
    """S_hat u = sum R_i^T S_i R_i u (solver.py:226-235)."""
    def apply(u):
        out = np.zeros(n)
        for op in ops:
            out[op.iface_index] += op.S @ u[op.iface_index]
        return out
    return apply


def interface_rhs(ops, n):
    """solver.py:238-242"""
    g = np.zeros(n)
    for op in ops:
        g[op.iface_index] += op.g
    return g


@dataclass
class GmresResult:
    iterations: int
    converged: bool
    solution: np.ndarray
    residual_history: list
    preconditioned_history: list
    extra: dict = field(default_factory=dict)


def gmres(operator, rhs, pc, rel_tol=1e-8, max_iter=300):
    """Full left-preconditioned GMRES, MGS twice, gelsd per step
    (solver.py:262-315)."""
    n = rhs.shape[0]
    z0 = pc.apply(rhs)
    ref = np.linalg.norm(z0)
    if ref == 0.0:
        return GmresResult(0, True, np.zeros(n), [0.0], [0.0])
    V = np.zeros((n, max_iter + 1))
    H = np.zeros((max_iter + 1, max_iter))
    V[:, 0] = z0 / ref
    e1 = np.zeros(max_iter + 1)
    e1[0] = ref
    x = np.zeros(n)
    th, ph = [], []
    conv = False
    it = 0
    for j in range(max_iter):
        w = pc.apply(operator(V[:, j]))
        for _pass in range(2):
            for i in range(j + 1):
                c = V[:, i] @ w
                H[i, j] += c
                w -= c * V[:, i]
        H[j + 1, j] = np.linalg.norm(w)
        y = scipy.linalg.lstsq(H[:j + 2, :j + 1], e1[:j + 2], lapack_driver="gelsd")[0]
        res = np.linalg.norm(e1[:j + 2] - H[:j + 2, :j + 1] @ y)
        x = V[:, :j + 1] @ y
        it = j + 1
        ph.append(res / ref)
        th.append(np.linalg.norm(rhs - operator(x)))
        if ph[-1] <= rel_tol:
            conv = True
            break
        if H[j + 1, j] <= 1e-14 * ref:
            conv = ph[-1] <= rel_tol
            break
        V[:, j + 1] = w / H[j + 1, j]
    return GmresResult(it, conv, x, th, ph)


def recover(ops, globs, system, u_hat):
    """Interior back-substitution (solver.py:318-326)."""
    u = system.dirichlet_values.copy()
    u[globs.interface_nodes] = u_hat
    for op in ops:
        u[op.interior_nodes] = op.lu_II.solve(op.f_I - op.A_IB @ u[op.interface_nodes])
    return u


# --------------------------------------------------------------------------
# whole hot path
# --------------------------------------------------------------------------

def run_pipeline(system, part, globs, theta_f, theta_e, variant="new", rel_tol=1e-8,
                 max_iter=300, keep=False):
    """Setup + solve + recovery with phase timings (seconds)."""
    t = {}
    t0 = time.perf_counter()
    ops = all_local_operators(system, part, globs)
    t["subdomain_ops"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    fam = scaling_families(globs, ops)
    t["scaling"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    for op in ops:
        op.bsym_inverse()
    t["bsym_inverse"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    transforms, reports = primal_space(globs, ops, fam, theta_f, theta_e, variant)
    t["gevp"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    pc = Preconditioner(ops, globs, transforms, fam)
    t["pc_setup"] = time.perf_counter() - t1
    n = globs.interface_nodes.size
    t1 = time.perf_counter()
    rep = gmres(interface_apply(ops, n), interface_rhs(ops, n), pc, rel_tol, max_iter)
    t["gmres"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    u = recover(ops, globs, system, rep.solution)
    t["recover"] = time.perf_counter() - t1
    t["total"] = time.perf_counter() - t0
    pf, pe, pv = primal_counts(globs, transforms)
    out = dict(iterations=rep.iterations, converged=rep.converged, solution=rep.solution, u=u,
               pnumF=pf, pnumE=pe, n_vertex=pv, n_c=pf + pe + pv,
               n_primal={k: t_[1] for k, t_ in enumerate(transforms)},
               eigenvalues={k: r.eigenvalues for k, r in reports.items()},
               residual_history=rep.residual_history,
               preconditioned_history=rep.preconditioned_history, timings=t)
    if keep:
        out.update(ops=ops, fam=fam, transforms=transforms, reports=reports, pc=pc)
    return out
