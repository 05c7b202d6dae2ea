"""Adaptive primal space (reference adaptive.py), computed on the device:
face GEPs, priors, new / old edge GEPs and the SVD change of basis all run in
csrc/globs.cu; this module keeps the reference's return types."""

import logging
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import lib, require_cuda, stream
from .engine import DevicePrimalSpace, dev_i32, dev_i64

log = logging.getLogger(__name__)

SVD_CUT = 1e-10


@dataclass
class GevpReport:
    """adaptive.py:36-47.  With the default detail=True of
    adaptive_primal_space every field is filled from the device run of the
    reference algorithm: pencil_left / pencil_right are (B, B~) of the pencil
    (face: B_F and the parallel sum; edge_new: M and the eliminated B~~;
    edge_old: B_E and the parallel-sum chain), vectors its eigenvectors
    (columns aligned with eigenvalues), degenerate the common-nullspace mask
    and constraint_matrix the selected rows (pencil_left v_sel)^T."""

    glob_id: str
    variant: str
    eigenvalues: np.ndarray
    n_primal: int
    constraint_matrix: np.ndarray
    n_dofs: int
    vectors: np.ndarray = None
    degenerate: np.ndarray = None
    pencil_left: np.ndarray = None
    pencil_right: np.ndarray = None


def _row_spaces(blocks, widths):
    """Device change of basis of a list of row blocks (m_k x n_k): [(Q_k, r_k)]
    with Q_k orthogonal and Q_k[:r_k] spanning the rows (bddc_row_space_batched)."""
    require_cuda()
    m = np.array([b.shape[0] for b in blocks], dtype=np.int64)
    n = np.asarray(widths, dtype=np.int64)
    roff = np.concatenate([[0], np.cumsum(m * n)])
    qoff = np.concatenate([[0], np.cumsum(n * n)])
    wsz = np.array([int(lib.bddc_ws_row_space(int(a), int(b))) for a, b in zip(m, n)], dtype=np.int64)
    woff = np.concatenate([[0], np.cumsum(wsz)])
    flat = np.concatenate([np.asarray(b, dtype=float).ravel() for b in blocks] + [np.zeros(1)])
    rows_d = torch.from_numpy(flat).cuda()
    Q = torch.empty(max(int(qoff[-1]), 1), dtype=torch.float64, device="cuda")
    rank = torch.zeros(len(blocks), dtype=torch.int32, device="cuda")
    ws = torch.empty(max(int(woff[-1]), 1), dtype=torch.float64, device="cuda")
    lib.bddc_row_space_batched(rows_d, dev_i64(roff[:-1]), dev_i32(m), dev_i32(n), len(blocks), Q,
                               dev_i64(qoff[:-1]), rank, ws, dev_i64(woff[:-1]),
                               int(max(m.max(initial=1), n.max(initial=1))), stream())
    Qh, rh = Q.cpu().numpy(), rank.cpu().numpy()
    return [(Qh[qoff[k]:qoff[k + 1]].reshape(n[k], n[k]).copy(), int(rh[k])) for k in range(len(blocks))]


def build_change_of_basis(n_dofs, rows):
    """adaptive.py:190-206: (Q, r), Q n x n orthogonal with Q[:r] an orthonormal
    basis of the constraint rows (rank cut s >= 1e-10 s_max), on the device.
    Q[:r] may differ from the reference's SVD basis by a rotation inside the
    constraint span; every basis-invariant quantity agrees."""
    rows = np.asarray(rows, dtype=float)
    if rows.size == 0:
        return np.eye(n_dofs), 0
    if rows.ndim != 2 or rows.shape[1] != n_dofs:
        raise ValueError(f"constraint rows have width {rows.shape[1]}, expected {n_dofs}")
    Q, r = _row_spaces([rows], [n_dofs])[0]
    if r < rows.shape[0]:
        log.info("change of basis: dropped %d dependent constraint rows", rows.shape[0] - r)
    return Q, r


def reduce_edge_constraints(report):
    """adaptive.py:172-187: difference-space edge rows -> an orthonormal basis of
    the row space of their per-sharer blocks (rows over the edge dofs)."""
    ne = report.n_dofs
    rows = report.constraint_matrix
    if rows is None or rows.size == 0:
        return np.zeros((0, ne))
    Q, r = _row_spaces([rows.reshape(-1, ne)], [ne])[0]
    return Q[:r]


def assemble_primal_space(reports, globs, variant):
    """adaptive.py:267-285: per-glob change of basis from the reports' rows
    (vertices fully primal), all globs in one device launch."""
    blocks, widths, idx = [], [], []
    for k, g in enumerate(globs.globs):
        if g.kind == "vertex":
            continue
        rep = reports[globs.glob_id(g)]
        rows = rep.constraint_matrix
        if g.kind == "edge" and rep.variant == "edge_new":
            rows = reduce_edge_constraints(rep)
        blocks.append(np.asarray(rows, dtype=float).reshape(-1, g.size))
        widths.append(g.size)
        idx.append(k)
    solved = dict(zip(idx, _row_spaces(blocks, widths))) if blocks else {}
    transforms = [(np.eye(g.size), g.size) if g.kind == "vertex" else solved[k]
                  for k, g in enumerate(globs.globs)]
    return PrimalBasis(globs, transforms, variant)


class PrimalBasis:
    """Per-glob (Q, n_primal) and primal numbering (adaptive.py:209-264).

    Built either from a device primal space (``device``) or, as in the
    reference tests, from an explicit list of (Q, k) per glob."""

    def __init__(self, globs, transforms=None, variant="new", device=None):
        self.globs = globs
        self.variant = variant
        self.device = device
        self._transforms = None
        if device is not None:
            r = device.r_host
        else:
            r = np.array([k for _, k in transforms], dtype=np.int64)
            self._transforms = [(np.asarray(Q, dtype=float), int(k)) for Q, k in transforms]
        self.r = np.asarray(r, dtype=np.int64)
        self.glob_primal_offset = list(np.concatenate([[0], np.cumsum(self.r)[:-1]]).astype(int))
        self.n_primal_total = int(self.r.sum())
        kinds = np.array([g.kind for g in globs.globs])
        self.pnumF = int(self.r[kinds == "face"].sum())
        self.pnumE = int(self.r[kinds == "edge"].sum())
        self.n_vertex = int(self.r[kinds == "vertex"].sum())

    @property
    def transforms(self):
        """[(Q, n_primal)] per glob; a device-built basis is copied to the host
        once (one bulk read of all Q blocks)."""
        if self._transforms is None:
            dev = self.device
            Qh = dev.Q.cpu().numpy()
            n = self.globs.globs
            self._transforms = [
                (Qh[dev.q_off[k]:dev.q_off[k] + g.size * g.size].reshape(g.size, g.size),
                 int(self.r[k])) for k, g in enumerate(n)]
        return self._transforms

    def glob_entries(self, op):
        """(glob, Q, n_primal, local positions, primal offset) for every glob
        on the subdomain's boundary (adaptive.py:232-239)."""
        out = []
        for g, (Q, k), off in zip(self.globs.globs, self.transforms, self.glob_primal_offset):
            if op.sub_id in g.sharers:
                out.append((g, Q, k, op.glob_index(g), off))
        return out

    def subdomain_transform(self, op):
        """Dense orthogonal transformation of the subdomain's B dofs (:241-246)."""
        Qi = np.eye(op.n_B)
        for _, Q, _, idx, _ in self.glob_entries(op):
            Qi[np.ix_(idx, idx)] = Q
        return Qi

    def subdomain_primal(self, op):
        """(local primal positions, global primal ids) in matching order (:248-255)."""
        loc, ids = [], []
        for _, _, k, idx, off in self.glob_entries(op):
            loc.extend(idx[:k])
            ids.extend(range(off, off + k))
        return np.array(loc, dtype=int), np.array(ids, dtype=int)

    def apply_interface(self, globs_index, u, transpose=False):
        """Assembled transformation (or its transpose) applied to a global
        interface vector (:257-264); computed on the device, globs grouped by
        size into batched products."""
        require_cuda()
        ud = torch.as_tensor(np.asarray(u, dtype=float)).cuda()
        out = ud.clone()
        groups = {}
        for (Q, _), idx in zip(self.transforms, globs_index):
            if Q is not None:
                groups.setdefault(len(idx), []).append((Q, idx))
        for n, items in groups.items():
            Qs = torch.from_numpy(np.stack([q for q, _ in items])).cuda()
            ix = torch.from_numpy(np.stack([np.asarray(i, dtype=np.int64) for _, i in items])).cuda()
            if transpose:
                Qs = Qs.transpose(1, 2)
            out[ix] = torch.bmm(Qs, ud[ix].unsqueeze(2)).squeeze(2)
        return out.cpu().numpy()


def adaptive_primal_space(globs, ops_list, scaling, theta_f, theta_e, variant, detail=True):
    """Reference signature (adaptive.py:288); returns (PrimalBasis, [GevpReport]).

    detail=True (the reference's behaviour) runs the reference algorithm
    verbatim on the device for every glob and fills every GevpReport field;
    detail=False uses the certified fast paths (same counts and spans, see
    DESIGN.md) and reports eigenvalues and counts only."""
    ls = ops_list[0].ls
    dev = DevicePrimalSpace(ls, scaling.device, theta_f, theta_e, variant, detail=detail)
    basis = PrimalBasis(globs, variant=variant, device=dev)
    reports = []
    eig = dev.all_eigenvalues()
    host = dev.detail.cpu().numpy() if detail else None
    for k, g in enumerate(globs.globs):
        if g.kind == "vertex":
            continue
        v = "face" if g.kind == "face" else ("edge_new" if variant == "new" else "edge_old")
        if detail:
            left, right, vecs, degen, rows = dev.glob_detail(k, host)
        else:
            left = right = vecs = degen = rows = None
        reports.append(GevpReport(globs.glob_id(g), v, eig.get(k, np.zeros(0)),
                                  int(dev.n_sel_host[k]), rows, g.size, vecs, degen, left, right))
    return basis, reports


__all__ = ["GevpReport", "PrimalBasis", "SVD_CUT", "adaptive_primal_space", "assemble_primal_space",
           "build_change_of_basis", "reduce_edge_constraints"]
