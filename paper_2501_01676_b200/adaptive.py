"""Adaptive primal space (reference adaptive.py), computed on the device:
face GEPs, priors, new / old edge GEPs and the SVD change of basis all run in
csrc/globs.cu; this module keeps the reference's return types."""

from dataclasses import dataclass

import numpy as np

from .engine import DevicePrimalSpace


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


class PrimalBasis:
    """Per-glob (Q, n_primal) and primal numbering (adaptive.py:209-264).

    Built either from a device primal space (``device``) or, as in the
    reference tests, from an explicit list of (Q, k) per glob."""

    def __init__(self, globs, transforms=None, variant="new", device=None):
        self.globs = globs
        self.variant = variant
        self.device = device
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
        if self.device is not None:
            return [(self.device.q(k), int(self.r[k])) for k in range(len(self.globs.globs))]
        return self._transforms


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


__all__ = ["GevpReport", "PrimalBasis", "adaptive_primal_space"]
