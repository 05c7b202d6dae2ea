"""Structured Kuhn-tetrahedral box meshes (host preprocessing, input side of
the hot path).

Same node numbering, element numbering and orientation as the reference's
``box_mesh`` (reference: pkg/src/adbddc/mesh.py:49-110): nodes lexicographic
in (ix, iy, iz) with iz fastest; six tetrahedra per cell, one block of
``n_cells`` elements per axis-step permutation (so element ``e`` sits in
cell ``e % n_cells``); negatively oriented tets get nodes 2 and 3 swapped.

Unlike the reference, nothing here loops over nodes in Python: the boundary
is a mask, and the dict of boundary tags is only built on request.
"""

import itertools

import numpy as np

_PERMS = list(itertools.permutations(range(3)))


class Mesh:
    """Conforming tetrahedral mesh of an axis-aligned box.

    Attributes mirror the reference ``Mesh`` (mesh.py:16-46): ``nodes``
    (n_nodes, 3), ``elements`` (n_elements, 4), ``box``, ``cells``.
    """

    def __init__(self, nodes, elements, box, cells, boundary_mask):
        self.nodes = nodes
        self.elements = elements
        self.box = box
        self.cells = cells
        self.boundary_mask = boundary_mask
        self._tags = None

    @property
    def n_nodes(self):
        return self.nodes.shape[0]

    @property
    def n_elements(self):
        return self.elements.shape[0]

    @property
    def n_cells(self):
        nx, ny, nz = self.cells
        return nx * ny * nz

    @property
    def boundary_nodes(self):
        return np.flatnonzero(self.boundary_mask)

    @property
    def boundary_tags(self):
        """node -> frozenset of face tags, as in the reference (mesh.py:94-108)."""
        if self._tags is None:
            nx, ny, nz = self.cells
            ijk = self.node_ijk()
            tags = {}
            names = (("x0", "x1", nx), ("y0", "y1", ny), ("z0", "z1", nz))
            for n in self.boundary_nodes.tolist():
                t = set()
                for ax, (lo, hi, cnt) in enumerate(names):
                    if ijk[n, ax] == 0:
                        t.add(lo)
                    elif ijk[n, ax] == cnt:
                        t.add(hi)
                tags[n] = frozenset(t)
            self._tags = tags
        return self._tags

    def node_ijk(self):
        nx, ny, nz = self.cells
        n = np.arange(self.n_nodes)
        iz = n % (nz + 1)
        iy = (n // (nz + 1)) % (ny + 1)
        ix = n // ((nz + 1) * (ny + 1))
        return np.stack([ix, iy, iz], axis=1)


def box_mesh(box, cells):
    """Mesh the box with ``cells[axis]`` grid cells per axis, six Kuhn tets
    per cell (reference mesh.py:49-110)."""
    (x0, x1), (y0, y1), (z0, z1) = box
    nx, ny, nz = (int(c) for c in cells)
    if min(nx, ny, nz) < 1:
        raise ValueError(f"cells must be >= 1 per axis, got {cells}")
    xs = np.linspace(x0, x1, nx + 1)
    ys = np.linspace(y0, y1, ny + 1)
    zs = np.linspace(z0, z1, nz + 1)
    X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
    nodes = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])

    sy, sx = nz + 1, (ny + 1) * (nz + 1)  # node strides
    ix, iy, iz = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    base = (ix.ravel() * sx + iy.ravel() * sy + iz.ravel()).astype(np.int64)
    stride = (sx, sy, 1)

    blocks = []
    for perm in _PERMS:
        offs = [0]
        cur = 0
        for axis in perm:
            cur += stride[axis]
            offs.append(cur)
        blocks.append(base[:, None] + np.asarray(offs, dtype=np.int64)[None, :])
    elements = np.vstack(blocks)

    # orientation is a per-permutation property on a box grid, but evaluate it
    # per element like the reference so skewed inputs behave identically
    verts = nodes[elements]
    det = np.linalg.det(verts[:, 1:] - verts[:, :1])
    neg = det < 0.0
    elements[neg, 2], elements[neg, 3] = elements[neg, 3].copy(), elements[neg, 2].copy()

    bx = np.zeros((nx + 1, ny + 1, nz + 1), dtype=bool)
    bx[0, :, :] = bx[-1, :, :] = True
    bx[:, 0, :] = bx[:, -1, :] = True
    bx[:, :, 0] = bx[:, :, -1] = True
    return Mesh(nodes, elements, box, (nx, ny, nz), bx.ravel())


def element_diameters(mesh):
    """Maximum pairwise vertex distance per element (reference mesh.py:119-123)."""
    verts = mesh.nodes[mesh.elements]
    best = np.zeros(verts.shape[0])
    for a, b in itertools.combinations(range(4), 2):
        d = verts[:, a] - verts[:, b]
        best = np.maximum(best, np.sqrt((d * d).sum(-1)))
    return best
