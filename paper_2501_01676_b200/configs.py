"""The BASELINE.json problem configurations as runnable inputs.

The reference harness only builds its own rotating-field example
(reference: pkg/src/adbddc/harness.py:38-57); the BASELINE configs are
generated here through the same library types (``Coefficients``,
``Partition``), with the deviations recorded in BASELINE.md / DESIGN.md:
the "Q1" mesh is the n^3 hex grid split into 6 Kuhn tets (P1), reaction
c = 1, the reference's left-preconditioned full GMRES.  All randomness is
``numpy.random.default_rng(seed)`` with the draw order documented per config.

Config k (1-based, BASELINE.json ``configs[k-1]``):
  1  n=16,  4^3 regular, nu=1e-2, b=(1,1,1)
  2  n=32,  4^3 regular, b=(-(y-1/2), x-1/2, 0.1), nu=1 with 8 channels of 1e-4
  3  n=64,  8^3 regular, nu=1e-3, b=(1,2,3)/sqrt(14)
  4  n=64,  BFS-grown irregular partition from 512 seeds (+ merge repair),
            nu = 10^U(-3,3) per 4^3-cell block, b=(1,1,1)
  5  n=128, 16^3 regular, nu=1e-2, b=(1,1,1)
"""

import math
from collections import deque
from dataclasses import dataclass

import numpy as np

from .decomposition import Partition, classify_globs, node_sharer_pairs, partition_regular
from .discretization import Coefficients, DeviceFields, assemble_system
from .mesh import box_mesh

UNIT = ((0.0, 1.0), (0.0, 1.0), (0.0, 1.0))
THETA = 10.0


def _const_velocity(b):
    b = np.asarray(b, dtype=float)
    return lambda p: np.tile(b, (len(p), 1))


def _coeffs(cell_nu, n, velocity, vel_affine):
    """Per-element viscosity from a per-cell field (element e is cell e % n^3,
    reference mesh.py:75-83).  vel_affine = (A, a0) with velocity(x) = A x + a0:
    the same fields in the form the device element kernel evaluates."""
    n3 = n ** 3
    A, a0 = vel_affine
    return Coefficients(
        viscosity=lambda cent: cell_nu[np.arange(len(cent)) % n3],
        velocity=velocity,
        reaction=lambda p: np.ones(len(p)),
        source=lambda p: np.ones(len(p)),
        dirichlet=lambda p: np.zeros(len(p)),
        device_fields=DeviceFields(np.asarray(A, dtype=float), np.asarray(a0, dtype=float),
                                   1.0, 1.0, np.asarray(cell_nu, dtype=float), n3),
    )


def channel_viscosity(n, n_channels=8, seed=0, background=1.0, channel=1e-4):
    """Config-2 field: per channel draw axis in {0,1,2} then the two
    transverse cell indices; every cell on that line gets ``channel``."""
    rng = np.random.default_rng(seed)
    nu = np.full((n, n, n), background)
    for _ in range(n_channels):
        axis = int(rng.integers(3))
        i, j = (int(v) for v in rng.integers(0, n, size=2))
        if axis == 0:
            nu[:, i, j] = channel
        elif axis == 1:
            nu[i, :, j] = channel
        else:
            nu[i, j, :] = channel
    return nu.ravel()


def block_lognormal_viscosity(n, block=4, lo=-3.0, hi=3.0, seed=0):
    """Config-4 field: 10^U(lo,hi) per block^3 cells, drawn in block
    lexicographic order (bx, by, bz), bz fastest."""
    rng = np.random.default_rng(seed)
    nb = n // block
    draws = 10.0 ** rng.uniform(lo, hi, size=(nb, nb, nb))
    idx = np.arange(n) // block
    return draws[idx[:, None, None], idx[None, :, None], idx[None, None, :]].ravel()


def bfs_cell_partition(n, n_seeds, seed=0):
    """Multi-source FIFO BFS on the 6-neighbour cell graph.

    Seeds: ``rng.choice(n^3, n_seeds, replace=False)``, enqueued in ascending
    cell index; region id = rank of the seed in that order.  The first
    visitor claims a cell; neighbours are visited -x,+x,-y,+y,-z,+z."""
    rng = np.random.default_rng(seed)
    seeds = np.sort(rng.choice(n ** 3, size=n_seeds, replace=False))
    owner = np.full(n ** 3, -1, dtype=np.int64)
    q = deque()
    for r, c in enumerate(seeds.tolist()):
        owner[c] = r
        q.append(c)
    nn = n * n
    while q:
        c = q.popleft()
        ix, rem = divmod(c, nn)
        iy, iz = divmod(rem, n)
        r = owner[c]
        for d, ok in ((-nn, ix > 0), (nn, ix < n - 1), (-n, iy > 0), (n, iy < n - 1),
                      (-1, iz > 0), (1, iz < n - 1)):
            if ok and owner[c + d] < 0:
                owner[c + d] = r
                q.append(c + d)
    return owner


def _cell_face_contacts(n, owner, r):
    """Shared cell-face counts between region r and each other region."""
    g = owner.reshape(n, n, n)
    cnt = {}
    for ax in range(3):
        a = np.moveaxis(g, ax, 0)
        lo, hi = a[:-1], a[1:]
        for x, y in ((lo, hi), (hi, lo)):
            m = (x == r) & (y != r)
            for t, c in zip(*np.unique(y[m], return_counts=True)):
                cnt[int(t)] = cnt.get(int(t), 0) + int(c)
    return cnt


def repair_no_interior(mesh, owner_cells, boundary_mask):
    """Merge regions without interior unknowns into the face neighbour with
    the most shared cell faces (ties -> smaller id), one at a time, smallest
    id first; then relabel consecutively (order preserved)."""
    n = mesh.cells[0]
    n3 = n ** 3
    owner = owner_cells.copy()
    cell_of_elem = np.arange(mesh.n_elements) % n3
    while True:
        part = Partition(owner[cell_of_elem], int(owner.max()) + 1)
        node, sub = node_sharer_pairs(mesh, part)
        count = np.bincount(node, minlength=mesh.n_nodes)
        single = (count[node] == 1) & ~boundary_mask[node]
        has_interior = np.zeros(part.n_subdomains, dtype=bool)
        has_interior[sub[single]] = True
        present = np.zeros(part.n_subdomains, dtype=bool)
        present[owner] = True
        bad = np.flatnonzero(present & ~has_interior)
        if bad.size == 0:
            break
        r = int(bad[0])
        cnt = _cell_face_contacts(n, owner, r)
        target = min(cnt, key=lambda t: (-cnt[t], t))
        owner[owner == r] = target
    labels, owner = np.unique(owner, return_inverse=True)
    return owner.astype(np.int64)


@dataclass
class Problem:
    config: int
    mesh: object
    partition: Partition
    globs: object
    system: object
    theta_f: float
    theta_e: float
    H_over_h: int
    coeffs: object = None

    @property
    def n_dofs(self):
        return self.system.n_free


def build_problem(config, n=None, subs=None, theta_f=THETA, theta_e=THETA, seed=0, device=None):
    """Mesh, partition, globs and element data of one BASELINE config.

    ``n`` / ``subs`` override the mesh and subdomain grid (same coefficients),
    which is how bounded CPU samples of a config are made.  ``device``
    ("cuda"): glob classification on the GPU (same globs)."""
    defaults = {1: (16, 4), 2: (32, 4), 3: (64, 8), 4: (64, None), 5: (128, 16)}
    n0, s0 = defaults[config]
    n = n or n0
    mesh = box_mesh(UNIT, (n, n, n))
    if config == 4:
        n_seeds = subs or 512
        owner = bfs_cell_partition(n, n_seeds, seed)
        owner = repair_no_interior(mesh, owner, mesh.boundary_mask)
        part = Partition(owner[np.arange(mesh.n_elements) % n ** 3], int(owner.max()) + 1)
        Hh = max(2, round((n ** 3 / part.n_subdomains) ** (1.0 / 3.0)))
    else:
        sd = subs or s0
        part = partition_regular(mesh, (sd, sd, sd))
        Hh = n // sd
    Z = np.zeros((3, 3))
    if config == 1:
        b = (1.0, 1.0, 1.0)
        cell_nu, vel, aff = np.full(n ** 3, 1e-2), _const_velocity(b), (Z, b)
    elif config == 2:
        cell_nu = channel_viscosity(n, seed=seed)
        vel = lambda p: np.column_stack([-(p[:, 1] - 0.5), p[:, 0] - 0.5, np.full(len(p), 0.1)])
        aff = ([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 0.0]], (0.5, -0.5, 0.1))
    elif config == 3:
        b = np.array([1.0, 2.0, 3.0]) / math.sqrt(14.0)
        cell_nu, vel, aff = np.full(n ** 3, 1e-3), _const_velocity(b), (Z, b)
    elif config == 4:
        b = (1.0, 1.0, 1.0)
        cell_nu, vel, aff = block_lognormal_viscosity(n, seed=seed), _const_velocity(b), (Z, b)
    elif config == 5:
        b = (1.0, 1.0, 1.0)
        cell_nu, vel, aff = np.full(n ** 3, 1e-2), _const_velocity(b), (Z, b)
    else:
        raise ValueError(f"unknown config {config}")
    globs = classify_globs(mesh, part, mesh.boundary_nodes, device=device)
    coeffs = _coeffs(cell_nu, n, vel, aff)
    system = assemble_system(mesh, coeffs)
    if theta_f is None:
        theta_f = 1.0 + math.log(Hh)
    return Problem(config, mesh, part, globs, system, theta_f, theta_e, Hh, coeffs)
