"""Element partitions and interface glob classification (host preprocessing,
input side of the hot path).

Produces exactly the reference's glob list and numbering (reference:
pkg/src/adbddc/decomposition.py:204-325): faces (two sharers) ordered by
sharer tuple, then edges ordered by first node, then vertices ordered by
node; glob ids are kind letter + list index; the global interface numbering
is the sorted unique interface nodes.  The parity of every downstream count
depends on this order, so the classification is restated rule for rule but
vectorised: sharer sets come from one sort of (node, subdomain) pairs, and
only the nodes shared by three or more subdomains (a small set) go through
the component / vertex-promotion logic.
"""

from collections import defaultdict, deque
from dataclasses import dataclass

import numpy as np


@dataclass
class Partition:
    """Element -> subdomain map (reference decomposition.py:20-29)."""

    subdomain_of: np.ndarray
    n_subdomains: int

    def elements_of(self, s):
        return np.flatnonzero(self.subdomain_of == s)

    def sizes(self):
        return np.bincount(self.subdomain_of, minlength=self.n_subdomains)


def partition_regular(mesh, subs):
    """Box grid of subdomains numbered (sx*Ny + sy)*Nz + sz
    (reference decomposition.py:32-44)."""
    nx, ny, nz = mesh.cells
    Nx, Ny, Nz = subs
    if nx % Nx or ny % Ny or nz % Nz:
        raise ValueError(f"cells {mesh.cells} not divisible by subdomain grid {subs}")
    (x0, x1), (y0, y1), (z0, z1) = mesh.box
    cent = mesh.nodes[mesh.elements].mean(axis=1)
    sx = np.floor((cent[:, 0] - x0) / (x1 - x0) * Nx).astype(np.int64).clip(0, Nx - 1)
    sy = np.floor((cent[:, 1] - y0) / (y1 - y0) * Ny).astype(np.int64).clip(0, Ny - 1)
    sz = np.floor((cent[:, 2] - z0) / (z1 - z0) * Nz).astype(np.int64).clip(0, Nz - 1)
    return Partition((sx * Ny + sy) * Nz + sz, Nx * Ny * Nz)


@dataclass(eq=False)
class Glob:
    """Face, edge or vertex equivalence class (reference decomposition.py:204-212)."""

    kind: str
    nodes: np.ndarray
    sharers: tuple

    @property
    def size(self):
        return len(self.nodes)


class GlobSet:
    """Globs plus the global interface numbering (reference decomposition.py:215-239)."""

    def __init__(self, globs):
        self.globs = globs
        if globs:
            self.interface_nodes = np.unique(np.concatenate([g.nodes for g in globs]))
        else:
            self.interface_nodes = np.zeros(0, dtype=np.int64)
        self._pos = {id(g): k for k, g in enumerate(globs)}
        self._flat = flatten_globs(globs)  # array form consumed by the symbolic plan

    @property
    def faces(self):
        return [g for g in self.globs if g.kind == "face"]

    @property
    def edges(self):
        return [g for g in self.globs if g.kind == "edge"]

    @property
    def vertices(self):
        return [g for g in self.globs if g.kind == "vertex"]

    def index(self, g):
        return self._pos[id(g)]

    def flat(self):
        """Flat arrays of the glob list (kind code, size, sharers, nodes),
        built with the GlobSet: the symbolic plan's input format."""
        return self._flat

    def glob_id(self, g):
        return f"{g.kind[0].upper()}{self._pos[id(g)]}"

    def interface_index(self, nodes):
        nodes = np.atleast_1d(np.asarray(nodes, dtype=np.int64))
        pos = np.searchsorted(self.interface_nodes, nodes)
        pos = np.minimum(pos, max(self.interface_nodes.size - 1, 0))
        if nodes.size and (self.interface_nodes.size == 0
                           or np.any(self.interface_nodes[pos] != nodes)):
            bad = nodes[self.interface_nodes[pos] != nodes][0] if self.interface_nodes.size else nodes[0]
            raise KeyError(int(bad))
        return pos.astype(np.int64)


_KIND_CODE = {"face": 0, "edge": 1, "vertex": 2}


def flatten_globs(globs):
    """(kind, size, sharer_count, sharers_flat, nodes_flat) of a glob list."""
    kind = np.fromiter((_KIND_CODE[g.kind] for g in globs), dtype=np.int32, count=len(globs))
    size = np.fromiter((len(g.nodes) for g in globs), dtype=np.int32, count=len(globs))
    nsh = np.fromiter((len(g.sharers) for g in globs), dtype=np.int64, count=len(globs))
    sharers = (np.fromiter((s for g in globs for s in g.sharers), dtype=np.int64, count=int(nsh.sum()))
               if globs else np.zeros(0, np.int64))
    nodes = np.concatenate([g.nodes for g in globs]).astype(np.int64) if globs else np.zeros(0, np.int64)
    return {"kind": kind, "size": size, "nsh": nsh, "sharers": sharers, "nodes": nodes}


_TET_EDGES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


def node_sharer_pairs(mesh, part):
    """Sorted unique (node, subdomain) pairs as two arrays."""
    N = int(part.n_subdomains)
    key = mesh.elements.astype(np.int64) * N + np.asarray(part.subdomain_of, dtype=np.int64)[:, None]
    key = np.unique(key.ravel())
    return key // N, key % N


def _adjacency_among(mesh, member_mask):
    """Undirected node adjacency (element edges) restricted to member nodes."""
    el = mesh.elements
    nbrs = defaultdict(set)
    for a, b in _TET_EDGES:
        u, v = el[:, a], el[:, b]
        keep = member_mask[u] & member_mask[v]
        if not keep.any():
            continue
        pairs = np.unique(np.stack([np.minimum(u[keep], v[keep]),
                                    np.maximum(u[keep], v[keep])], axis=1), axis=0)
        for x, y in pairs.tolist():
            nbrs[x].add(y)
            nbrs[y].add(x)
    return nbrs


def _components(members, adj):
    """Connected components in order of smallest start node; each sorted
    (reference decomposition.py:63-79)."""
    members = set(members)
    comps = []
    while members:
        start = min(members)
        comp = [start]
        members.remove(start)
        queue = deque([start])
        while queue:
            for nb in adj.get(queue.popleft(), ()):
                if nb in members:
                    members.remove(nb)
                    comp.append(nb)
                    queue.append(nb)
        comps.append(sorted(comp))
    return comps


def _faces_and_multi_host(mesh, part, dirichlet_nodes):
    """Face node groups (nodes sorted by (s0, s1, node) with their sharer pair)
    and the nodes with >= 3 sharers with their sharer tuples, on the host."""
    node, sub = node_sharer_pairs(mesh, part)
    n_nodes = mesh.n_nodes
    is_dir = np.zeros(n_nodes, dtype=bool)
    is_dir[np.asarray(dirichlet_nodes, dtype=np.int64)] = True
    count = np.bincount(node, minlength=n_nodes)
    start = np.zeros(n_nodes + 1, dtype=np.int64)
    np.cumsum(count, out=start[1:])
    two = np.flatnonzero((count == 2) & ~is_dir)
    s0 = sub[start[two]]
    s1 = sub[start[two] + 1]
    order = np.lexsort((two, s1, s0))
    multi = np.flatnonzero((count >= 3) & ~is_dir)
    mcount = count[multi]
    msub = sub[np.repeat(start[multi], mcount) + np.arange(int(mcount.sum())) -
               np.repeat(np.cumsum(mcount) - mcount, mcount)] if multi.size else np.zeros(0, np.int64)
    member = np.zeros(n_nodes, dtype=bool)
    member[multi] = True
    return two[order], s0[order], s1[order], multi, mcount, msub, _adjacency_among(mesh, member)


def _faces_and_multi_device(mesh, part, dirichlet_nodes, device):
    """Same outputs as _faces_and_multi_host; the sharer pairs of all element
    corners (a sort-unique of 4 x n_elements keys), the sharer counts, the face
    grouping sort and the member-edge filter run on the GPU (torch); only the
    small sets (face nodes, nodes with >= 3 sharers, their edges) come back."""
    import torch

    N = int(part.n_subdomains)
    n_nodes = mesh.n_nodes
    el = torch.from_numpy(np.ascontiguousarray(mesh.elements, dtype=np.int64)).to(device)
    so = torch.from_numpy(np.ascontiguousarray(part.subdomain_of, dtype=np.int64)).to(device)
    key = torch.unique((el * N + so[:, None]).reshape(-1))        # sorted (node, sub) pairs
    node, sub = key // N, key % N
    count = torch.bincount(node, minlength=n_nodes)
    start = torch.zeros(n_nodes + 1, dtype=torch.int64, device=device)
    torch.cumsum(count, 0, out=start[1:])
    is_dir = torch.zeros(n_nodes, dtype=torch.bool, device=device)
    is_dir[torch.from_numpy(np.asarray(dirichlet_nodes, dtype=np.int64)).to(device)] = True
    two = torch.nonzero((count == 2) & ~is_dir).squeeze(1)
    s0, s1 = sub[start[two]], sub[start[two] + 1]
    fkey = (s0 * N + s1) * n_nodes + two
    order = torch.sort(fkey).indices
    two, s0, s1 = two[order], s0[order], s1[order]
    multi = torch.nonzero((count >= 3) & ~is_dir).squeeze(1)
    mcount = count[multi]
    idx = torch.repeat_interleave(start[multi], mcount) + torch.arange(int(mcount.sum()), device=device) \
        - torch.repeat_interleave(torch.cumsum(mcount, 0) - mcount, mcount)
    msub = sub[idx]
    member = torch.zeros(n_nodes, dtype=torch.bool, device=device)
    member[multi] = True
    pairs = []
    for a, b in _TET_EDGES:
        u, v = el[:, a], el[:, b]
        keep = member[u] & member[v]
        pairs.append(torch.stack([torch.minimum(u[keep], v[keep]), torch.maximum(u[keep], v[keep])], 1))
    pairs = torch.unique(torch.cat(pairs), dim=0).cpu().numpy()
    nbrs = defaultdict(set)
    for x, y in pairs.tolist():
        nbrs[x].add(y)
        nbrs[y].add(x)
    host = lambda t: t.cpu().numpy()
    return host(two), host(s0), host(s1), host(multi), host(mcount), host(msub), nbrs


def classify_globs(mesh, part, dirichlet_nodes, device=None):
    """Faces / edges / vertices of the interface (reference decomposition.py:253-325).

    device (e.g. "cuda"): the sharer pairs, counts and face grouping are
    computed on the GPU (identical result, tests/test_gpu_elements.py)."""
    if device is not None:
        two, s0, s1, multi, mcount, msub, nbrs = _faces_and_multi_device(mesh, part,
                                                                         dirichlet_nodes, device)
    else:
        two, s0, s1, multi, mcount, msub, nbrs = _faces_and_multi_host(mesh, part, dirichlet_nodes)

    # faces: nodes with exactly two sharers, grouped by (s0, s1)
    globs = []
    if two.size:
        cut = np.flatnonzero((np.diff(s0) != 0) | (np.diff(s1) != 0)) + 1
        for a, b in zip(np.concatenate([[0], cut]), np.concatenate([cut, [two.size]])):
            globs.append(Glob("face", two[a:b].astype(np.int64), (int(s0[a]), int(s1[a]))))

    # three or more sharers: components, then vertex promotion
    classes = defaultdict(list)
    mstart = np.concatenate([[0], np.cumsum(mcount)]).astype(np.int64)
    for i, n in enumerate(multi.tolist()):
        classes[tuple(msub[mstart[i]:mstart[i + 1]].tolist())].append(n)

    edge_comps, vertices = [], []
    for s in sorted(classes):
        for comp in _components(classes[s], nbrs):
            if len(comp) == 1:
                vertices.append((comp[0], s))
            else:
                edge_comps.append((comp, s))

    while True:
        owner = {}
        for k, (comp, _) in enumerate(edge_comps):
            for n in comp:
                owner[n] = k
        vnodes = {n for n, _ in vertices}
        promote = set()
        for k, (comp, _) in enumerate(edge_comps):
            for n in comp:
                for nb in nbrs.get(n, ()):
                    if owner.get(nb, k) == k:
                        continue
                    separated = any(w in vnodes and n in nbrs.get(w, ())
                                    for w in nbrs.get(nb, ()))
                    if not separated:
                        promote.add(n)
                        promote.add(nb)
        if not promote:
            break
        nxt = []
        for comp, s in edge_comps:
            for n in comp:
                if n in promote:
                    vertices.append((n, s))
            for piece in _components([n for n in comp if n not in promote], nbrs):
                if len(piece) == 1:
                    vertices.append((piece[0], s))
                else:
                    nxt.append((piece, s))
        edge_comps = nxt

    for comp, s in sorted(edge_comps, key=lambda cs: cs[0][0]):
        globs.append(Glob("edge", np.asarray(comp, dtype=np.int64), tuple(s)))
    for n, s in sorted(vertices, key=lambda v: v[0]):
        globs.append(Glob("vertex", np.asarray([n], dtype=np.int64), tuple(s)))
    return GlobSet(globs)
