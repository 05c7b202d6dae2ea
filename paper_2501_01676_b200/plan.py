"""Host symbolic plan: index maps from (system, partition, globs) to the
batched device layout.  Integer work only; the numbers are all on the GPU.

Local numbering per subdomain (reference substructuring.py:85-96 sorts B and
I dofs by global node id; here B dofs are *glob-major*: the subdomain's globs
in glob order, each glob's nodes in glob order, so every glob is a
contiguous block and the per-glob change of basis, deluxe blocks and prior
rows are contiguous block operations).  Interior dofs stay sorted by node
id.  Nothing downstream depends on the ordering beyond rounding.
"""

import numpy as np

KIND = {"face": 0, "edge": 1, "vertex": 2}


def _ranges(starts, counts):
    """Concatenated aranges: [s0, s0+c0) ++ [s1, s1+c1) ++ ..."""
    counts = np.asarray(counts, dtype=np.int64)
    total = int(counts.sum())
    if total == 0:
        return np.zeros(0, dtype=np.int64)
    rep = np.repeat(np.asarray(starts, dtype=np.int64) - np.concatenate([[0], np.cumsum(counts)[:-1]]), counts)
    return rep + np.arange(total, dtype=np.int64)


def _excl(a):
    a = np.asarray(a, dtype=np.int64)
    out = np.zeros(a.size + 1, dtype=np.int64)
    np.cumsum(a, out=out[1:])
    return out


class Plan:
    def __init__(self, system, partition, globs):
        mesh = system.mesh
        N = int(partition.n_subdomains)
        sub_of = np.asarray(partition.subdomain_of, dtype=np.int64)
        el = np.asarray(mesh.elements, dtype=np.int64)
        n_nodes = mesh.n_nodes
        self.N = N
        self.n_hat = int(globs.interface_nodes.size)
        gl = globs.globs
        G = len(gl)
        self.G = G
        self.kind = np.array([KIND[g.kind] for g in gl], dtype=np.int32)
        self.gsize = np.array([g.size for g in gl], dtype=np.int32)
        nsh = np.array([len(g.sharers) for g in gl], dtype=np.int64)
        self.sh_start = _excl(nsh).astype(np.int32)
        self.sh_sub = (np.concatenate([np.asarray(g.sharers, dtype=np.int64) for g in gl])
                       if G else np.zeros(0, np.int64)).astype(np.int32)
        slot_glob = np.repeat(np.arange(G, dtype=np.int64), nsh)
        self.slot_glob = slot_glob.astype(np.int32)
        # D blocks per (glob, sharer) slot
        self.sh_doff = _excl(self.gsize[slot_glob].astype(np.int64) ** 2)
        self.d_total = int(self.sh_doff[-1])
        self.sh_doff = self.sh_doff[:-1]

        # per-subdomain glob lists in glob order
        order = np.lexsort((slot_glob, self.sh_sub.astype(np.int64)))
        self.sub_globs = slot_glob[order].astype(np.int32)
        pair_sub = self.sh_sub[order].astype(np.int64)
        self.sub_glob_sh = order.astype(np.int32)
        self.sub_glob_start = np.searchsorted(pair_sub, np.arange(N + 1)).astype(np.int32)
        sizes_k = self.gsize[self.sub_globs].astype(np.int64)
        cs = _excl(sizes_k)
        boff = cs[:-1] - cs[self.sub_glob_start[:-1]][np.repeat(np.arange(N), np.diff(self.sub_glob_start))] \
            if sizes_k.size else np.zeros(0, np.int64)
        self.sub_glob_boff = boff.astype(np.int32)
        self.sh_boff = np.empty(order.size, dtype=np.int32)
        self.sh_boff[order] = self.sub_glob_boff
        self.nB = np.bincount(pair_sub, weights=sizes_k, minlength=N).astype(np.int64)
        self.voff = _excl(self.nB)

        # glob-major B nodes and global interface positions
        gnodes = np.concatenate([g.nodes for g in gl]).astype(np.int64) if G else np.zeros(0, np.int64)
        gstart = _excl(self.gsize)
        idx = _ranges(gstart[self.sub_globs], sizes_k)
        self.B_nodes = gnodes[idx]
        self.iface_perm = np.searchsorted(globs.interface_nodes, self.B_nodes).astype(np.int32)
        self.pos2k = np.repeat(np.arange(self.sub_globs.size, dtype=np.int32), sizes_k)

        # interior nodes: free nodes touched by exactly one subdomain
        key = np.unique((el * N + sub_of[:, None]).ravel())
        node, sub = key // N, key % N
        cnt = np.bincount(node, minlength=n_nodes)
        free = np.asarray(system.node_to_free) >= 0
        interior = (cnt[node] == 1) & free[node]
        I_sub, I_node = sub[interior], node[interior]
        o = np.lexsort((I_node, I_sub))
        self.I_nodes = I_node[o]
        self.nI = np.bincount(I_sub, minlength=N).astype(np.int64)
        self.ioff = _excl(self.nI)
        self.nL = self.nI + self.nB

        # element lists and local indices of their nodes
        eorder = np.argsort(sub_of, kind="stable")
        self.elem_ids = eorder.astype(np.int64)
        self.elem_start = _excl(np.bincount(sub_of, minlength=N))
        self.max_elems = int(np.diff(self.elem_start).max()) if N else 0
        Bsub = np.repeat(np.arange(N, dtype=np.int64), self.nB)
        Bloc = np.arange(self.B_nodes.size, dtype=np.int64) - self.voff[Bsub] + self.nI[Bsub]
        Isub = np.repeat(np.arange(N, dtype=np.int64), self.nI)
        Iloc = np.arange(self.I_nodes.size, dtype=np.int64) - self.ioff[Isub]
        keys = np.concatenate([Bsub * n_nodes + self.B_nodes, Isub * n_nodes + self.I_nodes])
        vals = np.concatenate([Bloc, Iloc])
        ko = np.argsort(keys)
        keys, vals = keys[ko], vals[ko]
        q = sub_of[eorder][:, None] * n_nodes + el[eorder]
        pos = np.searchsorted(keys, q)
        pos = np.minimum(pos, keys.size - 1)
        found = keys[pos] == q
        big = np.int64(2 ** 30)
        self.loc4 = np.where(found, vals[pos], big).astype(np.int32)

        # local matrix layout [I|B] x [I|B|f]
        self.ld = (self.nL + 2) // 2 * 2  # >= nL + 1, even
        self.off = _excl(self.nL * self.ld)
        self.K_total = int(self.off[-1])
        self.off = self.off[:-1]
        self.soff = _excl(self.nB * self.nB)
        self.S_total = int(self.soff[-1])
        self.soff = self.soff[:-1]

        # interface CSR (gather-reduce of local vectors)
        src = np.argsort(self.iface_perm, kind="stable")
        self.tsrc = src.astype(np.int64)
        self.tstart = np.searchsorted(self.iface_perm[src], np.arange(self.n_hat + 1)).astype(np.int64)

    def check(self):
        """Reference errors of build_subdomain_operator (substructuring.py:93-96)."""
        for i in range(self.N):
            if self.elem_start[i + 1] == self.elem_start[i]:
                raise ValueError(f"subdomain {i} has no elements")
            if self.nB[i] == 0:
                raise ValueError(f"subdomain {i} has no interface unknowns")
            if self.nI[i] == 0:
                raise ValueError(f"subdomain {i} has no interior unknowns")

    def glob_positions(self, sub, g):
        """Glob-major local block (start, size) of glob g in subdomain sub."""
        k0, k1 = self.sub_glob_start[sub], self.sub_glob_start[sub + 1]
        ks = np.flatnonzero(self.sub_globs[k0:k1] == g)
        if ks.size == 0:
            return None
        return int(self.sub_glob_boff[k0 + ks[0]]), int(self.gsize[g])

    def nodal_order(self, sub):
        """Permutation p with B_glob_major[p] = sorted interface nodes of sub."""
        nodes = self.B_nodes[self.voff[sub]:self.voff[sub + 1]]
        return np.argsort(nodes, kind="stable")
