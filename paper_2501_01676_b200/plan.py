"""Symbolic plan: integer index maps from (system, partition, globs) to the
batched device layout.  No floating-point work.

Local numbering per subdomain (reference substructuring.py:85-96 sorts B and
I dofs by global node id; here B dofs are *glob-major*: the subdomain's globs
in glob order, each glob's nodes in glob order, so every glob is a
contiguous block and the per-glob change of basis, deluxe blocks and prior
rows are contiguous block operations).  Interior dofs: the *deep* ones first (no
element shared with an interface node, so their rows and columns have no
entries in the interface block and their elimination only touches the
interior block and the load column), then the shell; each group sorted by
node id.  ``nDeep`` (even: 16-byte aligned sub-blocks) is the number of
leading interior dofs eliminated in that restricted first phase.  Nothing
downstream depends on the ordering beyond rounding.

Two builders produce identical plans:
* ``Plan(system, partition, globs)`` — numpy on the host (reference for tests);
* ``Plan(..., device_inputs={"conn": ..., "sub_of": ...})`` — the per-element
  part (the only part that scales with the mesh: 4 x n_elements entries) runs
  as torch sort / unique / searchsorted on the GPU and stays resident there.
  The glob part (O(sum nB)) is always host numpy.

Sharding (one rank per GPU): ``owned=(s0, s1)`` restricts every
per-subdomain array (element lists, interior / interface dofs, the
subdomain -> glob incidence) to subdomains s0..s1-1, numbered locally from 0;
the per-glob tables (kinds, sizes, sharers, slot offsets ``sh_doff``) stay
global, ``slot_local`` maps each (glob, sharer) slot to its local subdomain
(-1 when another rank owns it), ``glob_mine`` marks the globs whose first
sharer is local (this rank computes their deluxe blocks and eigenproblems),
and the ``g_*`` arrays keep the global subdomain -> glob incidence that the
coarse numbering needs.  Interior dofs follow the reference's definition
(free and not an interface node, substructuring.py:88-91), which needs no
cross-rank node counts.
"""

import numpy as np

KIND = {"face": 0, "edge": 1, "vertex": 2}
NATIVE_GLOB_TABLES = True  # glob tables from the library's host routine (numpy path: reference)


def _ranges(starts, counts):
    """Concatenated aranges: [s0, s0+c0) ++ [s1, s1+c1) ++ ..."""
    counts = np.asarray(counts, dtype=np.int64)
    total = int(counts.sum())
    if total == 0:
        return np.zeros(0, dtype=np.int64)
    rep = np.repeat(np.asarray(starts, dtype=np.int64) - np.concatenate([[0], np.cumsum(counts)[:-1]]), counts)
    return rep + np.arange(total, dtype=np.int64)


def _up(a, dv):
    """Host array -> device, asynchronously through pinned staging."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    if t.numel() == 0:
        return torch.empty(t.shape, dtype=t.dtype, device=dv)
    return t.pin_memory().to(dv, non_blocking=True)


def _excl(a):
    a = np.asarray(a, dtype=np.int64)
    out = np.zeros(a.size + 1, dtype=np.int64)
    np.cumsum(a, out=out[1:])
    return out


class Plan:
    def __init__(self, system, partition, globs, device_inputs=None, owned=None):
        N_glob = int(partition.n_subdomains)
        s0, s1 = (0, N_glob) if owned is None else (int(owned[0]), int(owned[1]))
        if not 0 <= s0 <= s1 <= N_glob:
            raise ValueError(f"owned range {owned} outside 0..{N_glob}")
        self.N_glob = N_glob
        self.owned = (s0, s1)
        self.N = N_glob  # the glob part works on global subdomain ids first
        self.n_nodes = system.mesh.n_nodes
        self.n_hat = int(np.asarray(globs.interface_nodes).size)
        self.on_device = device_inputs is not None
        self._iface_nodes = np.asarray(globs.interface_nodes, dtype=np.int64)
        if self.on_device:
            # the sorts of the element part are queued first and run while the
            # host builds the glob part
            self._element_pre_torch(system, device_inputs, s1 - s0)
        self._glob_part(globs)
        self._restrict(s0, s1)
        if self.on_device:
            self._interface_maps_torch(device_inputs["conn"].device)
            self._element_post_torch(device_inputs)
        else:
            self._interface_maps_numpy()
            self._element_part_numpy(system, partition)
        self._layout()

    # -- globs: sharers, glob-major B order, interface maps (host) ----------
    def _glob_part(self, globs):
        N = self.N
        if hasattr(globs, "flat"):
            f = globs.flat()
        else:  # a reference GlobSet
            from .decomposition import flatten_globs
            f = flatten_globs(globs.globs)
        G = f["kind"].size
        self.G = G
        self.kind = f["kind"]
        self.gsize = f["size"]
        nsh = f["nsh"]
        if NATIVE_GLOB_TABLES and self._glob_part_native(f, N):
            return
        self.sh_start = _excl(nsh).astype(np.int32)
        self.sh_sub = f["sharers"].astype(np.int32)
        slot_glob = np.repeat(np.arange(G, dtype=np.int64), nsh)
        self.slot_glob = slot_glob.astype(np.int32)
        self.sh_doff = _excl(self.gsize[slot_glob].astype(np.int64) ** 2)
        self.d_total = int(self.sh_doff[-1])
        self.sh_doff = self.sh_doff[:-1]
        # slots by (sharer, glob): one stable argsort of a combined key (unique pairs)
        # (the slots are glob-major already, so a stable sort by sharer orders them by
        # (sharer, glob); 16-bit keys take numpy's radix sort)
        if N <= 0xffff:
            order = np.argsort(self.sh_sub.astype(np.uint16), kind="stable")
        else:
            order = np.argsort(self.sh_sub.astype(np.int64) * max(G, 1) + slot_glob, kind="stable")
        self.sub_globs = slot_glob[order].astype(np.int32)
        pair_sub = self.sh_sub[order].astype(np.int64)
        self.sub_glob_sh = order.astype(np.int32)
        self.sub_glob_start = np.searchsorted(pair_sub, np.arange(N + 1)).astype(np.int32)
        sizes_k = self.gsize[self.sub_globs].astype(np.int64)
        cs = _excl(sizes_k)
        if sizes_k.size:
            owner = np.repeat(np.arange(N), np.diff(self.sub_glob_start))
            boff = cs[:-1] - cs[self.sub_glob_start[:-1]][owner]
        else:
            boff = np.zeros(0, np.int64)
        self.sub_glob_boff = boff.astype(np.int32)
        self.sh_boff = np.empty(order.size, dtype=np.int32)
        self.sh_boff[order] = self.sub_glob_boff
        self.nB = np.bincount(pair_sub, weights=sizes_k, minlength=N).astype(np.int64)
        self.voff = _excl(self.nB)
        gnodes = f["nodes"]
        self._gnodes = gnodes
        gstart = _excl(self.gsize)
        # B nodes (glob-major interface nodes of every subdomain) = concatenated
        # ranges of gnodes; built on the device for the device plan, on the host
        # only when a host consumer asks (B_nodes property)
        self._B_starts = gstart[self.sub_globs].astype(np.int64)
        self._B_counts = sizes_k
        self._B_range = (0, int(sizes_k.sum()))
        self._B_nodes = None
        self._pos2k = None  # per local interface position: its (subdomain, glob) pair; lazy

    def _glob_part_native(self, f, N):
        """The same tables from the library's host routine (csrc/plan_host.cu:
        plain loops, ~0.2 ms instead of ~3 ms of numpy array passes at cfg5).
        Returns False when the library is not built (the numpy path runs)."""
        import ctypes

        try:
            from ._lib import lib
            lib.load()
        except (RuntimeError, OSError):
            return False
        G = self.G
        gsize = np.ascontiguousarray(self.gsize, dtype=np.int32)
        nsh = np.ascontiguousarray(f["nsh"], dtype=np.int64)
        sharers = np.ascontiguousarray(f["sharers"], dtype=np.int64)
        ns = int(sharers.size)
        out = dict(sh_start=np.empty(G + 1, np.int32), slot_glob=np.empty(ns, np.int32),
                   sh_doff=np.empty(ns + 1, np.int64), sub_globs=np.empty(ns, np.int32),
                   sub_glob_sh=np.empty(ns, np.int32), sub_glob_start=np.empty(N + 1, np.int32),
                   sub_glob_boff=np.empty(ns, np.int32), sh_boff=np.empty(ns, np.int32),
                   nB=np.empty(N, np.int64), b_starts=np.empty(ns, np.int64))
        ptr = lambda a: ctypes.c_void_p(a.ctypes.data)
        rc = lib.bddc_plan_glob_tables(G, N, ptr(gsize), ptr(nsh), ptr(sharers),
                                       *[ptr(out[k]) for k in ("sh_start", "slot_glob", "sh_doff",
                                                               "sub_globs", "sub_glob_sh",
                                                               "sub_glob_start", "sub_glob_boff",
                                                               "sh_boff", "nB", "b_starts")])
        if rc:
            raise ValueError(f"glob sharer lists are inconsistent with {N} subdomains ({rc})")
        self.gsize = gsize
        self.sh_start, self.slot_glob = out["sh_start"], out["slot_glob"]
        self.sh_sub = sharers.astype(np.int32)
        self.d_total = int(out["sh_doff"][-1])
        self.sh_doff = out["sh_doff"][:-1]
        self.sub_globs, self.sub_glob_sh = out["sub_globs"], out["sub_glob_sh"]
        self.sub_glob_start, self.sub_glob_boff = out["sub_glob_start"], out["sub_glob_boff"]
        self.sh_boff, self.nB = out["sh_boff"], out["nB"]
        self.voff = _excl(self.nB)
        self._gnodes = f["nodes"]
        self._B_starts = out["b_starts"]
        self._B_counts = self.gsize[self.sub_globs].astype(np.int64)
        self._B_range = (0, int(self.voff[-1]))
        self._B_nodes = None
        self._pos2k = None
        return True

    def _restrict(self, s0, s1):
        """Keep subdomains s0..s1-1 (local ids 0..s1-s0-1)."""
        self.g_sub_globs = self.sub_globs
        self.g_sub_glob_start = self.sub_glob_start
        self.g_sub_glob_boff = self.sub_glob_boff
        self.g_nB = self.nB
        sh = self.sh_sub.astype(np.int64)
        self.slot_local = np.where((sh >= s0) & (sh < s1), sh - s0, -1).astype(np.int32)
        first = self.sh_sub[self.sh_start[:-1]] if self.G else np.zeros(0, np.int32)
        self.glob_mine = (first >= s0) & (first < s1)
        self.N = s1 - s0
        if (s0, s1) == (0, self.N_glob):
            return
        a, b = int(self.sub_glob_start[s0]), int(self.sub_glob_start[s1])
        self.sub_globs = self.sub_globs[a:b]
        self.sub_glob_sh = self.sub_glob_sh[a:b]
        self.sub_glob_boff = self.sub_glob_boff[a:b]
        self.sub_glob_start = (self.sub_glob_start[s0:s1 + 1] - a).astype(np.int32)
        self.nB = self.g_nB[s0:s1]
        v0, v1 = int(self.voff[s0]), int(self.voff[s1])
        self.voff = self.voff[s0:s1 + 1] - v0
        self._B_range = (v0, v1)

    @property
    def pos2k(self):
        """Index into sub_globs of every local interface position (host copy)."""
        if self._pos2k is None:
            sizes = self.gsize[self.sub_globs].astype(np.int64)
            self._pos2k = np.repeat(np.arange(self.sub_globs.size, dtype=np.int32), sizes)
        return self._pos2k

    def pos2k_device(self, dv):
        import torch

        sizes = _up(self.gsize[self.sub_globs].astype(np.int64), dv)
        return torch.repeat_interleave(torch.arange(self.sub_globs.size, dtype=torch.int32, device=dv),
                                       sizes, output_size=int(self.voff[-1]))

    @property
    def B_nodes(self):
        if self._B_nodes is None:
            v0, v1 = self._B_range
            self._B_nodes = self._gnodes[_ranges(self._B_starts, self._B_counts)][v0:v1]
        return self._B_nodes

    def _interface_maps_numpy(self):
        self.iface_perm = np.searchsorted(self._iface_nodes, self.B_nodes).astype(np.int32)
        src = np.argsort(self.iface_perm, kind="stable")
        self.tsrc = src.astype(np.int64)
        self.tstart = np.searchsorted(self.iface_perm[src], np.arange(self.n_hat + 1)).astype(np.int64)

    def _interface_maps_torch(self, dv):
        import torch

        self._node_maps_device(dv)
        total = int(self._B_counts.sum())
        counts = _up(self._B_counts, dv)
        base = _up(self._B_starts, dv) - (torch.cumsum(counts, 0) - counts)
        idx = torch.repeat_interleave(base, counts, output_size=total)
        idx += torch.arange(total, device=dv)
        v0, v1 = self._B_range
        Bn = self._gn_d[idx[v0:v1]]
        ifn = self._iface_nodes_d
        perm = torch.searchsorted(ifn, Bn)
        self.iface_perm_d = perm.to(torch.int32)
        srt = torch.sort(perm, stable=True)
        self.tsrc_d = srt.indices
        self.tstart_d = torch.searchsorted(srt.values, torch.arange(self.n_hat + 1, device=dv))
        self._B_nodes_d = Bn

    @property
    def iface_perm_host(self):
        return self.iface_perm_d.cpu().numpy() if self.on_device else self.iface_perm

    # -- elements: interior dofs, element lists, element-local indices ------
    def _element_part_numpy(self, system, partition):
        N, n_nodes = self.N, self.n_nodes
        s0, s1 = self.owned
        sub_all = np.asarray(partition.subdomain_of, dtype=np.int64)
        mine = np.flatnonzero((sub_all >= s0) & (sub_all < s1))
        sub_of = sub_all[mine] - s0
        el = np.asarray(system.mesh.elements, dtype=np.int64)[mine]
        key = np.unique((el * max(N, 1) + sub_of[:, None]).ravel())
        node, sub = key // max(N, 1), key % max(N, 1)
        free = np.asarray(system.node_to_free) >= 0
        on_iface = np.zeros(n_nodes, dtype=bool)
        on_iface[self._iface_nodes] = True
        interior = free[node] & ~on_iface[node]
        I_sub, I_node = sub[interior], node[interior]
        # deep interior nodes (no element shared with an interface node) first
        shell = np.zeros(n_nodes, dtype=bool)
        shell[el[on_iface[el].any(axis=1)].ravel()] = True
        o = np.lexsort((I_node, shell[I_node], I_sub))
        self.I_nodes = I_node[o]
        self.nI = np.bincount(I_sub, minlength=N).astype(np.int64)
        self.ioff = _excl(self.nI)
        self.nDeep = np.bincount(I_sub[~shell[I_node]], minlength=N).astype(np.int64) & ~np.int64(1)
        eorder = np.argsort(sub_of, kind="stable")
        self.elem_ids = mine[eorder].astype(np.int64)
        self.elem_start = _excl(np.bincount(sub_of, minlength=N))
        # loc4 is indexed like the element inputs (element id), not by sorted position
        self.loc4 = np.full((sub_all.size, 4), 2 ** 30, dtype=np.int32)
        self.loc4[mine] = self._local_index_numpy(el, sub_of)

    def _local_index_numpy(self, conn, sub):
        N, n_nodes = self.N, self.n_nodes
        Bsub = np.repeat(np.arange(N, dtype=np.int64), self.nB)
        Bloc = np.arange(self.B_nodes.size, dtype=np.int64) - self.voff[Bsub] + self.nI[Bsub]
        Isub = np.repeat(np.arange(N, dtype=np.int64), self.nI)
        Iloc = np.arange(self.I_nodes.size, dtype=np.int64) - self.ioff[Isub]
        keys = np.concatenate([Bsub * n_nodes + self.B_nodes, Isub * n_nodes + self.I_nodes])
        vals = np.concatenate([Bloc, Iloc])
        ko = np.argsort(keys)
        keys, vals = keys[ko], vals[ko]
        q = sub[:, None] * n_nodes + conn
        pos = np.minimum(np.searchsorted(keys, q), keys.size - 1)
        found = keys[pos] == q
        return np.where(found, vals[pos], np.int64(2 ** 30)).astype(np.int32)

    def _element_pre_torch(self, system, dev, N):
        """Device work of the element part that needs no glob table: interior
        dofs (deep first), their counts, the element order.  No host sync."""
        import torch

        n_nodes = self.n_nodes
        s0 = self.owned[0]
        conn = dev["conn"]                 # (E_local, 4) int64 on the GPU, input order
        sub_g = dev["sub_of"]              # (E_local,) global subdomain ids
        dv = conn.device
        sub_of = sub_g - s0
        free = dev.get("free")
        if free is None:
            free = _up(np.asarray(system.node_to_free) >= 0, dv)
        self._iface_nodes_d = _up(self._iface_nodes, dv)
        # interior nodes: free, not on the interface, touched by a (single) local
        # subdomain -- its owner, read off any element containing it
        owner = torch.full((n_nodes,), -1, dtype=torch.int64, device=dv)
        owner[conn.reshape(-1)] = sub_of[:, None].expand(-1, 4).reshape(-1)
        on_iface = torch.zeros(n_nodes, dtype=torch.bool, device=dv)
        on_iface[self._iface_nodes_d] = True
        interior = free & ~on_iface & (owner >= 0)
        # deep interior nodes (no element shared with an interface node) first
        # (integer scatter-add of the per-element flag: order-independent)
        touch = on_iface[conn].any(dim=1).to(torch.int32)
        shell = torch.zeros(n_nodes, dtype=torch.int32, device=dv)
        shell.index_add_(0, conn.reshape(-1), touch[:, None].expand(-1, 4).reshape(-1))
        # Nothing here synchronises with the host (no nonzero / bincount / mask
        # indexing): every node gets the key 2 * owner + shell, non-interior nodes a
        # sentinel that sorts last; one stable sort orders the interior nodes by
        # (subdomain, shell, node id) and the counts come from an integer scatter-add.
        # The interior prefix is cut off once the counts are on the host.
        key = torch.where(interior, owner * 2 + (shell > 0), torch.full_like(owner, 2 * N))
        self._node_order_d = torch.sort(key, stable=True).indices
        self._owner_d = owner
        one = torch.ones((), dtype=torch.int64, device=dv)
        self._cnt_d = torch.zeros(2 * N + 1, dtype=torch.int64, device=dv).index_add_(
            0, key, one.expand(n_nodes))
        self.elem_ids_d = torch.sort(sub_of, stable=True).indices
        self._ecnt_d = torch.zeros(N, dtype=torch.int64, device=dv).index_add_(
            0, sub_of, one.expand(sub_of.numel()))

    def _element_post_torch(self, dev):
        import torch

        from ._lib import lib, stream

        N, n_nodes = self.N, self.n_nodes
        conn, dv = dev["conn"], dev["conn"].device
        cnt_h = self._cnt_d[:2 * N].view(N, 2).cpu().numpy().astype(np.int64)  # the one sync
        self.nI = cnt_h.sum(axis=1)
        self.nDeep = cnt_h[:, 0] & ~np.int64(1)
        self.ioff = _excl(self.nI)
        self.elem_start = _excl(self._ecnt_d.cpu().numpy())
        I_node = self._node_order_d[:int(self.nI.sum())]
        I_sub = self._owner_d[I_node]
        self.I_nodes_d = I_node
        iloc = torch.full((n_nodes,), -1, dtype=torch.int32, device=dv)
        iloc[I_node] = (torch.arange(I_node.numel(), device=dv) - _up(self.ioff, dv)[I_sub]).to(torch.int32)
        self.loc4_d = torch.empty((conn.shape[0], 4), dtype=torch.int32, device=dv)
        lib.bddc_plan_loc4(conn, dev["sub_of"], conn.shape[0], self.owned[0], iloc,
                           self._glob_of_node_d, self._pos_in_glob_d, _up(self.sh_start, dv),
                           _up(self.sh_sub, dv), _up(self.sh_boff, dv),
                           _up(self.nI, dv), self.loc4_d, stream())
        del self._cnt_d, self._ecnt_d, self._node_order_d, self._owner_d

    def _node_maps_device(self, dv):
        """node -> glob index and position in the glob (-1 off the interface),
        scattered on the device from the glob-ordered interface nodes."""
        import torch

        gn = _up(self._gnodes.astype(np.int64), dv)
        self._gn_d = gn
        gsz = _up(self.gsize.astype(np.int64), dv)
        gid = torch.repeat_interleave(torch.arange(self.G, device=dv), gsz,
                                      output_size=int(self._gnodes.size))
        gst = torch.cumsum(gsz, 0) - gsz
        gof = torch.full((self.n_nodes,), -1, dtype=torch.int32, device=dv)
        pos = torch.zeros(self.n_nodes, dtype=torch.int32, device=dv)
        gof[gn] = gid.to(torch.int32)
        pos[gn] = (torch.arange(gn.numel(), device=dv) - gst[gid]).to(torch.int32)
        self._glob_of_node_d = gof
        self._pos_in_glob_d = pos

    def _layout(self):
        self.nL = self.nI + self.nB
        self.max_elems = int(np.diff(self.elem_start).max()) if self.N else 0
        self.ld = (self.nL + 2) // 2 * 2  # >= nL + 1, even
        self.off = _excl(self.nL * self.ld)
        self.K_total = int(self.off[-1])
        self.off = self.off[:-1]
        self.soff = _excl(self.nB * self.nB)
        self.S_total = int(self.soff[-1])
        self.soff = self.soff[:-1]

    # -- host views of the element part -----------------------------------
    @property
    def I_nodes_host(self):
        return self.I_nodes_d.cpu().numpy() if self.on_device else self.I_nodes

    def check(self):
        """Reference errors of build_subdomain_operator (substructuring.py:93-96)."""
        bad_e = np.flatnonzero(np.diff(self.elem_start) == 0)
        bad_b = np.flatnonzero(self.nB == 0)
        bad_i = np.flatnonzero(self.nI == 0)
        s0 = self.owned[0]
        for i in sorted(set(bad_e.tolist()) | set(bad_b.tolist()) | set(bad_i.tolist())):
            if i in bad_e:
                raise ValueError(f"subdomain {i + s0} has no elements")
            if i in bad_b:
                raise ValueError(f"subdomain {i + s0} has no interface unknowns")
            raise ValueError(f"subdomain {i + s0} has no interior unknowns")

    def nodal_order(self, sub):
        """Permutation p with B_glob_major[p] = sorted interface nodes of sub."""
        nodes = self.B_nodes[self.voff[sub]:self.voff[sub + 1]]
        return np.argsort(nodes, kind="stable")
