"""The reference preconditioner's partially coupled space on the device
(solver.py:54-176): the index sets (dual_loc, primal_loc, gprimal,
gdual_pos, primal_pos, dual_offsets, wt_size), the dense transformed deluxe
weights Dbar, and the building-block operators transform / inject /
inject_t / scale, plus averaging_and_jump (solver.py:216-220).

The fused apply (engine.DevicePreconditioner) never materialises these; they
are built on first use for diagnostics and for callers of the reference's
building blocks.  Index sets follow the reference exactly (nodal B order of
each subdomain, dual = complement of the primal locals, ascending); vectors
of the partially coupled space ("wt") are laid out like the reference's:
the dual block of every subdomain in order, then the n_primal coarse dofs.

The change of basis is the one the preconditioner applies (its Q, possibly
in Householder form: same primal spans as the primal basis).
All arithmetic runs in the C-ABI kernels: bddc_pc_dbar (Q D Q^T blocks),
bddc_local_gemv (Dbar x, Q u per glob), bddc_gather_reduce (injections and
subassembly, fixed summation order).
"""

from collections.abc import Sequence

import numpy as np
import torch

from ._lib import lib, stream
from .engine import F64, _multi, dev_f64, dev_i32, dev_i64
from .plan import _excl


def _csr(keys, n):
    """(start, src): for each target t < n the positions i with keys[i] == t, ascending."""
    src = np.argsort(keys, kind="stable").astype(np.int64)
    start = np.searchsorted(keys[src], np.arange(n + 1)).astype(np.int64)
    return start, src


class _DeviceBlocks(Sequence):
    """Mutable list view of per-subdomain dense blocks held on the device:
    reading returns a host copy, assigning uploads (and refreshes the
    transposed copy the transpose operators read)."""

    def __init__(self, owner):
        self._o = owner

    def __len__(self):
        return self._o.N

    def __getitem__(self, i):
        o = self._o
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        n, a = int(o.nB[i]), int(o.soff[i])
        return o.Dbar_d[a:a + n * n].view(n, n).cpu().numpy()

    def __setitem__(self, i, M):
        o = self._o
        n, a = int(o.nB[i]), int(o.soff[i])
        M = np.asarray(M, dtype=np.float64)
        if M.shape != (n, n):
            raise ValueError(f"Dbar[{i}] must be {n} x {n}, got {M.shape}")
        o.Dbar_d[a:a + n * n] = dev_f64(M.ravel())
        o.DbarT_d[a:a + n * n] = dev_f64(M.T.ravel())


class PartiallyCoupledSpace:
    """Reference BddcPreconditioner internals for a device preconditioner."""

    def __init__(self, pc):
        ls = pc.ls
        if _multi(ls.comm):
            raise NotImplementedError("the partially coupled space is built on one rank")
        p, d, st = ls.plan, ls.d, stream()
        self.pc, self.N = pc, p.N
        N = p.N
        nB = p.nB.astype(np.int64)
        voff = np.asarray(p.voff, dtype=np.int64)
        self.nB, self.soff = nB, np.asarray(p.soff, dtype=np.int64)
        r = np.asarray(pc.r_host if hasattr(pc, "r_host") else pc._r, dtype=np.int64)
        go = _excl(r)
        # glob-major local position -> nodal local position, every subdomain
        B_nodes = np.asarray(p.B_nodes, dtype=np.int64)
        sub_of_pos = np.repeat(np.arange(N, dtype=np.int64), nB)
        order = np.lexsort((B_nodes, sub_of_pos))
        nodal = np.empty(order.size, dtype=np.int64)
        nodal[order] = np.arange(order.size, dtype=np.int64) - voff[sub_of_pos[order]]
        self._nodal = nodal
        # interface position of each nodal local B position (op.iface_index)
        iface_gm = np.asarray(p.iface_perm_host, dtype=np.int64)
        iface_nodal = np.empty_like(iface_gm)
        iface_nodal[voff[sub_of_pos] + nodal] = iface_gm
        # primal locals per subdomain in glob order (adaptive.py:248-255)
        sg_start = np.asarray(p.sub_glob_start, dtype=np.int64)
        sub_globs = np.asarray(p.sub_globs, dtype=np.int64)
        boff = np.asarray(p.sub_glob_boff, dtype=np.int64)
        self.dual_loc, self.primal_loc, self.gprimal, self.gdual_pos = [], [], [], []
        self.dual_offsets = []
        src = np.empty(int(voff[-1]), dtype=np.int64)
        tot = 0
        dual_parts = []
        for b in range(N):
            ks = sub_globs[sg_start[b]:sg_start[b + 1]]
            bo = boff[sg_start[b]:sg_start[b + 1]]
            cnt = r[ks]
            gm = np.concatenate([o + np.arange(c) for o, c in zip(bo, cnt)]) if cnt.sum() else np.zeros(0, np.int64)
            loc = nodal[voff[b] + gm]
            gids = np.concatenate([go[k] + np.arange(c) for k, c in zip(ks, cnt)]) if cnt.sum() else np.zeros(0, np.int64)
            dual = np.setdiff1d(np.arange(nB[b]), loc)
            self.primal_loc.append(loc.astype(int))
            self.gprimal.append(gids.astype(int))
            self.dual_loc.append(dual.astype(int))
            self.gdual_pos.append(iface_nodal[voff[b] + dual].astype(int))
            self.dual_offsets.append(tot)
            src[voff[b] + dual] = tot + np.arange(dual.size)
            dual_parts.append(self.gdual_pos[-1])
            tot += dual.size
        self.n_dual_total = tot
        self.n_primal = int(r.sum())
        self.wt_size = tot + self.n_primal
        self.n_hat = p.n_hat
        # primal dofs at the leading positions of their glob (solver.py:63-67)
        gpos_nodes = [ls.globs.interface_index(g.nodes) for g in ls.globs.globs]
        self.primal_pos = np.concatenate([pos[:k] for pos, k in zip(gpos_nodes, r)]).astype(int) \
            if self.n_primal else np.zeros(0, int)
        for b in range(N):
            src[voff[b] + self.primal_loc[b]] = tot + self.gprimal[b]
        # device maps: nodal-layout gather index, subassembly CSR, injections
        self.d_src = dev_i32(src)
        ws, wsrc = _csr(src, self.wt_size)
        self.d_wstart, self.d_wsrc = dev_i64(ws), dev_i64(wsrc)
        ipos = np.concatenate(dual_parts + [self.primal_pos]).astype(np.int64)
        self.d_inj_start = dev_i64(np.arange(self.wt_size + 1, dtype=np.int64))
        self.d_inj_src = dev_i64(ipos)
        ts, tsrc = _csr(ipos, self.n_hat)
        self.d_injt_start, self.d_injt_src = dev_i64(ts), dev_i64(tsrc)
        self.d_voff = dev_i64(voff)
        self.d_nB = dev_i32(nB)
        self.d_soff = dev_i64(self.soff)
        self.max_nB = int(nB.max())
        # dense Dbar (nodal order) = blockdiag(Q_g D_g Q_g^T) and its transpose
        self.Dbar_d = torch.zeros(max(int(p.S_total), 1), dtype=F64, device="cuda")
        W = torch.empty(max(p.d_total, 1), dtype=F64, device="cuda")
        lib.bddc_pc_dbar(d.slot_glob, d.slot_local, d.gsize, d.sh_boff, d.sh_doff, pc.Q_used,
                         pc.q_off_used, pc.TT, d.nB, d.soff, d.voff, dev_i32(nodal), W, self.Dbar_d,
                         int(p.sh_sub.size), st)
        del W
        self.DbarT_d = torch.empty_like(self.Dbar_d)
        lib.bddc_transpose_batched(self.Dbar_d, d.soff, d.nB, N, self.DbarT_d, st)
        self.Dbar = _DeviceBlocks(self)
        # per-glob transform (interface positions of each glob's nodes)
        gsz = p.gsize.astype(np.int64)
        gpos = np.concatenate(gpos_nodes).astype(np.int64)
        self.d_gpos = dev_i32(gpos)
        self.d_goff = dev_i64(_excl(gsz))
        self.d_gsize = dev_i32(gsz)
        gs, gsrc = _csr(gpos, self.n_hat)
        self.d_gstart, self.d_gsrc = dev_i64(gs), dev_i64(gsrc)
        self.QT = torch.empty_like(pc.Q_used)
        lib.bddc_transpose_batched(pc.Q_used, pc.q_off_used, self.d_gsize, p.G, self.QT, st)
        self.G, self.max_ng = p.G, int(gsz.max())
        self._yv = torch.empty(max(int(voff[-1]), 1), dtype=F64, device="cuda")
        self._yg = torch.empty(max(int(gsz.sum()), 1), dtype=F64, device="cuda")

    # -- operators (device tensors in, device tensors out) ---------------------
    def transform_device(self, u, transpose=False):
        """Qhat u (or Qhat^T u) on interface vectors (solver.py:142-145)."""
        out = torch.empty(self.n_hat, dtype=F64, device="cuda")
        lib.bddc_local_gemv(self.d_gsize, self.pc.q_off_used, self.d_goff, self.d_gpos,
                            self.QT if transpose else self.pc.Q_used, u, self._yg, None, None, None,
                            None, self.G, self.max_ng, 1, stream())
        lib.bddc_gather_reduce(self.d_gstart, self.d_gsrc, self._yg, out, self.n_hat, stream())
        return out

    def inject_device(self, v):
        """Rtil v (solver.py:147-153)."""
        w = torch.empty(self.wt_size, dtype=F64, device="cuda")
        lib.bddc_gather_reduce(self.d_inj_start, self.d_inj_src, v, w, self.wt_size, stream())
        return w

    def inject_t_device(self, w):
        """Rtil^T w (solver.py:155-161)."""
        v = torch.empty(self.n_hat, dtype=F64, device="cuda")
        lib.bddc_gather_reduce(self.d_injt_start, self.d_injt_src, w, v, self.n_hat, stream())
        return v

    def scale_device(self, w, transpose=False):
        """Dtil w (or Dtil^T w), subassembled over the coupled primal dofs (solver.py:163-178)."""
        out = torch.empty(self.wt_size, dtype=F64, device="cuda")
        lib.bddc_local_gemv(self.d_nB, self.d_soff, self.d_voff, self.d_src,
                            self.DbarT_d if transpose else self.Dbar_d, w, self._yv, None, None,
                            None, None, self.N, self.max_nB, 2, stream())
        lib.bddc_gather_reduce(self.d_wstart, self.d_wsrc, self._yv, out, self.wt_size, stream())
        return out


def _dev(x):
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=F64).contiguous()
    return dev_f64(np.asarray(x, dtype=np.float64))


def _host(fn, x, *a):
    out = fn(_dev(x), *a)
    return out if isinstance(x, torch.Tensor) else out.cpu().numpy()


class CoupledMixin:
    """Reference internals on BddcPreconditioner (built on first access)."""

    @property
    def coupled(self):
        if getattr(self, "_coupled", None) is None:
            self._coupled = PartiallyCoupledSpace(self)
        return self._coupled

    dual_loc = property(lambda self: self.coupled.dual_loc)
    primal_loc = property(lambda self: self.coupled.primal_loc)
    gprimal = property(lambda self: self.coupled.gprimal)
    gdual_pos = property(lambda self: self.coupled.gdual_pos)
    primal_pos = property(lambda self: self.coupled.primal_pos)
    dual_offsets = property(lambda self: self.coupled.dual_offsets)
    n_dual_total = property(lambda self: self.coupled.n_dual_total)
    wt_size = property(lambda self: self.coupled.wt_size)
    Dbar = property(lambda self: self.coupled.Dbar)

    def transform(self, u, transpose=False):
        return _host(self.coupled.transform_device, u, transpose)

    def inject(self, v):
        return _host(self.coupled.inject_device, v)

    def inject_t(self, w):
        return _host(self.coupled.inject_t_device, w)

    def scale(self, w, transpose=False):
        return _host(self.coupled.scale_device, w, transpose)


def averaging_and_jump(pc, wt):
    """(E_D wt, P_D wt) with E_D = Rtil Rtil^T Dtil (solver.py:216-220), on the device."""
    c = pc.coupled
    w = _dev(wt)
    e = c.inject_device(c.inject_t_device(c.scale_device(w)))
    jump = w - e
    if isinstance(wt, torch.Tensor):
        return e, jump
    return e.cpu().numpy(), jump.cpu().numpy()
