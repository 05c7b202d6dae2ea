"""Subdomain sharding over ranks (one process per GPU).

The reference solves every subdomain in one process; its data
parallelism is the loop over subdomains.  Here rank r owns the contiguous
subdomain block ``block_range(N, R, r)`` (x-slabs for the regular
partitions) and everything per subdomain (assembly, Schur elimination,
Bsym^-1, local preconditioner operators, interior recovery) runs only there.
The data plane is the one north_star names:

* interface vectors are distributed (``InterfaceLayout``): each rank holds the
  interface dofs its subdomains touch, owned dofs first (the owner of a dof
  is the rank of the first sharer of its glob), then ghosts; subassembled
  sums (S_hat u, M^-1 r, g_hat) are completed by a **neighbour halo
  exchange**: ghosts' partial sums go to the owner, the owner adds them in
  rank order and sends the totals back (two point-to-point rounds);
* GMRES dot products and norms run over the owned entries, followed by one
  **allreduce** of the m partial dots;
* the coarse right-hand side is **reduced to rank 0**, which holds the only
  coarse factorisation (the subdomain contributions C_i are reduced to it
  once in setup), solves, and **broadcasts** the coarse solution;
* in setup, only the blocks of globs whose sharers live on different ranks
  move (``SlotExchange``): Bsym / Bsym^-1 / prior blocks to the rank that
  owns the glob eigenproblem, deluxe blocks and changes of basis back to the
  sharers' ranks; the small per-glob results (counts, eigenvalues) and the
  final nodal solution are allreduced once.

``TorchComm`` wraps ``torch.distributed`` (NCCL for CUDA tensors; with gloo
the CUDA tensors are staged through host memory); ``LoopbackComm`` runs R
ranks as threads of one process (tests on one GPU: every exchange is a
host-side rendezvous after a stream synchronize, no kernel ever waits on
another rank's kernel).
"""

import threading

import numpy as np


def block_range(n, size, rank):
    """Contiguous balanced split of range(n): [s0, s1) of `rank`."""
    q, r = divmod(int(n), int(size))
    s0 = rank * q + min(rank, r)
    return s0, s0 + q + (1 if rank < r else 0)


def rank_of_subdomain(n, size):
    """Owner rank of every subdomain under block_range."""
    out = np.empty(int(n), dtype=np.int64)
    for r in range(size):
        a, b = block_range(n, size, r)
        out[a:b] = r
    return out


class Comm:
    """Single-rank communicator (every collective is the identity)."""

    rank = 0
    size = 1

    def allreduce_(self, t):
        """In-place elementwise sum over ranks; returns t."""
        return t

    def reduce_(self, t, root=0):
        """In-place sum onto `root` (other ranks' t is left unspecified)."""
        return t

    def broadcast_(self, t, root=0):
        return t

    def exchange(self, sends, recvs):
        """Point-to-point: sends {dst: tensor}, recvs {src: tensor} (filled)."""
        if sends or recvs:
            raise ValueError("single-rank communicator has no peers")

    def barrier(self):
        pass

    def owned(self, n):
        return block_range(n, self.size, self.rank)


class TorchComm(Comm):
    """torch.distributed process group (nccl for CUDA tensors, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def _staged(self, t):
        """gloo with a CUDA tensor: work on a host copy."""
        return (t.cpu(), True) if (t.is_cuda and not self.nccl) else (t, False)

    def allreduce_(self, t):
        if self.size > 1 and t.numel():
            x, staged = self._staged(t)
            self.dist.all_reduce(x, group=self.group)
            if staged:
                t.copy_(x)
        return t

    def reduce_(self, t, root=0):
        if self.size > 1 and t.numel():
            x, staged = self._staged(t)
            self.dist.reduce(x, dst=root, group=self.group)
            if staged and self.rank == root:
                t.copy_(x)
        return t

    def broadcast_(self, t, root=0):
        if self.size > 1 and t.numel():
            x, staged = self._staged(t)
            self.dist.broadcast(x, src=root, group=self.group)
            if staged:
                t.copy_(x)
        return t

    def exchange(self, sends, recvs):
        if self.size == 1 or not (sends or recvs):
            return
        d = self.dist
        ops, back = [], []
        for dst in sorted(sends):
            x, _ = self._staged(sends[dst].contiguous())
            ops.append(d.P2POp(d.isend, x, dst, group=self.group))
        for src in sorted(recvs):
            x, staged = self._staged(recvs[src])
            ops.append(d.P2POp(d.irecv, x, src, group=self.group))
            if staged:
                back.append((recvs[src], x))
        for w in d.batch_isend_irecv(ops):
            w.wait()
        for t, x in back:
            t.copy_(x)

    def barrier(self):
        if self.size > 1:
            self.dist.barrier(group=self.group)


class _LoopbackHub:
    def __init__(self, size):
        self.size = size
        self.bar = threading.Barrier(size)
        self.slots = [None] * size
        self.mail = {}
        self.result = None


class LoopbackComm(Comm):
    """Rank `rank` of `size` threads sharing one process and one GPU."""

    def __init__(self, hub, rank):
        self.hub, self.rank, self.size = hub, rank, hub.size

    @staticmethod
    def group(size):
        hub = _LoopbackHub(size)
        return [LoopbackComm(hub, r) for r in range(size)]

    @staticmethod
    def _sync(t):
        if t.is_cuda:
            import torch

            torch.cuda.current_stream().synchronize()

    def _combine(self, t, root):
        """Sum of every rank's t computed by rank 0 (rank order); returned to
        every rank (root None) or only to `root`."""
        if self.size == 1:
            return t
        self._sync(t)
        h = self.hub
        h.slots[self.rank] = t
        h.bar.wait()
        if self.rank == 0:
            acc = h.slots[0].clone()
            for x in h.slots[1:]:
                acc += x.to(acc.device)
            self._sync(acc)
            h.result = acc
        h.bar.wait()
        if root is None or self.rank == root:
            t.copy_(h.result.to(t.device))
            self._sync(t)
        h.bar.wait()
        return t

    def allreduce_(self, t):
        return self._combine(t, None)

    def reduce_(self, t, root=0):
        return self._combine(t, root)

    def broadcast_(self, t, root=0):
        if self.size == 1:
            return t
        self._sync(t)
        h = self.hub
        if self.rank == root:
            h.result = t.clone()
            self._sync(h.result)
        h.bar.wait()
        if self.rank != root:
            t.copy_(h.result.to(t.device))
            self._sync(t)
        h.bar.wait()
        return t

    def exchange(self, sends, recvs):
        if self.size == 1:
            return
        h = self.hub
        for dst, t in sends.items():
            c = t.clone()
            self._sync(c)
            h.mail[(self.rank, dst)] = c
        h.bar.wait()
        for src, t in recvs.items():
            t.copy_(h.mail[(src, self.rank)].to(t.device))
            self._sync(t)
        h.bar.wait()
        for dst in sends:
            h.mail.pop((self.rank, dst), None)
        h.bar.wait()

    def barrier(self):
        if self.size > 1:
            self.hub.bar.wait()


def run_threads(size, fn):
    """fn(comm) on `size` loopback ranks; returns the per-rank results
    (re-raises the first exception)."""
    comms = LoopbackComm.group(size)
    out = [None] * size
    err = [None] * size

    def body(r):
        try:
            out[r] = fn(comms[r])
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e
            comms[r].hub.bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return out


def allreduce_np(comm, a):
    """Sum of a host numpy array over ranks (via a CPU / CUDA tensor)."""
    if comm is None or comm.size == 1:
        return a
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    if isinstance(comm, TorchComm) and comm.nccl:
        t = t.cuda()
    comm.allreduce_(t)
    return t.cpu().numpy()


# ---------------------------------------------------------------------------
# distributed interface layout and the setup-phase slot exchange
# ---------------------------------------------------------------------------

def interface_owner_rank(plan, size):
    """Owner rank of every global interface dof: the rank of the first sharer
    of the dof's glob (glob sharers are sorted, so it is the lowest rank
    touching the dof)."""
    rank_of = rank_of_subdomain(plan.N_glob, size)
    gnodes = np.asarray(plan._gnodes, dtype=np.int64)
    q_of = np.searchsorted(plan._iface_nodes, gnodes)
    glob_of_node = np.repeat(np.arange(plan.G, dtype=np.int64), plan.gsize.astype(np.int64))
    first = plan.sh_sub[plan.sh_start[:-1]].astype(np.int64)
    owner = np.empty(plan.n_hat, dtype=np.int64)
    owner[q_of] = rank_of[first[glob_of_node]]
    # ranks touching each dof: through its glob's sharers (for the halo lists)
    return owner, q_of, glob_of_node, rank_of


class InterfaceLayout:
    """Rank-local numbering of the interface dofs a rank's subdomains touch:
    [owned (ascending global id) | ghosts (ascending global id)], plus the
    halo lists.  Built from the replicated glob tables only (no
    communication).  Single rank: the identity layout."""

    def __init__(self, plan, comm):
        self.comm = comm
        size = comm.size if comm is not None else 1
        rank = comm.rank if comm is not None else 0
        self.multi = size > 1
        n_hat = plan.n_hat
        self.n_hat = n_hat
        self._dev = None
        if not self.multi:  # identity layout: nothing to build (no device read of the plan)
            self.n_loc = self.n_own = n_hat
            self.glob_ids = np.arange(n_hat, dtype=np.int64)
            self.perm_loc = None
            self.to_owner, self.from_touchers = {}, {}
            return
        perm = np.asarray(plan.iface_perm_host, dtype=np.int64)  # local B dof -> global interface id
        owner, q_of, glob_of_node, rank_of = interface_owner_rank(plan, size)
        touched = np.unique(perm)
        own = touched[owner[touched] == rank]
        ghost = touched[owner[touched] != rank]
        self.glob_ids = np.concatenate([own, ghost])
        self.n_own, self.n_loc = own.size, touched.size
        loc_of = np.full(n_hat, -1, dtype=np.int64)
        loc_of[self.glob_ids] = np.arange(self.n_loc)
        self.perm_loc = loc_of[perm]
        # ranks touching each dof (through the sharers of its glob)
        glob_of_q = np.empty(n_hat, dtype=np.int64)
        glob_of_q[q_of] = glob_of_node
        sh_rank = rank_of[plan.sh_sub.astype(np.int64)]
        # ghosts -> their owner; owned dofs <- every other rank touching them
        self.to_owner = {}
        for s in np.unique(owner[ghost]):
            q = ghost[owner[ghost] == s]
            self.to_owner[int(s)] = loc_of[q]
        self.from_touchers = {}
        if own.size:
            g = glob_of_q[own]
            starts = plan.sh_start.astype(np.int64)
            for s in range(size):
                if s == rank:
                    continue
                # does rank s own a sharer of glob g?
                has = np.zeros(plan.G, dtype=bool)
                has[np.repeat(np.arange(plan.G), np.diff(starts))[sh_rank == s]] = True
                q = own[has[g]]
                if q.size:
                    self.from_touchers[s] = loc_of[q]

    # -- device index arrays -------------------------------------------------
    def _device(self):
        if self._dev is None:
            import torch

            def up(a):
                return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()
            self._dev = {
                "to_owner": {s: up(i) for s, i in self.to_owner.items()},
                "from_touchers": {s: up(i) for s, i in self.from_touchers.items()},
                "own_glob": up(self.glob_ids[:self.n_own]),
                "loc_glob": up(self.glob_ids),
            }
        return self._dev

    def halo_sum_(self, y):
        """Complete subassembled partial sums on a local vector in place:
        ghosts' partials -> owners (added in rank order), totals -> ghosts."""
        if not self.multi:
            return y
        import torch

        from ._lib import lib, stream

        dv = self._device()
        st = stream()
        sends = {}
        for s, idx in dv["to_owner"].items():
            b = torch.empty(idx.numel(), dtype=y.dtype, device=y.device)
            lib.bddc_gather_idx(y, idx, idx.numel(), b, st)
            sends[s] = b
        recvs = {s: torch.empty(idx.numel(), dtype=y.dtype, device=y.device)
                 for s, idx in dv["from_touchers"].items()}
        self.comm.exchange(sends, recvs)
        for s in sorted(recvs):
            idx = dv["from_touchers"][s]
            lib.bddc_scatter_idx(y, idx, idx.numel(), recvs[s], 1, st)
        # round 2: owners' totals back to every rank touching them
        sends = {}
        for s, idx in dv["from_touchers"].items():
            b = torch.empty(idx.numel(), dtype=y.dtype, device=y.device)
            lib.bddc_gather_idx(y, idx, idx.numel(), b, st)
            sends[s] = b
        recvs = {s: torch.empty(idx.numel(), dtype=y.dtype, device=y.device)
                 for s, idx in dv["to_owner"].items()}
        self.comm.exchange(sends, recvs)
        for s in sorted(recvs):
            idx = dv["to_owner"][s]
            lib.bddc_scatter_idx(y, idx, idx.numel(), recvs[s], 0, st)
        return y

    def to_local(self, v):
        """Global interface vector (device) -> this rank's local vector."""
        if not self.multi:
            return v
        return v[self._device()["loc_glob"]]

    def to_global(self, x):
        """Local vector -> the global interface vector on every rank (owned
        entries of all ranks, one allreduce)."""
        if not self.multi:
            return x
        import torch

        out = torch.zeros(self.n_hat, dtype=x.dtype, device=x.device)
        out[self._device()["own_glob"]] = x[:self.n_own]
        self.comm.allreduce_(out)
        return out

    def halo_bytes(self):
        """Bytes one halo_sum_ moves out of this rank (both rounds)."""
        return 8 * (sum(i.size for i in self.to_owner.values())
                    + sum(i.size for i in self.from_touchers.values()))


class SlotExchange:
    """Point-to-point exchange of per-(glob, sharer) slot blocks between the
    rank that owns a glob (first sharer) and the ranks of its other sharers.

    ``to_owner``: slots whose sharer is local and whose glob is owned
    elsewhere go to the glob's owner; ``to_sharers``: slots of locally owned
    globs whose sharer lives elsewhere go to that sharer's rank.  Blocks are
    addressed by (offset, size) per slot, so any slot-layout buffer (Bsym
    blocks, deluxe weights, prior X blocks) uses the same plan."""

    def __init__(self, plan, comm):
        self.comm = comm
        size, rank = comm.size, comm.rank
        rank_of = rank_of_subdomain(plan.N_glob, size)
        slot_glob = plan.slot_glob.astype(np.int64)
        first = plan.sh_sub[plan.sh_start[:-1]].astype(np.int64)
        self.glob_owner = rank_of[first]
        self.slot_rank = rank_of[plan.sh_sub.astype(np.int64)]
        self.slot_owner = self.glob_owner[slot_glob]
        cross = self.slot_rank != self.slot_owner
        self.cross = cross
        self.rank = rank

    def _pairs(self, direction):
        """{peer: ascending slot ids} to send and to receive."""
        mine_sh = self.slot_rank == self.rank
        mine_ow = self.slot_owner == self.rank
        send, recv = {}, {}
        if direction == "to_owner":
            s_mask, s_peer = self.cross & mine_sh, self.slot_owner
            r_mask, r_peer = self.cross & mine_ow, self.slot_rank
        else:
            s_mask, s_peer = self.cross & mine_ow, self.slot_rank
            r_mask, r_peer = self.cross & mine_sh, self.slot_owner
        for p in np.unique(s_peer[s_mask]):
            send[int(p)] = np.flatnonzero(s_mask & (s_peer == p))
        for p in np.unique(r_peer[r_mask]):
            recv[int(p)] = np.flatnonzero(r_mask & (r_peer == p))
        return send, recv

    @staticmethod
    def _index(slots, off, sizes):
        if not slots.size:
            return np.zeros(0, dtype=np.int64)
        o = np.asarray(off, dtype=np.int64)[slots]
        n = np.asarray(sizes, dtype=np.int64)[slots]
        from .plan import _ranges
        return _ranges(o, n)

    def run(self, buf, off, sizes, direction, per_glob=None):
        """Move the cross-rank slots of `buf` (slot k at off[k], sizes[k]
        entries) in `direction` ("to_owner" / "to_sharers").  per_glob (the
        slot -> glob map): the buffer is per glob (off / sizes index slots but
        address the glob's block), so each (glob, peer) pair moves once.
        Returns the bytes this rank sent."""
        import torch

        from ._lib import lib, stream

        send, recv = self._pairs(direction)
        if per_glob is not None:
            def dedupe(d):
                out = {}
                for p, sl in d.items():
                    _, first = np.unique(per_glob[sl], return_index=True)
                    out[p] = sl[np.sort(first)]
                return out
            send, recv = dedupe(send), dedupe(recv)
        st = stream()
        sends, recvs, unpack = {}, {}, {}
        sent = 0
        for p, slots in send.items():
            idx = torch.from_numpy(self._index(slots, off, sizes)).cuda()
            b = torch.empty(idx.numel(), dtype=buf.dtype, device=buf.device)
            lib.bddc_gather_idx(buf, idx, idx.numel(), b, st)
            sends[p] = b
            sent += 8 * idx.numel()
        for p, slots in recv.items():
            idx = torch.from_numpy(self._index(slots, off, sizes)).cuda()
            recvs[p] = torch.empty(idx.numel(), dtype=buf.dtype, device=buf.device)
            unpack[p] = idx
        self.comm.exchange(sends, recvs)
        for p in sorted(recvs):
            idx = unpack[p]
            lib.bddc_scatter_idx(buf, idx, idx.numel(), recvs[p], 0, st)
        return sent
