"""Subdomain sharding over ranks (one process per GPU).

The reference solves every subdomain in one process; its data
parallelism is the loop over subdomains.  Here rank r owns the contiguous
subdomain block ``block_range(N, R, r)`` and everything per-subdomain
(assembly, Schur elimination, Bsym^-1, local preconditioner operators,
interior recovery) runs only there.  The exchange points are sum-allreduces
of buffers laid out globally with zeros in the slots other ranks own:

* slot blocks of Bsym / Bsym^-1 (``bddc_extract_slot_blocks``) before the
  glob phase; deluxe blocks, face results, edge X blocks and edge results
  after each glob sub-phase (each glob is computed by the rank owning its
  first sharer);
* the per-subdomain coarse blocks C_i (the coarse LU is factorised
  redundantly on every rank, it is small next to the subdomain work);
* per Krylov step: the partial S_hat v, the coarse right-hand side and the
  partial M^-1 r (interface vectors are replicated, so GMRES itself is
  redundant and deterministic on every rank);
* the interior values of the recovered solution.

``TorchComm`` wraps ``torch.distributed`` (NCCL on GPUs, gloo on CPU);
``LoopbackComm`` runs R ranks as threads of one process (tests on one
GPU: every exchange is a host-side barrier after a stream synchronize, no
kernel ever waits on another rank's kernel).
"""

import threading

import numpy as np


def block_range(n, size, rank):
    """Contiguous balanced split of range(n): [s0, s1) of `rank`."""
    q, r = divmod(int(n), int(size))
    s0 = rank * q + min(rank, r)
    return s0, s0 + q + (1 if rank < r else 0)


class Comm:
    rank = 0
    size = 1

    def allreduce_(self, t):
        """In-place elementwise sum over ranks; returns t."""
        return t

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

    def allreduce_(self, t):
        if self.size > 1 and t.numel():
            self.dist.all_reduce(t, group=self.group)
        return t

    def barrier(self):
        if self.size > 1:
            self.dist.barrier(group=self.group)


class _LoopbackHub:
    def __init__(self, size):
        self.size = size
        self.bar = threading.Barrier(size)
        self.slots = [None] * size
        self.result = None


class LoopbackComm(Comm):
    """Rank `rank` of `size` threads sharing one process and one GPU."""

    def __init__(self, hub, rank):
        self.hub, self.rank, self.size = hub, rank, hub.size

    @staticmethod
    def group(size):
        hub = _LoopbackHub(size)
        return [LoopbackComm(hub, r) for r in range(size)]

    def allreduce_(self, t):
        if self.size == 1:
            return t
        import torch

        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        h = self.hub
        h.slots[self.rank] = t
        h.bar.wait()
        if self.rank == 0:
            acc = h.slots[0].clone()
            for x in h.slots[1:]:
                acc += x.to(acc.device)
            if acc.is_cuda:
                torch.cuda.current_stream().synchronize()
            h.result = acc
        h.bar.wait()
        t.copy_(h.result.to(t.device))
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        h.bar.wait()
        return t

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
    if isinstance(comm, TorchComm) and comm.dist.get_backend(comm.group) == "nccl":
        t = t.cuda()
    comm.allreduce_(t)
    return t.cpu().numpy()
