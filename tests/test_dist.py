"""Subdomain sharding (dist.py / Plan(owned=...)) on the CPU: the per-rank
plans tile the global plan exactly, every glob and every (glob, sharer) slot
has exactly one owner, and a world-size-2 gloo group reproduces the
interface operator S_hat v = sum_i R_i^T S_i R_i v (reference
solver.py:226-235) from per-rank partial products and one sum-allreduce."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_01676_b200.dist import TorchComm, allreduce_np, block_range
from paper_2501_01676_b200.plan import Plan
from tests.cases import inputs


def test_block_range_tiles():
    for n in (0, 1, 7, 512, 4096):
        for size in (1, 2, 3, 8):
            rs = [block_range(n, size, r) for r in range(size)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs[:-1], rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


@pytest.mark.parametrize("name,size", [("jump", 2), ("jump", 3), ("cfg4_small", 4)])
def test_sharded_plans_tile_global_plan(name, size):
    system, part, globs = inputs(name)
    full = Plan(system, part, globs)
    parts = [Plan(system, part, globs, owned=block_range(part.n_subdomains, size, r))
             for r in range(size)]
    cat = lambda f: np.concatenate([f(q) for q in parts])
    assert np.array_equal(cat(lambda q: q.nI), full.nI)
    assert np.array_equal(cat(lambda q: q.nB), full.nB)
    assert np.array_equal(cat(lambda q: q.I_nodes), full.I_nodes)
    assert np.array_equal(cat(lambda q: q.B_nodes), full.B_nodes)
    assert np.array_equal(cat(lambda q: q.iface_perm), full.iface_perm)
    assert np.array_equal(cat(lambda q: q.elem_ids), full.elem_ids)
    sub_of = np.asarray(part.subdomain_of)
    for q in parts:  # loc4 is indexed by element id: each rank fills its own elements
        mine = (sub_of >= q.owned[0]) & (sub_of < q.owned[1])
        assert np.array_equal(q.loc4[mine], full.loc4[mine])
    assert np.array_equal(cat(lambda q: q.sub_glob_sh), full.sub_glob_sh)
    assert np.array_equal(cat(lambda q: q.pos2k + full.sub_glob_start[q.owned[0]]), full.pos2k)
    # glob tables replicated, ownership a partition
    for q in parts:
        assert np.array_equal(q.sh_doff, full.sh_doff) and np.array_equal(q.g_nB, full.nB)
    own = np.stack([q.glob_mine for q in parts]).astype(int)
    assert np.all(own.sum(0) == 1)
    slot_owned = np.stack([q.slot_local >= 0 for q in parts]).astype(int)
    assert np.all(slot_owned.sum(0) == 1)
    for q in parts:
        s0 = q.owned[0]
        loc = q.slot_local >= 0
        assert np.array_equal(q.slot_local[loc] + s0, q.sh_sub[loc])
    # the local subdomain -> glob incidence is the global one, renumbered
    for q in parts:
        s0, s1 = q.owned
        for s in range(s0, s1):
            a, b = full.sub_glob_start[s], full.sub_glob_start[s + 1]
            la, lb = q.sub_glob_start[s - s0], q.sub_glob_start[s - s0 + 1]
            assert np.array_equal(full.sub_globs[a:b], q.sub_globs[la:lb])
            assert np.array_equal(full.sub_glob_boff[a:b], q.sub_glob_boff[la:lb])


def test_sharded_plan_errors_use_global_ids():
    from paper_2501_01676_b200.decomposition import classify_globs, partition_regular
    from paper_2501_01676_b200.discretization import assemble_system
    from paper_2501_01676_b200.mesh import box_mesh
    from tests.cases import const_coefficients

    mesh = box_mesh(((0, 1), (0, 1), (0, 1)), (2, 2, 2))  # 1-cell subdomains: no interior
    part = partition_regular(mesh, (2, 2, 2))
    globs = classify_globs(mesh, part, mesh.boundary_nodes)
    system = assemble_system(mesh, const_coefficients())
    with pytest.raises(ValueError, match="subdomain 4 has no interior"):
        Plan(system, part, globs, owned=(4, 8)).check()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, size, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=size)
        comm = TorchComm()
        from oracle import bddc_oracle as O

        system, part, globs = inputs("jump")
        s0, s1 = comm.owned(part.n_subdomains)
        plan = Plan(system, part, globs, owned=(s0, s1))
        n = globs.interface_nodes.size
        v = np.random.default_rng(7).standard_normal(n)
        y = np.zeros(n)
        g = np.zeros(n)
        for s in range(s0, s1):
            op = O.local_operator(system, part, globs, s)
            # the plan's local B dofs are this subdomain's interface nodes
            loc = plan.B_nodes[plan.voff[s - s0]:plan.voff[s - s0 + 1]]
            assert np.array_equal(np.sort(loc), op.interface_nodes)
            y[op.iface_index] += op.S @ v[op.iface_index]
            g[op.iface_index] += op.g
        y = allreduce_np(comm, y)
        g = allreduce_np(comm, g)
        counts = allreduce_np(comm, np.array([plan.nI.sum(), plan.nB.sum()], dtype=np.int64))
        if rank == 0:
            full = O.all_local_operators(system, part, globs)
            ref = np.zeros(n)
            refg = np.zeros(n)
            for op in full:
                ref[op.iface_index] += op.S @ v[op.iface_index]
                refg[op.iface_index] += op.g
            fp = Plan(system, part, globs)
            q.put((float(np.abs(y - ref).max() / np.abs(ref).max()),
                   float(np.abs(g - refg).max() / max(np.abs(refg).max(), 1e-300)),
                   counts.tolist(), [int(fp.nI.sum()), int(fp.nB.sum())]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surfaced to the parent
        q.put(repr(e))
        raise


def test_gloo_world2_interface_operator():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
    assert not isinstance(res, str), res
    dy, dg, counts, ref_counts = res
    assert dy <= 1e-13 and dg <= 1e-13
    assert counts == ref_counts
    assert all(p.exitcode == 0 for p in ps)


@pytest.mark.parametrize("name,size", [("jump", 2), ("jump", 3), ("cfg4_small", 4)])
def test_interface_layout_and_slot_exchange_plans(name, size):
    """Owned sets partition the interface; every rank's ghost list towards an
    owner is exactly that owner's list of dofs it receives from the rank (same
    global ids, same order); slot-exchange send / receive lists pair up."""
    from paper_2501_01676_b200.dist import InterfaceLayout, SlotExchange

    class FakeComm:
        def __init__(self, rank):
            self.rank, self.size = rank, size

    system, part, globs = inputs(name)
    plans = [Plan(system, part, globs, owned=block_range(part.n_subdomains, size, r)) for r in range(size)]
    lays = [InterfaceLayout(plans[r], FakeComm(r)) for r in range(size)]
    n_hat = globs.interface_nodes.size
    owned = np.concatenate([l.glob_ids[:l.n_own] for l in lays])
    assert np.array_equal(np.sort(owned), np.arange(n_hat))
    for r, lr in enumerate(lays):
        assert np.array_equal(np.sort(lr.glob_ids), np.unique(plans[r].iface_perm))
        for s, idx in lr.to_owner.items():
            back = lays[s].from_touchers[r]
            assert np.array_equal(lr.glob_ids[idx], lays[s].glob_ids[back])
        for s, idx in lr.from_touchers.items():
            assert r in lays[s].to_owner
    xs = [SlotExchange(plans[r], FakeComm(r)) for r in range(size)]
    for d in ("to_owner", "to_sharers"):
        pairs = [x._pairs(d) for x in xs]
        for r in range(size):
            send, _ = pairs[r]
            for s, slots in send.items():
                assert np.array_equal(slots, pairs[s][1][r])


def _halo_worker(rank, size, port, q):
    """World-size-2 gloo: S_hat v assembled from per-rank partial sums over each
    rank's touched dofs with the halo exchange (point-to-point send / recv), in
    the rank-local layout, equals the global subassembly."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=size)
        comm = TorchComm()
        from oracle import bddc_oracle as O
        from paper_2501_01676_b200.dist import InterfaceLayout

        system, part, globs = inputs("jump")
        s0, s1 = comm.owned(part.n_subdomains)
        plan = Plan(system, part, globs, owned=(s0, s1))
        lay = InterfaceLayout(plan, comm)
        n = globs.interface_nodes.size
        v = np.random.default_rng(7).standard_normal(n)
        loc = np.full(n, -1)
        loc[lay.glob_ids] = np.arange(lay.n_loc)
        y = np.zeros(lay.n_loc)
        for s in range(s0, s1):
            op = O.local_operator(system, part, globs, s)
            y[loc[op.iface_index]] += op.S @ v[op.iface_index]
        # the two halo rounds of InterfaceLayout.halo_sum_, on host tensors
        yt = torch.from_numpy(y)
        sends = {s: yt[torch.from_numpy(i)].clone() for s, i in lay.to_owner.items()}
        recvs = {s: torch.empty(len(i), dtype=torch.float64) for s, i in lay.from_touchers.items()}
        comm.exchange(sends, recvs)
        for s in sorted(recvs):
            yt[torch.from_numpy(lay.from_touchers[s])] += recvs[s]
        sends = {s: yt[torch.from_numpy(i)].clone() for s, i in lay.from_touchers.items()}
        recvs = {s: torch.empty(len(i), dtype=torch.float64) for s, i in lay.to_owner.items()}
        comm.exchange(sends, recvs)
        for s in sorted(recvs):
            yt[torch.from_numpy(lay.to_owner[s])] = recvs[s]
        full = np.zeros(n)
        full[lay.glob_ids[:lay.n_own]] = yt.numpy()[:lay.n_own]
        full = allreduce_np(comm, full)
        ref = np.zeros(n)
        for op in O.all_local_operators(system, part, globs):
            ref[op.iface_index] += op.S @ v[op.iface_index]
        ghost_ok = np.allclose(yt.numpy(), ref[lay.glob_ids], rtol=1e-13, atol=1e-13 * np.abs(ref).max())
        if rank == 0:
            q.put((float(np.abs(full - ref).max() / np.abs(ref).max()), bool(ghost_ok)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surfaced to the parent
        q.put(repr(e))
        raise


def test_gloo_world2_halo_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_halo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = q.get(timeout=600)
    for p in ps:
        p.join(timeout=120)
    assert not isinstance(res, str), res
    err, ghost_ok = res
    assert err <= 1e-13 and ghost_ok
    assert all(p.exitcode == 0 for p in ps)
