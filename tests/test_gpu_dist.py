"""Sharded hot path on one GPU: R loopback ranks (threads, dist.py), each
owning a contiguous block of subdomains, exchange only through the
sum-allreduces the NCCL path uses.  Results must match the reference
fixtures with the same bars as the single-rank path, and the single-rank
run itself to rounding."""

import numpy as np
import pytest

from tests.cases import counts_match, gevp_values, golden, inputs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name,size", [("jump", 2), ("jump", 3), ("cfg4_small", 4), ("cfg2", 2)])
def test_sharded_pipeline_matches_reference(name, size):
    from paper_2501_01676_b200 import pipeline
    from paper_2501_01676_b200.dist import run_threads

    g = golden(name)
    system, part, globs = inputs(name)
    kinds = [gl.kind for gl in globs.globs]
    v = "new"
    th_f, th_e = float(g["theta_f"]), float(g["theta_e"])
    single = pipeline.run(system, part, globs, th_f, th_e, v, keep=True)

    def rank(comm):
        res = pipeline.run(system, part, globs, th_f, th_e, v, keep=True, comm=comm)
        return (res.iterations, res.solution.cpu().numpy(), res.u.cpu().numpy(), res.n_primal,
                res.space.all_eigenvalues(), res.pc.apply(g["probe"]), res.op(g["probe"]),
                res.ls.plan.owned)

    outs = run_threads(size, rank)
    owned = [o[7] for o in outs]
    assert owned[0][0] == 0 and owned[-1][1] == part.n_subdomains
    ref_eig = gevp_values(g, v)
    th = lambda k: th_f if kinds[k] == "face" else th_e
    for it, x, u, n_primal, eig, Mp, Sp, _ in outs:
        assert abs(it - int(g[f"{v}_iterations"])) <= 1
        assert counts_match(n_primal, g[f"{v}_n_primal"], None, ref_eig, th) == []
        for k, ev in ref_eig.items():
            fin = np.isfinite(ev)
            scale = np.abs(ev[fin]).max(initial=1.0)
            np.testing.assert_allclose(eig[k][fin], ev[fin], rtol=1e-8, atol=1e-10 * scale)
        assert _rel(Sp, g["Sprobe"]) <= 1e-12
        assert _rel(Mp, g[f"{v}_Mprobe"]) <= 1e-7
        assert _rel(x, g[f"{v}_solution"]) <= 1e-8
        assert _rel(u, g[f"{v}_u"]) <= 1e-8
        # against the unsharded device run: same algorithm, different summation order only
        assert it == single.iterations
        assert np.array_equal(n_primal, single.n_primal)
        assert _rel(x, single.solution.cpu().numpy()) <= 1e-10
    # every rank holds the same replicated result
    for o in outs[1:]:
        assert np.array_equal(o[1], outs[0][1])


def test_sharded_device_elements_match_single():
    """Sharded ranks building their own element blocks on the device (BASELINE
    coefficient fields, per-rank element subsets) reproduce the single-rank run."""
    import torch

    from paper_2501_01676_b200 import configs, pipeline
    from paper_2501_01676_b200.dist import run_threads

    prob = configs.build_problem(2, n=16, subs=2)
    args = (prob.system, prob.partition, prob.globs, 1.0 + np.log(8.0), 10.0, "new")
    single = pipeline.run(*args)
    ref = single.solution.cpu().numpy()

    def rank(comm):
        res = pipeline.run(*args, comm=comm)
        torch.cuda.synchronize()
        return res.iterations, res.solution.cpu().numpy(), res.u.cpu().numpy()

    for it, x, u in run_threads(3, rank):
        assert it == single.iterations
        assert _rel(x, ref) <= 1e-10
        assert _rel(u, single.u.cpu().numpy()) <= 1e-10


def test_sharded_ranks_with_staged_uploads_match_single():
    """What bench.py does per rank: page-locked per-rank element subsets
    (stage_inputs(owned=...)), the staged upload with its late inputs on the
    copy stream, then the sharded pipeline."""
    import torch

    from paper_2501_01676_b200 import configs, pipeline
    from paper_2501_01676_b200.dist import run_threads
    from paper_2501_01676_b200.engine import stage_inputs, upload_staged

    prob = configs.build_problem(2, n=16, subs=2)
    args = (prob.system, prob.partition, prob.globs, 1.0 + np.log(8.0), 10.0, "new")
    single = pipeline.run(*args)

    def rank(comm):
        owned = comm.owned(prob.partition.n_subdomains)
        staged = stage_inputs(prob.system, prob.partition, owned=owned)
        out = []
        for _ in range(2):
            inp = upload_staged(staged)
            assert inp.get("_late") is not None
            res = pipeline.run(*args, inputs=inp, comm=comm)
            torch.cuda.synchronize()
            out.append((res.iterations, res.solution.cpu().numpy(), res.u.cpu().numpy()))
        return out

    for runs in run_threads(2, rank):
        for it, x, u in runs:
            assert it == single.iterations
            assert _rel(x, single.solution.cpu().numpy()) <= 1e-10
            assert _rel(u, single.u.cpu().numpy()) <= 1e-10
        assert np.array_equal(runs[0][1], runs[1][1]) and np.array_equal(runs[0][2], runs[1][2])


def _gloo_gpu_worker(rank, size, port, q, name):
    import os

    import torch
    import torch.distributed as dist

    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=size)
        from paper_2501_01676_b200 import pipeline
        from paper_2501_01676_b200.dist import TorchComm

        comm = TorchComm()
        g = golden(name)
        system, part, globs = inputs(name)
        res = pipeline.run(system, part, globs, float(g["theta_f"]), float(g["theta_e"]), "new",
                           comm=comm, keep=True)
        lay = res.ls.layout
        out = (res.iterations, _rel(res.solution.cpu().numpy(), g["new_solution"]),
               _rel(res.u.cpu().numpy(), g["new_u"]), res.pnumF, res.pnumE, res.n_vertex,
               lay.n_own, lay.n_loc, lay.halo_bytes())
        q.put((rank, out))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surfaced to the parent
        q.put((rank, repr(e)))
        raise


@pytest.mark.parametrize("name", ["jump", "cfg4_small"])
def test_two_processes_torchcomm_end_to_end(name):
    """pipeline.run(comm=TorchComm()) in two processes on one GPU (gloo,
    device buffers staged through the host; no kernel waits on the other
    rank's): halo exchange, owned-entry dots, coarse reduce / solve on rank 0 /
    broadcast, point-to-point glob-block exchange; against the golden fixture."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_gpu_worker, args=(r, 2, port, q, name)) for r in range(2)]
    for p in ps:
        p.start()
    outs = dict(q.get(timeout=900) for _ in range(2))
    for p in ps:
        p.join(timeout=120)
    g = golden(name)
    for r in (0, 1):
        assert not isinstance(outs[r], str), outs[r]
        it, dx, du, F, E, V, n_own, n_loc, hb = outs[r]
        assert abs(it - int(g["new_iterations"])) <= 1
        assert dx <= 1e-8 and du <= 1e-8
        assert (F, E, V) == (int(g["new_pnumF"]), int(g["new_pnumE"]), int(g["new_n_vertex"]))
        assert 0 < n_own <= n_loc and hb > 0
    assert outs[0][6] + outs[1][6] == int(g["n_hat"])
    assert all(p.exitcode == 0 for p in ps)
