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
