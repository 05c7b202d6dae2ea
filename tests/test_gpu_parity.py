"""Parity of the CUDA path against the reference golden fixtures (and the
oracle for intermediate quantities).  Bars (north_star): per-glob primal
counts exact except eigenvalues within 1e-8 relative of the threshold,
GMRES iterations +-1, solutions relative difference <= 1e-8 in fp64."""

import numpy as np
import pytest

from tests.cases import FIXTURES, counts_match, gevp_values, golden, inputs, probe_vector, variants

pytestmark = pytest.mark.gpu

FAST = [n for n in FIXTURES if n not in ("cfg3", "cfg4", "cfg5")]


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", FAST)
def test_pipeline_matches_reference(name):
    from paper_2501_01676_b200 import pipeline
    from paper_2501_01676_b200.substructuring import SubdomainOperator

    g = golden(name)
    system, part, globs = inputs(name)
    kinds = [gl.kind for gl in globs.globs]
    for v in variants(g):
        res = pipeline.run(system, part, globs, float(g["theta_f"]), float(g["theta_e"]), v,
                           keep=True)
        ls = res.ls
        assert np.array_equal(ls.plan.nB, g["nB"])
        for i in g["S_ids"].tolist():
            op = SubdomainOperator(ls, i)
            assert _rel(op.S, g[f"S_{i}"]) <= 1e-12, i
            assert _rel(op.g, g[f"g_{i}"]) <= 1e-12, i
            assert _rel(op.bsym_inverse(), g[f"Binv_{i}"]) <= 1e-10, i
        assert _rel(res.op.rhs_device().cpu().numpy(), g["rhs"]) <= 1e-12
        assert _rel(res.op(g["probe"]), g["Sprobe"]) <= 1e-12
        ref_eig = gevp_values(g, v)
        mine = res.space.all_eigenvalues()
        for k, ev in ref_eig.items():
            fin = np.isfinite(ev)
            assert mine[k].shape == ev.shape, k
            assert np.array_equal(np.isfinite(mine[k]), fin), k
            scale = np.abs(ev[fin]).max(initial=1.0)
            np.testing.assert_allclose(mine[k][fin], ev[fin], rtol=1e-8, atol=1e-10 * scale)
        th = lambda k: float(g["theta_f"]) if kinds[k] == "face" else float(g["theta_e"])
        assert counts_match(res.n_primal, g[f"{v}_n_primal"], None, ref_eig, th) == []
        assert (res.pnumF, res.pnumE, res.n_vertex) == (
            int(g[f"{v}_pnumF"]), int(g[f"{v}_pnumE"]), int(g[f"{v}_n_vertex"]))
        assert abs(res.iterations - int(g[f"{v}_iterations"])) <= 1
        assert _rel(res.pc.apply(g["probe"]), g[f"{v}_Mprobe"]) <= 1e-7
        assert _rel(res.solution.cpu().numpy(), g[f"{v}_solution"]) <= 1e-8
        assert _rel(res.u.cpu().numpy(), g[f"{v}_u"]) <= 1e-8


@pytest.mark.parametrize("name", [n for n in ("cfg3", "cfg4", "cfg5") if n in FIXTURES])
def test_large_configs_match_reference(name):
    """BASELINE configs[2] (512 subdomains), configs[3] (irregular BFS
    partition, 511 subdomains, faces up to 193 dofs) and configs[4] (the
    bench workload: 128^3 cells, 4,096 subdomains, 2,048,383 DOFs) against
    the reference.  The cfg5 fixture is lean (make_golden.py): the interface
    solution in full, rhs / S_hat probe / M^-1 probe / nodal u at 20,000
    seeded entries."""
    from paper_2501_01676_b200 import pipeline

    g = golden(name)
    system, part, globs = inputs(name)
    kinds = [gl.kind for gl in globs.globs]
    v = "new"
    res = pipeline.run(system, part, globs, float(g["theta_f"]), float(g["theta_e"]), v, keep=True)
    assert np.array_equal(res.ls.plan.nB, g["nB"])
    ref_eig = gevp_values(g, v)
    mine = res.space.all_eigenvalues()
    # cfg4's nu spans 1e-3..1e3: its pencils are ill-conditioned enough that
    # LAPACK and the device eigensolvers agree to ~1e-8 relative on the largest
    # eigenvalues (1e5); the selection margin to theta is 3.5e-4
    rtol = 1e-6 if name == "cfg4" else 1e-8
    for k, ev in ref_eig.items():
        fin = np.isfinite(ev)
        scale = np.abs(ev[fin]).max(initial=1.0)
        np.testing.assert_allclose(mine[k][fin], ev[fin], rtol=rtol, atol=1e-10 * scale)
    th = lambda k: float(g["theta_f"]) if kinds[k] == "face" else float(g["theta_e"])
    assert counts_match(res.n_primal, g[f"{v}_n_primal"], None, ref_eig, th) == []
    assert (res.pnumF, res.pnumE, res.n_vertex) == (
        int(g[f"{v}_pnumF"]), int(g[f"{v}_pnumE"]), int(g[f"{v}_n_vertex"]))
    assert abs(res.iterations - int(g[f"{v}_iterations"])) <= 1
    assert _rel(res.solution.cpu().numpy(), g[f"{v}_solution"]) <= 1e-8
    sub_hat = g.get("sub_hat")
    sub_u = g.get("sub_u")
    u = res.u.cpu().numpy()
    assert _rel(u if sub_u is None else u[sub_u], g[f"{v}_u"]) <= 1e-8
    if sub_hat is not None:  # lean fixture: sampled rhs / operator / preconditioner probes
        probe = probe_vector(g)
        assert _rel(res.op.rhs_device().cpu().numpy()[sub_hat], g["rhs"]) <= 1e-12
        assert _rel(res.op(probe)[sub_hat], g["Sprobe"]) <= 1e-12
        assert _rel(res.pc.apply(probe)[sub_hat], g[f"{v}_Mprobe"]) <= 1e-7


@pytest.mark.parametrize("name", [n for n in ("jump", "cfg2", "cfg4_small", "cfg1") if n in FIXTURES])
def test_general_gep_path_matches_reference(name):
    """The face / edge eigenproblems with every certified shortcut disabled
    (eigen-based pseudo-inverse parallel sums, the general pencil solver of
    linalg.py:116-214) reproduce the reference's eigenvalues, counts,
    iterations and solution, and agree with the default fast path."""
    from paper_2501_01676_b200 import pipeline

    g = golden(name)
    system, part, globs = inputs(name)
    kinds = [gl.kind for gl in globs.globs]
    for v in variants(g):
        res = pipeline.run(system, part, globs, float(g["theta_f"]), float(g["theta_e"]), v,
                           keep=True, general=True)
        assert res.space.general
        ref_eig = gevp_values(g, v)
        mine = res.space.all_eigenvalues()
        for k, ev in ref_eig.items():
            fin = np.isfinite(ev)
            assert np.array_equal(np.isfinite(mine[k]), fin), k
            scale = np.abs(ev[fin]).max(initial=1.0)
            np.testing.assert_allclose(mine[k][fin], ev[fin], rtol=1e-8, atol=1e-10 * scale)
        th = lambda k: float(g["theta_f"]) if kinds[k] == "face" else float(g["theta_e"])
        assert counts_match(res.n_primal, g[f"{v}_n_primal"], None, ref_eig, th) == []
        assert abs(res.iterations - int(g[f"{v}_iterations"])) <= 1
        assert _rel(res.solution.cpu().numpy(), g[f"{v}_solution"]) <= 1e-8
