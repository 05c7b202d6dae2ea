"""The round-2 fast paths against their plain counterparts on the same inputs:
two-phase elimination vs one phase, the fused GMRES step vs the separate
vector kernels, the overlapped coarse branch vs the single-stream apply."""

import numpy as np
import pytest

from tests.cases import golden, inputs

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", ["jump", "cfg4_small", "cfg2"])
def test_two_phase_elimination_matches_one_phase(name, monkeypatch):
    """Deep-first ordering + column hole vs the plain elimination: same S, g and
    recovered interiors to rounding (the interior order differs, the operators
    do not)."""
    import torch

    from paper_2501_01676_b200 import engine

    system, part, globs = inputs(name)
    a = engine.LocalSystem(system, part, globs)
    monkeypatch.setattr(engine, "TWO_PHASE", False)
    b = engine.LocalSystem(system, part, globs)
    assert int(a.plan.nDeep.max()) > 0
    for k in ("S", "g"):
        x, y = getattr(a, k).cpu().numpy(), getattr(b, k).cpu().numpy()
        assert np.abs(x - y).max() <= 1e-12 * np.abs(y).max(), k
    u_hat = torch.linspace(-1.0, 2.0, a.plan.n_hat, dtype=torch.float64, device="cuda")
    ub = engine.recover_device(b, u_hat).cpu().numpy()
    monkeypatch.setattr(engine, "TWO_PHASE", True)
    ua = engine.recover_device(a, u_hat).cpu().numpy()
    assert _rel(ua, ub) <= 1e-12


@pytest.mark.parametrize("name", ["jump", "cfg4_small"])
def test_fused_gmres_step_matches_separate_kernels(name, monkeypatch):
    from paper_2501_01676_b200 import engine, pipeline

    g = golden(name)
    system, part, globs = inputs(name)
    th_f, th_e = float(g["theta_f"]), float(g["theta_e"])
    monkeypatch.setattr(engine, "FUSED_GMRES", True)
    a = pipeline.run(system, part, globs, th_f, th_e, "new")
    monkeypatch.setattr(engine, "FUSED_GMRES", False)
    b = pipeline.run(system, part, globs, th_f, th_e, "new")
    assert a.iterations == b.iterations == int(g["new_iterations"])
    assert _rel(a.solution.cpu().numpy(), b.solution.cpu().numpy()) <= 1e-10
    # same residual histories to rounding (different reduction trees)
    np.testing.assert_allclose(a.pre_hist, b.pre_hist, rtol=1e-6)
    np.testing.assert_allclose(a.true_hist, b.true_hist, rtol=1e-6)


@pytest.mark.parametrize("name", ["jump", "cfg4_small"])
def test_overlapped_coarse_branch_is_bitwise_the_same_apply(name, monkeypatch):
    import torch

    from paper_2501_01676_b200 import engine, pipeline

    g = golden(name)
    system, part, globs = inputs(name)
    res = pipeline.run(system, part, globs, float(g["theta_f"]), float(g["theta_e"]), "new",
                       keep=True)
    r = torch.linspace(-1.0, 1.0, res.ls.plan.n_hat, dtype=torch.float64, device="cuda")
    monkeypatch.setattr(engine, "OVERLAP_COARSE", True)
    ya = res.pc.apply_device(r).cpu().numpy()
    monkeypatch.setattr(engine, "OVERLAP_COARSE", False)
    yb = res.pc.apply_device(r).cpu().numpy()
    assert ya.tobytes() == yb.tobytes()
    assert _rel(ya, res.pc.apply(r.cpu().numpy())) <= 1e-14


@pytest.mark.parametrize("name", ["jump", "cfg4_small", "cfg2"])
def test_staged_upload_is_bitwise_the_plain_upload(name):
    """upload_inputs(pinned=True): page-locked buffers, the late inputs (nodes,
    viscosity table, Dirichlet values) and the element kernel on the copy
    stream behind the plan -- same bits as the blocking upload, run after run."""
    from paper_2501_01676_b200 import engine, pipeline

    g = golden(name)
    system, part, globs = inputs(name)
    th_f, th_e = float(g["theta_f"]), float(g["theta_e"])
    ref = pipeline.run(system, part, globs, th_f, th_e, "new",
                       inputs=engine.upload_inputs(system, part))
    staged = engine.stage_inputs(system, part)
    for _ in range(3):
        inp = engine.upload_staged(staged)
        assert inp.get("_late") is not None
        res = pipeline.run(system, part, globs, th_f, th_e, "new", inputs=inp)
        assert res.iterations == ref.iterations == int(g["new_iterations"])
        assert np.array_equal(res.u.cpu().numpy(), ref.u.cpu().numpy())
    # the pieces on their own (no pipeline): LocalSystem orders itself behind the copies
    a = engine.LocalSystem(system, part, globs, inputs=engine.upload_staged(staged))
    b = engine.LocalSystem(system, part, globs, inputs=engine.upload_inputs(system, part))
    assert np.array_equal(a.S.cpu().numpy(), b.S.cpu().numpy())
    assert np.array_equal(a.g.cpu().numpy(), b.g.cpu().numpy())
