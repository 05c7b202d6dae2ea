"""The reference's diagnostics and correctness gate against the device
preconditioner (reference solver.py:54-259, diagnostics.py:81-250,
tests/test_solver.py:79-222): partially coupled space internals, the
averaging projection E_D, the dense interface oracle, partition of unity,
Loewner bounds of the parallel sums, the field of values of the
preconditioned operator, the SPD-limit spectrum and the jump-energy bounds
behind the threshold selection.  Every operator is computed on the device;
numpy / scipy only check."""

import functools
import math

import numpy as np
import pytest
import scipy.linalg

from tests.cases import EX_DOMAIN, golden, inputs

pytestmark = pytest.mark.gpu

THETA_F = 1.0 + math.log(4.0)


def _api():
    import paper_2501_01676_b200 as P

    return P


@functools.lru_cache(maxsize=None)
def _ops(name="jump"):
    P = _api()
    system, part, globs = inputs(name)
    ops = [P.build_subdomain_operator(system, part, globs, i) for i in range(part.n_subdomains)]
    return system, part, globs, ops, P.build_scaling(globs, ops)


def _solver(variant, name="jump", theta_f=THETA_F, theta_e=10.0):
    P = _api()
    system, part, globs, ops, scaling = _ops(name)
    basis, reports = P.adaptive_primal_space(globs, ops, scaling, theta_f, theta_e, variant)
    return system, globs, ops, scaling, basis, reports, P.build_preconditioner(ops, basis, scaling)


@pytest.mark.parametrize("variant", ["old", "new"])
def test_averaging_is_a_projection(variant):
    P = _api()
    *_, pc = _solver(variant)
    rng = np.random.default_rng(7)
    assert pc.wt_size == pc.n_dual_total + pc.n_primal
    wt = rng.standard_normal(pc.wt_size)
    e1, p1 = P.averaging_and_jump(pc, wt)
    assert np.abs(e1 + p1 - wt).max() < 1e-14 * max(1.0, np.abs(wt).max())
    e2, _ = P.averaging_and_jump(pc, e1)
    assert np.abs(e2 - e1).max() <= 1e-10 * max(1.0, np.abs(e1).max())


def test_continuous_vectors_are_fixed_and_dbar_mutation_breaks_projection():
    P = _api()
    *_, pc = _solver("old")
    rng = np.random.default_rng(8)
    v = rng.standard_normal(pc.n_hat)
    wt = pc.inject(v)
    e, p = P.averaging_and_jump(pc, wt)
    assert np.abs(e - wt).max() <= 1e-10 * np.abs(wt).max()
    assert np.abs(p).max() <= 1e-10 * np.abs(wt).max()
    np.testing.assert_allclose(pc.inject_t(pc.inject(v)) / v, np.bincount(
        np.concatenate([*pc.gdual_pos, pc.primal_pos]), minlength=pc.n_hat), rtol=1e-14)
    # transform is orthogonal
    np.testing.assert_allclose(pc.transform(pc.transform(v), transpose=True), v, atol=1e-12)
    # partition-of-unity violation (reference test_solver.py:140-148)
    pc.Dbar[0] = 1.21 * pc.Dbar[0]
    wt = rng.standard_normal(pc.wt_size)
    e1, _ = P.averaging_and_jump(pc, wt)
    e2, _ = P.averaging_and_jump(pc, e1)
    assert np.abs(e2 - e1).max() > 1e-6


def test_internals_index_sets_and_dual_certificate():
    for variant in ("old", "new"):
        system, globs, ops, scaling, basis, reports, pc = _solver(variant)
        assert len(pc.dual_loc) == len(ops)
        for i, op in enumerate(ops):
            loc, gids = basis.subdomain_primal(op)
            assert np.array_equal(pc.primal_loc[i], loc) and np.array_equal(pc.gprimal[i], gids)
            d = pc.dual_loc[i]
            assert np.array_equal(d, np.setdiff1d(np.arange(op.n_B), loc))
            assert np.array_equal(pc.gdual_pos[i], op.iface_index[d])
            if d.size:  # reference test_solver.py:79-90
                assert np.linalg.eigvalsh(0.5 * (op.S + op.S.T)[np.ix_(d, d)]).min() > 0
        D0 = pc.Dbar[0]
        assert D0.shape == (ops[0].n_B, ops[0].n_B)


def test_scale_matches_dense_reference_formula():
    """Dtil against its definition with the host copies of Dbar (solver.py:163-178)."""
    *_, pc = _solver("new")
    rng = np.random.default_rng(4)
    w = rng.standard_normal(pc.wt_size)
    for transpose in (False, True):
        ref = np.zeros_like(w)
        acc = np.zeros(pc.n_primal)
        wp = w[pc.n_dual_total:]
        for i in range(len(pc.dual_loc)):
            sl = slice(pc.dual_offsets[i], pc.dual_offsets[i] + pc.dual_loc[i].size)
            x = np.zeros(pc.Dbar[i].shape[0])
            x[pc.dual_loc[i]] = w[sl]
            x[pc.primal_loc[i]] = wp[pc.gprimal[i]]
            D = pc.Dbar[i]
            y = D.T @ x if transpose else D @ x
            ref[sl] = y[pc.dual_loc[i]]
            np.add.at(acc, pc.gprimal[i], y[pc.primal_loc[i]])
        ref[pc.n_dual_total:] = acc
        np.testing.assert_allclose(pc.scale(w, transpose=transpose), ref, rtol=1e-12, atol=1e-12)


def test_dense_schur_and_direct_solve():
    """assemble_dense_schur / direct_schur_solve (solver.py:245-259) against
    the golden S_hat probe, a sparse direct solve and linearity
    (reference test_solver.py:109-116, :186-222)."""
    from paper_2501_01676_b200.discretization import solve_direct

    P = _api()
    g = golden("jump")
    system, part, globs, ops, scaling = _ops()
    n = globs.interface_nodes.size
    S = P.assemble_dense_schur(ops, n)
    np.testing.assert_allclose(S @ g["probe"], g["Sprobe"], rtol=1e-12, atol=1e-12 * np.abs(g["Sprobe"]).max())
    rhs = P.interface_rhs(ops, n)
    x = P.direct_schur_solve(ops, globs, rhs)
    x_ref = solve_direct(system)[globs.interface_nodes]
    assert np.linalg.norm(x - x_ref) <= 1e-9 * np.linalg.norm(x_ref)
    rng = np.random.default_rng(12)
    r1, r2 = rng.standard_normal(n), rng.standard_normal(n)
    x12 = P.direct_schur_solve(ops, globs, 2.0 * r1 - r2)
    assert np.allclose(x12, 2.0 * P.direct_schur_solve(ops, globs, r1) - P.direct_schur_solve(ops, globs, r2),
                       rtol=1e-9, atol=1e-11)
    u = P.recover_interior(ops, globs, system, x)
    res = system.matrix @ u[system.free_nodes] - system.rhs
    assert np.linalg.norm(res) <= 1e-8 * max(1.0, np.linalg.norm(system.rhs))
    # full primal space: M^-1 is the exact inverse (test_solver.py:109-116)
    basis = P.PrimalBasis(globs, [(np.eye(gl.size), gl.size) for gl in globs.globs], "old")
    pc = P.build_preconditioner(ops, basis, scaling)
    y = pc.apply(rhs)
    assert np.linalg.norm(y - x) <= 1e-9 * np.linalg.norm(x)
    for variant in ("old", "new"):  # GMRES agrees with the direct oracle (test_solver.py:167-176)
        *_, pcv = _solver(variant)
        rep = P.gmres_solve(P.interface_operator(ops, n), rhs, pcv)
        assert rep.converged and np.linalg.norm(rep.solution - x) <= 1e-6 * np.linalg.norm(x)


def test_partition_of_unity_and_parallel_sum_loewner():
    """diagnostics.py:81-125 on the device scaling and parallel sums."""
    from paper_2501_01676_b200 import linalg
    from paper_2501_01676_b200.substructuring import glob_schur_block

    system, part, globs, ops, scaling = _ops()
    worst = 0.0
    for G in globs.globs:
        fam = scaling.of(G)
        worst = max(worst, np.abs(sum(fam.values()) - np.eye(G.size)).max())
    assert worst <= 1e-10
    worst = 0.0
    for F in globs.faces:
        i, j = F.sharers
        Bi, Bj = glob_schur_block(ops[i], F), glob_schur_block(ops[j], F)
        Pm = linalg.parallel_sum(Bi, Bj)
        scale = max(np.abs(Bi).max(), np.abs(Bj).max())
        for B in (Bi, Bj):
            worst = max(worst, -scipy.linalg.eigvalsh(B - Pm).min() / scale)
    assert worst <= 1e-9


@pytest.mark.parametrize("variant", ["old", "new"])
def test_field_of_values_and_lemma_bounds(variant):
    """diagnostics.py:136-225: <Bhat w, T w> > 0 with bounded growth for the
    dense preconditioned operator T = M^-1 S_hat, and the jump energy of
    constrained samples within 2 Theta (faces / old edges) or
    2 (|n(E)|-1) Theta (new edges) of the Bsym energy."""
    import torch

    from paper_2501_01676_b200.substructuring import glob_principal_block

    P = _api()
    system, globs, ops, scaling, basis, reports, pc = _solver(variant)
    n = globs.interface_nodes.size
    S = P.assemble_dense_schur(ops, n)
    Sd = torch.from_numpy(S).cuda()
    T = torch.stack([pc.apply_device(Sd[:, k].contiguous()) for k in range(n)], dim=1).cpu().numpy()
    Bh = 0.5 * (S + S.T)
    rng = np.random.default_rng(307)
    lo, hi = np.inf, 0.0
    for _ in range(100):
        w = rng.standard_normal(n)
        Bw, Tw = Bh @ w, T @ w
        den = w @ Bw
        lo, hi = min(lo, (Bw @ Tw) / den), max(hi, (Tw @ (Bh @ Tw)) / den)
    assert lo > 0.0 and hi < 1e4
    gm = {globs.glob_id(g): g for g in globs.globs}
    rng = np.random.default_rng(211)
    for rep in reports:
        G = gm[rep.glob_id]
        theta = THETA_F if rep.variant == "face" else 10.0
        diff = rep.variant == "edge_new"
        const = 2.0 * ((len(G.sharers) - 1) if diff else 1) * theta
        sh = list(G.sharers)
        idx = {s: ops[s].glob_index(G) for s in sh}
        D = scaling.of(G)
        rows = rep.constraint_matrix
        for _ in range(10):
            w = {s: rng.standard_normal(ops[s].n_B) for s in sh}
            if rows.size:
                rp = np.linalg.pinv(rows)
                base = w[sh[0]][idx[sh[0]]]
                if diff:
                    chk = np.concatenate([w[s][idx[s]] - base for s in sh[1:]])
                    chk = chk - rp @ (rows @ chk)
                    for b, s in enumerate(sh[1:]):
                        w[s][idx[s]] = base + chk[b * G.size:(b + 1) * G.size]
                else:
                    for s in sh[1:]:
                        e = w[s][idx[s]]
                        w[s][idx[s]] = e + rp @ (rows @ (base - e))
            wl = [w[s][idx[s]] for s in sh]
            avg = sum(D[s] @ x for s, x in zip(sh, wl))
            lhs = sum(float((x - avg) @ glob_principal_block(ops[s], G) @ (x - avg)) for s, x in zip(sh, wl))
            rhs = sum(w[s] @ ops[s].Bsym @ w[s] for s in sh)
            assert lhs <= const * rhs + 1e-8 * max(1.0, rhs), rep.glob_id


def test_spd_limit_spectrum():
    """diagnostics.py:228-242: no advection, unit viscosity: the preconditioned
    operator's eigenvalues lie in [1, 40 Theta^2]."""
    import torch

    P = _api()
    from paper_2501_01676_b200.decomposition import classify_globs, partition_regular
    from paper_2501_01676_b200.discretization import Coefficients, assemble_system
    from paper_2501_01676_b200.mesh import box_mesh

    mesh = box_mesh(EX_DOMAIN, (6, 6, 6))
    coeffs = Coefficients(viscosity=lambda c: np.ones(len(c)), velocity=lambda p: np.zeros((len(p), 3)),
                          reaction=lambda p: np.ones(len(p)), source=lambda p: np.zeros(len(p)),
                          dirichlet=lambda p: np.where(p[:, 2] < 1e-12, 1.0, 0.0))
    part = partition_regular(mesh, (2, 2, 2))
    globs = classify_globs(mesh, part, mesh.boundary_nodes)
    system = assemble_system(mesh, coeffs)
    ops = [P.build_subdomain_operator(system, part, globs, i) for i in range(8)]
    scaling = P.build_scaling(globs, ops)
    theta_f = 1.0 + math.log(3.0)
    basis, _ = P.adaptive_primal_space(globs, ops, scaling, theta_f, 10.0, "old")
    pc = P.build_preconditioner(ops, basis, scaling)
    n = globs.interface_nodes.size
    Sd = torch.from_numpy(P.assemble_dense_schur(ops, n)).cuda()
    T = torch.stack([pc.apply_device(Sd[:, k].contiguous()) for k in range(n)], dim=1).cpu().numpy()
    lam = scipy.linalg.eigvals(T).real
    assert lam.min() >= 1.0 - 1e-8 and lam.max() <= 40.0 * max(theta_f, 10.0) ** 2
