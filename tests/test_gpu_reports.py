"""GevpReport fields and PrimalBasis helpers of the drop-in API on the
reference test-suite's jump case (reference tests/test_coarse.py:46-144,
:424-444; adaptive.py:36-47, :190-285): every eigenpair of every glob pencil
satisfies the reference's residual bound, the selection and the constraint
rows are consistent with the eigenvalues, the detail eigenvalues equal the
golden fixture, and the basis helpers reproduce the reference's numbering."""

import math

import numpy as np
import pytest
import scipy.linalg

from tests.cases import gevp_values, golden, inputs

pytestmark = pytest.mark.gpu

THETA_F = 1.0 + math.log(4.0)


def _space(variant):
    import paper_2501_01676_b200 as P

    system, part, globs = inputs("jump")
    ops = [P.build_subdomain_operator(system, part, globs, i) for i in range(part.n_subdomains)]
    scaling = P.build_scaling(globs, ops)
    basis, reports = P.adaptive_primal_space(globs, ops, scaling, THETA_F, 10.0, variant)
    return globs, ops, scaling, basis, reports


@pytest.mark.parametrize("variant", ["old", "new"])
def test_report_pencil_residuals_and_selection(variant):
    globs, ops, scaling, basis, reports = _space(variant)
    g = golden("jump")
    ref = gevp_values(g, variant)
    ids = {globs.glob_id(gl): k for k, gl in enumerate(globs.globs)}
    checked = 0
    for rep in reports:
        B, Bt = rep.pencil_left, rep.pencil_right
        n = rep.eigenvalues.size
        assert B.shape == Bt.shape == rep.vectors.shape == (n, n)
        nb, nt = np.linalg.norm(B), np.linalg.norm(Bt)
        for lam, v, deg in zip(rep.eigenvalues, rep.vectors.T, rep.degenerate):
            nv = np.linalg.norm(v)
            if deg:
                assert np.linalg.norm(B @ v) <= 1e-9 * nb * nv
                assert np.linalg.norm(Bt @ v) <= 1e-9 * nt * nv
            elif np.isinf(lam):
                assert np.linalg.norm(Bt @ v) <= 1e-9 * nt * nv
            else:
                assert np.linalg.norm(B @ v - lam * (Bt @ v)) <= 1e-9 * (nb + abs(lam) * nt) * nv
            checked += 1
        mask = (rep.eigenvalues >= (THETA_F if rep.variant == "face" else 10.0)) & ~rep.degenerate
        assert rep.n_primal == int(mask.sum())
        assert rep.constraint_matrix.shape == (rep.n_primal, n)
        np.testing.assert_allclose(rep.constraint_matrix, (B @ rep.vectors[:, mask]).T,
                                   rtol=1e-12, atol=1e-12 * max(nb, 1.0) * max(np.abs(rep.vectors).max(), 1.0))
        fin = np.isfinite(rep.eigenvalues)
        ev = ref[ids[rep.glob_id]]
        np.testing.assert_allclose(rep.eigenvalues[fin], ev[np.isfinite(ev)], rtol=1e-8,
                                   atol=1e-10 * np.abs(ev[np.isfinite(ev)]).max(initial=1.0))
        if rep.variant != "edge_new" and n and np.linalg.eigvalsh(Bt).min() > 1e-8 * nt:
            lam = scipy.linalg.eigh(B, Bt, eigvals_only=True)
            np.testing.assert_allclose(np.sort(lam)[::-1], rep.eigenvalues, rtol=1e-8, atol=1e-10)
    assert checked > 0


def test_change_of_basis_and_assembly_helpers():
    from paper_2501_01676_b200.adaptive import (assemble_primal_space, build_change_of_basis,
                                                reduce_edge_constraints)

    globs, ops, scaling, basis, reports = _space("new")
    rng = np.random.default_rng(3)
    rows = rng.standard_normal((3, 7))
    rows[2] = rows[0] + rows[1]  # dependent row is dropped
    Q, r = build_change_of_basis(7, rows)
    assert r == 2
    np.testing.assert_allclose(Q @ Q.T, np.eye(7), atol=1e-13)
    # rows lie in span(Q[:r])
    assert np.linalg.norm(rows - rows @ Q[:r].T @ Q[:r]) <= 1e-12 * np.linalg.norm(rows)
    assert build_change_of_basis(5, np.zeros((0, 5)))[1] == 0
    with pytest.raises(ValueError):
        build_change_of_basis(4, np.ones((1, 5)))
    rep_map = {rep.glob_id: rep for rep in reports}
    for rep in reports:
        if rep.variant == "edge_new" and rep.n_primal:
            red = reduce_edge_constraints(rep)
            stacked = rep.constraint_matrix.reshape(-1, rep.n_dofs)
            assert np.linalg.norm(stacked - stacked @ red.T @ red) <= 1e-10 * np.linalg.norm(stacked)
    rebuilt = assemble_primal_space(rep_map, globs, "new")
    assert (rebuilt.pnumF, rebuilt.pnumE, rebuilt.n_vertex) == (basis.pnumF, basis.pnumE, basis.n_vertex)
    for (Qa, ka), (Qb, kb) in zip(rebuilt.transforms, basis.transforms):
        assert ka == kb
        if ka:  # same primal span
            assert np.linalg.norm(Qa[:ka] - Qa[:ka] @ Qb[:kb].T @ Qb[:kb]) <= 1e-8


def test_primal_basis_numbering_helpers():
    globs, ops, scaling, basis, reports = _space("old")
    glob_pos = [globs.interface_index(g.nodes) for g in globs.globs]
    total = 0
    for op in ops:
        ent = basis.glob_entries(op)
        assert all(op.sub_id in g.sharers for g, *_ in ent)
        Qi = basis.subdomain_transform(op)
        np.testing.assert_allclose(Qi @ Qi.T, np.eye(op.n_B), atol=1e-12)
        loc, gids = basis.subdomain_primal(op)
        assert loc.size == gids.size
        total += loc.size
        for g, Q, k, idx, off in ent:
            assert np.array_equal(loc[np.isin(gids, np.arange(off, off + k))], idx[:k])
    assert total >= basis.n_primal_total
    u = np.random.default_rng(5).standard_normal(globs.interface_nodes.size)
    v = basis.apply_interface(glob_pos, u)
    back = basis.apply_interface(glob_pos, v, transpose=True)
    np.testing.assert_allclose(back, u, atol=1e-12)
    for (Q, _), pos in zip(basis.transforms, glob_pos):
        np.testing.assert_allclose(v[pos], Q @ u[pos], atol=1e-12)
