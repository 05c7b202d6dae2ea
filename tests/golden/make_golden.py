"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [case ...]

Inputs are built with the reference's own mesh / partition / glob /
assembly functions from the coefficient callables of
``paper_2501_01676_b200.configs`` (the BASELINE configs), then the reference
hot path runs unchanged: build_subdomain_operator, build_scaling,
bsym_inverse, adaptive_primal_space, build_preconditioner, gmres_solve,
recover_interior.  Each case writes ``tests/golden/<case>.npz`` with
per-glob eigenvalues and primal counts, pnumF/pnumE/n_vertex, iteration
counts, residual histories, the interface solution, the recovered nodal
solution, one preconditioner apply on a seeded vector and the dense S of a
few subdomains.  Nothing on the GPU box reads /root/reference; the tests
read only these committed fixtures.
"""

import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, REF)

import adbddc.adaptive as ra  # noqa: E402
import adbddc.decomposition as rd  # noqa: E402
import adbddc.discretization as rdi  # noqa: E402
import adbddc.harness as rh  # noqa: E402
import adbddc.mesh as rm  # noqa: E402
import adbddc.scaling as rs  # noqa: E402
import adbddc.solver as rsol  # noqa: E402
import adbddc.substructuring as rsub  # noqa: E402

from paper_2501_01676_b200 import configs  # noqa: E402


def ref_inputs_from_config(cfg, **kw):
    p = configs.build_problem(cfg, **kw)
    mesh = rm.box_mesh(p.mesh.box, p.mesh.cells)
    part = rd.Partition(p.partition.subdomain_of.copy(), p.partition.n_subdomains)
    globs = rd.classify_globs(mesh, part, mesh.boundary_nodes)
    c = p.coeffs
    coeffs = rdi.Coefficients(viscosity=c.viscosity, velocity=c.velocity, reaction=c.reaction,
                              source=c.source, dirichlet=c.dirichlet)
    system = rdi.assemble_system(mesh, coeffs)
    return mesh, part, globs, system, p


def ref_inputs_jump():
    """The reference test-suite's jump case (reference tests/test_coarse.py:46-51)."""
    mesh = rm.box_mesh(rh.EX_DOMAIN, (8, 8, 8))
    visc = lambda cent: np.where(cent[:, 0] < 0.0, 1e-1, 1e-5)
    part = rd.partition_regular(mesh, (2, 2, 2))
    globs = rd.classify_globs(mesh, part, mesh.boundary_nodes)
    system = rdi.assemble_system(mesh, rh.example_coefficients(visc))
    return mesh, part, globs, system, None


def run_reference(mesh, part, globs, system, theta_f, theta_e, variants, n_S=4, lean=False):
    """``lean`` (cfg5): the interface solution is stored in full; the long
    vectors (rhs, S_hat / M^-1 probes, nodal u) only at a seeded subsample
    of 20,000 entries (``sub_hat`` / ``sub_u``), to keep the fixture small."""
    out = {}
    t0 = time.perf_counter()
    ops = [rsub.build_subdomain_operator(system, part, globs, i) for i in range(part.n_subdomains)]
    t_ops = time.perf_counter()
    scaling = rs.build_scaling(globs, ops)
    for op in ops:
        op.bsym_inverse()
    out["ref_seconds_ops"] = t_ops - t0
    out["ref_seconds_scaling_binv"] = time.perf_counter() - t_ops
    n = globs.interface_nodes.shape[0]
    operator = rsol.interface_operator(ops, n)
    rhs = rsol.interface_rhs(ops, n)
    out["rhs"] = rhs
    out["n_hat"] = n
    out["nB"] = np.array([op.n_B for op in ops])
    out["nI"] = np.array([op.interior_nodes.size for op in ops])
    pick = np.unique(np.linspace(0, part.n_subdomains - 1, n_S).astype(int)) if n_S else np.zeros(0, int)
    out["S_ids"] = pick
    for i in pick:
        out[f"S_{i}"] = ops[i].S
        out[f"g_{i}"] = ops[i].g
        out[f"Binv_{i}"] = ops[i].bsym_inverse()
    rng = np.random.default_rng(7)
    probe = rng.standard_normal(n)
    Sprobe = operator(probe)
    if lean:
        sub_hat = np.sort(np.random.default_rng(11).choice(n, 20000, replace=False))
        sub_u = np.sort(np.random.default_rng(12).choice(mesh.n_nodes, 20000, replace=False))
        out["sub_hat"], out["sub_u"] = sub_hat, sub_u
        out["rhs"] = rhs[sub_hat]
        out["Sprobe"] = Sprobe[sub_hat]
    else:
        out["probe"] = probe
        out["Sprobe"] = Sprobe
    for variant in variants:
        ta = time.perf_counter()
        basis, reports = ra.adaptive_primal_space(globs, ops, scaling, theta_f, theta_e, variant)
        tb = time.perf_counter()
        pc = rsol.build_preconditioner(ops, basis, scaling)
        tc = time.perf_counter()
        rep = rsol.gmres_solve(operator, rhs, pc)
        td = time.perf_counter()
        u = rsol.recover_interior(ops, globs, system, rep.solution)
        v = variant
        out[f"{v}_ref_seconds"] = np.array([tb - ta, tc - tb, td - tc, time.perf_counter() - td])
        out[f"{v}_pnumF"] = basis.pnumF
        out[f"{v}_pnumE"] = basis.pnumE
        out[f"{v}_n_vertex"] = basis.n_vertex
        out[f"{v}_n_primal"] = np.array([k for _, k in basis.transforms])
        out[f"{v}_iterations"] = rep.iterations
        out[f"{v}_converged"] = rep.converged
        out[f"{v}_solution"] = rep.solution
        out[f"{v}_u"] = u[out["sub_u"]] if lean else u
        out[f"{v}_true_hist"] = np.array(rep.residual_history)
        out[f"{v}_pre_hist"] = np.array(rep.preconditioned_history)
        Mp = pc.apply(probe)
        out[f"{v}_Mprobe"] = Mp[out["sub_hat"]] if lean else Mp
        gl = {r.glob_id: r for r in reports}
        ids = sorted(gl, key=lambda s: int(s[1:]))
        out[f"{v}_gevp_ids"] = np.array([int(s[1:]) for s in ids])
        lens = np.array([gl[s].eigenvalues.size for s in ids])
        out[f"{v}_gevp_len"] = lens
        out[f"{v}_gevp_vals"] = np.concatenate([gl[s].eigenvalues for s in ids]) if ids else np.zeros(0)
        out[f"{v}_gevp_nsel"] = np.array([gl[s].n_primal for s in ids])
    out["ref_seconds"] = time.perf_counter() - t0
    return out


CASES = {
    # name: (input builder, theta_f, theta_e, variants)
    "cfg1": (lambda: ref_inputs_from_config(1), 10.0, 10.0, ("new", "old"), 4),
    "cfg1_lnH": (lambda: ref_inputs_from_config(1), 1.0 + math.log(4), 10.0, ("new",), 0),
    "cfg2": (lambda: ref_inputs_from_config(2), 10.0, 10.0, ("new",), 1),
    "cfg2_lnH": (lambda: ref_inputs_from_config(2), 1.0 + math.log(8), 10.0, ("new",), 0),
    "cfg4_small": (lambda: ref_inputs_from_config(4, n=16, subs=24), 10.0, 10.0, ("new",), 2),
    "cfg5_small": (lambda: ref_inputs_from_config(5, n=24, subs=3), 10.0, 10.0, ("new",), 1),
    "jump": (ref_inputs_jump, 1.0 + math.log(4), 10.0, ("new", "old"), 8),
    "cfg3": (lambda: ref_inputs_from_config(3), 10.0, 10.0, ("new",), 0),
    "cfg4": (lambda: ref_inputs_from_config(4), 10.0, 10.0, ("new",), 0),
    # the bench workload (BASELINE configs[4]): ~500 s and ~46 GB of host RAM
    "cfg5": (lambda: ref_inputs_from_config(5), 10.0, 10.0, ("new",), 0),
}
LEAN = {"cfg5"}


def main(names):
    for name in names:
        build, tf, te, variants, n_S = CASES[name]
        mesh, part, globs, system, _ = build()
        res = run_reference(mesh, part, globs, system, tf, te, variants, n_S, lean=name in LEAN)
        res["theta_f"] = tf
        res["theta_e"] = te
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **res)
        summ = ", ".join(f"{v}: {res[f'{v}_iterations']}({res[f'{v}_pnumF']},{res[f'{v}_pnumE']})"
                         for v in variants)
        print(f"{name}: N={part.n_subdomains} n_hat={res['n_hat']} {summ} "
              f"[{res['ref_seconds']:.1f}s] -> {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main(sys.argv[1:] or [k for k in CASES if k not in ("cfg3", "cfg4", "cfg5")])
