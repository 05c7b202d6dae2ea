"""Shared test inputs: the golden cases rebuilt with the package's own
host preprocessing (mesh / partition / globs / element blocks), which the
fixtures' generator built with the reference's functions; tests pin that
both produce identical inputs."""

import functools
import math
import os

import numpy as np

from paper_2501_01676_b200 import configs
from paper_2501_01676_b200.decomposition import classify_globs, partition_regular
from paper_2501_01676_b200.discretization import Coefficients, assemble_system
from paper_2501_01676_b200.mesh import box_mesh

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
EX_DOMAIN = ((-0.5, 0.5), (-0.5, 0.5), (0.0, 1.0))


def rotating_coefficients(viscosity):
    """The reference harness example (reference harness.py:41-57)."""
    return Coefficients(
        viscosity=viscosity,
        velocity=lambda p: np.column_stack([-2.0 * np.pi * p[:, 1], 2.0 * np.pi * p[:, 0],
                                            np.sin(2.0 * np.pi * p[:, 0])]),
        reaction=lambda p: np.ones(len(p)),
        source=lambda p: np.zeros(len(p)),
        dirichlet=lambda p: np.where(p[:, 2] < 1e-12, 1.0, 0.0),
    )


def const_coefficients(nu=1.0, a=(0.0, 0.0, 0.0), c=1.0):
    a = np.asarray(a, dtype=float)
    return Coefficients(viscosity=lambda cent: np.full(len(cent), nu),
                        velocity=lambda p: np.tile(a, (len(p), 1)),
                        reaction=lambda p: np.full(len(p), c),
                        source=lambda p: np.zeros(len(p)),
                        dirichlet=lambda p: np.zeros(len(p)))


@functools.lru_cache(maxsize=None)
def inputs(name):
    """(system, partition, globs) for a golden case name."""
    if name == "jump":
        mesh = box_mesh(EX_DOMAIN, (8, 8, 8))
        part = partition_regular(mesh, (2, 2, 2))
        globs = classify_globs(mesh, part, mesh.boundary_nodes)
        system = assemble_system(mesh, rotating_coefficients(
            lambda cent: np.where(cent[:, 0] < 0.0, 1e-1, 1e-5)))
        return system, part, globs
    if name == "sym":
        mesh = box_mesh(((0.0, 1.0),) * 3, (6, 6, 6))
        part = partition_regular(mesh, (2, 2, 2))
        globs = classify_globs(mesh, part, mesh.boundary_nodes)
        return assemble_system(mesh, const_coefficients()), part, globs
    kw = {"cfg1": (1, {}), "cfg1_lnH": (1, {}), "cfg2": (2, {}), "cfg2_lnH": (2, {}),
          "cfg3": (3, {}), "cfg4": (4, {}), "cfg5": (5, {}), "cfg4_small": (4, dict(n=16, subs=24)),
          "cfg5_small": (5, dict(n=24, subs=3))}[name]
    p = configs.build_problem(kw[0], **kw[1])
    return p.system, p.partition, p.globs


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))


def probe_vector(g):
    """The seeded S_hat / M^-1 probe of a fixture (stored in full, or, for the
    lean cfg5 fixture, regenerated from its seed as make_golden.py drew it)."""
    if "probe" in g:
        return g["probe"]
    return np.random.default_rng(7).standard_normal(int(g["n_hat"]))


def variants(g):
    return [v for v in ("new", "old") if f"{v}_iterations" in g]


def gevp_values(g, v):
    """{glob index: eigenvalues} from a fixture."""
    ids, lens, vals = g[f"{v}_gevp_ids"], g[f"{v}_gevp_len"], g[f"{v}_gevp_vals"]
    out, off = {}, 0
    for k, n in zip(ids.tolist(), lens.tolist()):
        out[k] = vals[off:off + n]
        off += n
    return out


def counts_match(n_primal, ref_n_primal, eig, ref_eig, theta_of):
    """Per-glob primal counts equal, except globs with a finite eigenvalue
    within 1e-8 relative of the threshold (north_star exception)."""
    bad = []
    for k in range(len(ref_n_primal)):
        if int(n_primal[k]) == int(ref_n_primal[k]):
            continue
        th = theta_of(k)
        ev = ref_eig.get(k, np.zeros(0))
        ev = ev[np.isfinite(ev)]
        if ev.size and np.min(np.abs(ev / th - 1.0)) <= 1e-8:
            continue
        bad.append(k)
    return bad


FIXTURES = [n for n in ("cfg1", "cfg1_lnH", "cfg2", "cfg2_lnH", "cfg4_small", "cfg5_small", "jump", "cfg3", "cfg4",
                        "cfg5")
            if os.path.exists(os.path.join(GOLDEN, f"{n}.npz"))]
