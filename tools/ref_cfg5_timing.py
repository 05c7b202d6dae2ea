"""One-shot timing of the UNMODIFIED reference (baseline/_ref) on the full
bench workload (BASELINE configs[4], cfg5: 128^3 cells, 4,096 subdomains,
2,048,383 DOFs) on a GPU box's host cores, phase by phase, with the result
checked against the committed fixture.  Too long for bench.py's timed
region (~10 min, ~46 GB of host RAM); bench.py reports the committed JSON as
"cpu_reference_same_config".

    python tools/ref_cfg5_timing.py [--threads T] [--out profiles/ref_cfg5_timing_r02.json]
"""

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ref_cfg5_timing_r02.json"))
    args = ap.parse_args()
    from threadpoolctl import threadpool_limits

    import bench
    from adbddc.adaptive import adaptive_primal_space
    from adbddc.scaling import build_scaling
    from adbddc.solver import (build_preconditioner, gmres_solve, interface_operator, interface_rhs,
                               recover_interior)
    from adbddc.substructuring import build_subdomain_operator

    t0 = time.perf_counter()
    prob = bench.cpu_sample_problem(5, None, None)
    case = bench.ReferenceCase(prob)
    t_pre = time.perf_counter() - t0
    part, globs, system = case.part, case.globs, case.system
    ph = {}
    with threadpool_limits(limits=args.threads):
        t = time.perf_counter()
        ops = [build_subdomain_operator(system, part, globs, i) for i in range(part.n_subdomains)]
        ph["subdomain_ops"] = time.perf_counter() - t
        t = time.perf_counter()
        scaling = build_scaling(globs, ops)
        ph["scaling"] = time.perf_counter() - t
        t = time.perf_counter()
        for op in ops:
            op.bsym_inverse()
        ph["bsym_inverse"] = time.perf_counter() - t
        t = time.perf_counter()
        n = globs.interface_nodes.shape[0]
        operator = interface_operator(ops, n)
        rhs = interface_rhs(ops, n)
        basis, _ = adaptive_primal_space(globs, ops, scaling, 10.0, 10.0, "new")
        ph["gevp"] = time.perf_counter() - t
        t = time.perf_counter()
        pc = build_preconditioner(ops, basis, scaling)
        ph["pc_setup"] = time.perf_counter() - t
        t = time.perf_counter()
        rep = gmres_solve(operator, rhs, pc)
        ph["gmres"] = time.perf_counter() - t
        t = time.perf_counter()
        recover_interior(ops, globs, system, rep.solution)
        ph["recover"] = time.perf_counter() - t
    total = sum(ph.values())
    g = np.load(os.path.join(ROOT, "tests", "golden", "cfg5.npz"))
    rel = float(np.linalg.norm(rep.solution - g["new_solution"]) / np.linalg.norm(g["new_solution"]))
    out = {
        "what": "unmodified reference (baseline/_ref) hot path on the full cfg5 workload "
                "(the bench config), one run on the GPU box's host",
        "value": prob.n_dofs / total, "unit": "DOF/s", "seconds": total, "phases_s": ph,
        "threads": args.threads, "host_cpus": os.cpu_count(), "cpu": platform.processor() or platform.machine(),
        "iterations": rep.iterations, "pnumF": basis.pnumF, "pnumE": basis.pnumE,
        "solution_rel_diff_vs_fixture": rel, "input_build_s_untimed": t_pre,
    }
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
