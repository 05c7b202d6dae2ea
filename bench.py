"""Benchmark: BDDC-GMRES DOFs/s (setup + solve) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]
                    [--config 5] [--n N --subs S]

One step = the whole hot path on one problem: symbolic plan (index maps, on
the device), local assembly and Schur
elimination, Bsym^-1, deluxe scaling, face and new-edge GEPs with their
change of basis, preconditioner setup with the coarse LU, left-preconditioned
GMRES (rtol 1e-8) and interior recovery.  ``value`` is with element blocks,
connectivity, partition and Dirichlet data resident in HBM; ``e2e`` starts
from host (numpy) arrays through the package API and includes the
host->device copies and the device->host copy of the nodal solution.  Workload (BASELINE.json configs[4]): 128^3 cells (6 Kuhn tets /
cell, 2,048,383 DOFs), 16^3 subdomains (H/h = 8), nu = 1e-2, b = (1,1,1),
f = 1, c = 1, Theta = 10.  Working set (~50 GB) >> L2, so no flush is needed.
The last timed step's counts, iterations and solution are checked against
the unmodified reference's cfg5 fixture (tests/golden/cfg5.npz): "parity".

``--gpus N`` without a torchrun environment re-executes itself under
``torch.distributed.run`` with N ranks (one per GPU; fails if fewer GPUs are
visible); the subdomains of the one problem are sharded over the ranks.

``--impl reference``: the UNMODIFIED reference package (installed at
baseline/_ref, driven through its own API in the harness order,
harness.py:250-292) on a bounded sample of the same workload (same H/h,
coefficients and thresholds; 48^3 cells, 6^3 subdomains by default) on this
host's cores; under torchrun only rank 0 runs it.  If baseline/_ref is
missing, the oracle port (oracle/bddc_oracle.py) stands in and the line says
so ("kind": "port").
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BDDC-GMRES DOFs/s (setup+solve)"
THETA = 10.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--subs", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # reference arm sample (timed steps) and my arm's cpu_baseline sample
    ap.add_argument("--sample-n", type=int, default=48)
    ap.add_argument("--sample-subs", type=int, default=6)
    ap.add_argument("--cpu-sample-n", type=int, default=32)
    ap.add_argument("--cpu-sample-subs", type=int, default=4)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_desc(cfg, n, subs, prob, world=1):
    return {
        "workload": f"BASELINE configs[{cfg - 1}]: unit cube {n}^3 cells x 6 Kuhn tets, "
                    f"{prob.partition.n_subdomains} subdomains (H/h={prob.H_over_h}), theta_F=theta_E={THETA:g}, "
                    "new edge GEP, left-preconditioned full GMRES rtol 1e-8, c=1",
        "dofs": int(prob.n_dofs),
        "n_subdomains": int(prob.partition.n_subdomains),
        "n_hat": int(prob.globs.interface_nodes.size),
        "l2": "working set (~GBs of dense subdomain matrices) > 126 MB L2; no flush",
        "host": "Python cyclic GC paused inside each timed step (collected between steps)",
        "parallelism": ("subdomain batch on one GPU" if world == 1 else
                        f"subdomains sharded over {world} GPUs (contiguous blocks); glob eigenproblems by "
                        "first-sharer rank with point-to-point exchange of cross-rank glob blocks; "
                        "interface halo exchange (NCCL send/recv), owned-entry dot allreduces, coarse "
                        "rhs reduced to GPU 0 (single coarse factor) and solution broadcast"),
    }


# ---------------------------------------------------------------------------
# CPU reference timing (reference arm and cpu_baseline)
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def cpu_sample_problem(cfg, sample_n, sample_subs):
    from paper_2501_01676_b200 import configs
    return configs.build_problem(cfg, n=sample_n, subs=sample_subs)


def reference_available():
    return os.path.isdir(os.path.join(REF_DIR, "adbddc"))


class ReferenceCase:
    """The unmodified reference package (baseline/_ref) on one problem: inputs
    built once with the reference's own mesh / partition / glob / assembly
    functions from the config's coefficient callables (not timed), then the
    hot path through its public API in the harness order (harness.py:250-292)
    plus recover_interior."""

    def __init__(self, prob):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import adbddc.decomposition as rd
        import adbddc.discretization as rdi
        import adbddc.mesh as rm
        mesh = rm.box_mesh(prob.mesh.box, prob.mesh.cells)
        self.part = rd.Partition(prob.partition.subdomain_of.copy(), prob.partition.n_subdomains)
        self.globs = rd.classify_globs(mesh, self.part, mesh.boundary_nodes)
        c = prob.coeffs
        self.system = rdi.assemble_system(mesh, rdi.Coefficients(
            viscosity=c.viscosity, velocity=c.velocity, reaction=c.reaction, source=c.source,
            dirichlet=c.dirichlet))
        self.n_dofs = prob.n_dofs

    def run(self):
        from adbddc.adaptive import adaptive_primal_space
        from adbddc.scaling import build_scaling
        from adbddc.solver import (build_preconditioner, gmres_solve, interface_operator,
                                   interface_rhs, recover_interior)
        from adbddc.substructuring import build_subdomain_operator
        part, globs, system = self.part, self.globs, self.system
        ops = [build_subdomain_operator(system, part, globs, i) for i in range(part.n_subdomains)]
        scaling = build_scaling(globs, ops)
        for op in ops:
            op.bsym_inverse()
        n = globs.interface_nodes.shape[0]
        operator = interface_operator(ops, n)
        rhs = interface_rhs(ops, n)
        basis, _ = adaptive_primal_space(globs, ops, scaling, THETA, THETA, "new")
        pc = build_preconditioner(ops, basis, scaling)
        rep = gmres_solve(operator, rhs, pc)
        recover_interior(ops, globs, system, rep.solution)
        return {"iterations": rep.iterations, "pnumF": basis.pnumF, "pnumE": basis.pnumE}


class OracleCase:
    """Fallback when baseline/_ref is absent: the oracle port (test infrastructure)."""

    def __init__(self, prob):
        self.prob, self.n_dofs = prob, prob.n_dofs

    def run(self):
        from oracle import bddc_oracle as O
        p = self.prob
        return O.run_pipeline(p.system, p.partition, p.globs, THETA, THETA, "new")


def cpu_case(prob):
    if reference_available():
        return ReferenceCase(prob), "reference"
    return OracleCase(prob), "port"


def time_case(case, threads):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        res = case.run()
        dt = time.perf_counter() - t0
    return dt, res


def best_threads(case):
    """(threads, seconds): the faster of 1 BLAS thread and all host cores."""
    ncpu = os.cpu_count() or 1
    t1, _ = time_case(case, 1)
    if ncpu == 1:
        return 1, t1
    tn, _ = time_case(case, ncpu)
    return (1, t1) if t1 <= tn else (ncpu, tn)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:  # under torchrun only rank 0 runs the CPU reference arm
        return
    prob = cpu_sample_problem(args.config, args.sample_n, args.sample_subs)
    case, kind = cpu_case(prob)
    # warm-up on the sample also picks the BLAS thread count (1 vs all cores)
    threads, _ = best_threads(case)
    for _ in range(max(args.warmup - 2, 0)):
        time_case(case, threads)
    times = []
    for _ in range(args.steps):
        dt, res = time_case(case, threads)
        times.append(dt)
    tstep = sum(times) / len(times)
    value = prob.n_dofs / tstep
    what = ("unmodified reference package (baseline/_ref, adbddc API in harness order)" if kind == "reference"
            else "oracle port of the reference hot path (baseline/_ref missing)")
    sample = (f"{what} on {args.sample_n}^3 cells, {args.sample_subs}^3 subdomains with "
              f"configs[{args.config - 1}]'s H/h, coefficients and thresholds ({prob.n_dofs} DOFs, "
              f"{res['iterations']} iterations); hot path only (inputs built once, untimed)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tstep * 1e3,
        "ms_each_step": [round(t * 1e3, 1) for t in times],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(workload_desc(args.config, args.sample_n, args.sample_subs, prob),
                       parallelism=f"host CPU, {threads} BLAS thread(s) (no GPU)"),
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampling
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def fp64_peak():
    """Measured FP64 DMMA peak (tools/fp64_peak.cu on this pool's B200; not in
    MEASURED_PEAKS.json, which has HBM and bf16 only)."""
    path = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
    try:
        d = json.load(open(path))
        return max(v["dmma_m8n8k4_tflops"] for k, v in d.items() if k.startswith("tpb")), "measured DMMA m8n8k4 (profiles/fp64_peak_r01.json)"
    except (OSError, ValueError, KeyError):
        return 37.0, "fallback: DMMA m8n8k4 measured 37.1 TF/s on B200"


def trailing_traffic():
    """DRAM bytes per trailing-update launch from the committed ncu capture
    (tools/traffic.py -> profiles/trailing_traffic_*.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "trailing_traffic_*.json")))
    if not files:
        return None, None
    d = json.load(open(files[-1]))
    return d["traffic_bytes_per_launch"], (f"{os.path.basename(files[-1])}: dram read+write per "
                                          f"launch, mean over {d['mode0_launches']} launches of "
                                          f"one cfg5 step (ncu --set full)")


def hbm_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def parity_check(cfg, args, res):
    """Counts, iterations and solution of the last timed step against the
    unmodified reference's fixture of this workload (north_star bars: per-glob
    primal counts exact except eigenvalues within 1e-8 of theta, iterations
    +-1, solution relative difference <= 1e-8)."""
    path = os.path.join(ROOT, "tests", "golden", f"cfg{cfg}.npz")
    if args.n is not None or args.subs is not None or not os.path.exists(path):
        return {"status": "no fixture for this workload"}
    g = np.load(path)
    v = "new"
    ref_np = g[f"{v}_n_primal"]
    mine = np.asarray(res.n_primal)[:ref_np.size]
    ids, lens, vals = g[f"{v}_gevp_ids"], g[f"{v}_gevp_len"], g[f"{v}_gevp_vals"]
    starts = np.concatenate([[0], np.cumsum(lens)])
    ev_of = {int(k): vals[starts[j]:starts[j + 1]] for j, k in enumerate(ids)}
    bad = []
    for k in np.flatnonzero(mine != ref_np):
        ev = ev_of.get(int(k), np.zeros(0))
        ev = ev[np.isfinite(ev)]
        if not (ev.size and np.min(np.abs(ev / THETA - 1.0)) <= 1e-8):
            bad.append(int(k))
    x = res.solution.cpu().numpy()
    xr = g[f"{v}_solution"]
    rel = float(np.linalg.norm(x - xr) / np.linalg.norm(xr))
    it_ok = abs(res.iterations - int(g[f"{v}_iterations"])) <= 1
    tot_ok = (res.pnumF, res.pnumE, res.n_vertex) == (int(g[f"{v}_pnumF"]), int(g[f"{v}_pnumE"]),
                                                      int(g[f"{v}_n_vertex"]))
    ok = it_ok and tot_ok and not bad and rel <= 1e-8
    return {"status": "ok" if ok else "FAIL", "fixture": f"tests/golden/cfg{cfg}.npz (unmodified reference)",
            "iterations": [int(res.iterations), int(g[f"{v}_iterations"])],
            "pnum_FEV": [res.pnumF, res.pnumE, res.n_vertex],
            "glob_count_mismatches": len(bad), "solution_rel_diff": rel}


def reference_cfg5_timing():
    """One-shot timing of the unmodified reference on the full cfg5 workload
    on a GPU box's host (tools/ref_cfg5_timing.py -> profiles/), if committed."""
    path = os.path.join(ROOT, "profiles", "ref_cfg5_timing_r02.json")
    try:
        return json.load(open(path))
    except (OSError, ValueError):
        return None


def run_mine(args):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    from paper_2501_01676_b200 import build as _build
    _build.build()
    from paper_2501_01676_b200 import configs, pipeline
    from paper_2501_01676_b200._lib import lib
    from paper_2501_01676_b200.engine import trailing_flops, upload_inputs

    cfg = args.config
    t0 = time.perf_counter()
    prob = configs.build_problem(cfg, n=args.n, subs=args.subs, device="cuda")
    t_pre = time.perf_counter() - t0
    n_cells = prob.mesh.cells[0]
    comm, owned = None, None
    if world > 1:
        # strong scaling: the subdomains of the one problem are sharded over the ranks
        from paper_2501_01676_b200.dist import TorchComm
        comm = TorchComm()
        owned = comm.owned(prob.partition.n_subdomains)
    inputs = upload_inputs(prob.system, prob.partition, owned=owned)
    torch.cuda.synchronize()

    def step(kernel_timing=False, keep=False):
        # the symbolic plan (index maps) is rebuilt inside every step
        return pipeline.run(prob.system, prob.partition, prob.globs, THETA, THETA, "new",
                            inputs=inputs, kernel_timing=kernel_timing, keep=keep, comm=comm)

    import gc

    clocks = ClockSampler(local)
    nwarm = max(args.warmup, 3)
    for i in range(nwarm):
        if i == nwarm - 1:  # nvidia-smi spins up during the last warm-up step
            clocks.start()
        res = step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    from paper_2501_01676_b200.engine import GRAPH_STATS
    lib.bddc_launch_count_reset()
    g0 = dict(GRAPH_STATS)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    lib.bddc_trailing_log(1)  # CUDA events around the trailing launches (pool created here)
    # the Python cyclic GC stays off inside the timed region (a collection
    # mid-step stalls the host that feeds the GPU); it runs between regions
    gc.collect()
    gc.disable()
    torch.cuda.synchronize()
    e0.record()
    phases = {}
    step_ev = [e0]
    per_step_phases = []
    for _ in range(args.steps):
        res = step()
        per_step_phases.append({k: round(v, 2) for k, v in res.times_ms.items()})
        for k, v in res.times_ms.items():
            phases[k] = phases.get(k, 0.0) + v / args.steps
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        step_ev.append(ev)
    e1.record()
    torch.cuda.synchronize()
    gc.enable()
    if world > 1:
        torch.distributed.barrier()
    launches = (int(lib.bddc_launch_count()) - (GRAPH_STATS["captured"] - g0["captured"])
                + (GRAPH_STATS["replayed"] - g0["replayed"])) // args.steps
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms_each = [round(step_ev[i].elapsed_time(step_ev[i + 1]), 3) for i in range(args.steps)]
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    dofs = prob.n_dofs
    value = dofs / (ms * 1e-3)

    lib.bddc_trailing_log(0)
    t_ms, t_n = ctypes.c_double(0.0), ctypes.c_longlong(0)
    lib.bddc_trailing_collect(ctypes.cast(ctypes.pointer(t_ms), ctypes.c_void_p),
                              ctypes.cast(ctypes.pointer(t_n), ctypes.c_void_p))
    trail_ms = [t_ms.value / args.steps]

    # apply-path bandwidth: one M^-1 and one S_hat application (HBM bound)
    keep = step(keep=True)
    plan = keep.ls.plan
    pc, op = keep.pc, keep.op
    n_vec = keep.ls.n_loc  # rank-local interface vector length (n_hat on one GPU)
    r = torch.randn(n_vec, dtype=torch.float64, device="cuda")
    out = torch.empty_like(r)
    for _ in range(3):
        pc.apply_device(r, out)
        op.apply_device(r, out)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    a0.record()
    for _ in range(reps):
        op.apply_device(r, out)
    a1.record()
    torch.cuda.synchronize()
    op_ms = a0.elapsed_time(a1) / reps
    a0.record()
    for _ in range(reps):
        pc.apply_device(r, out)
    a1.record()
    torch.cuda.synchronize()
    pc_ms = a0.elapsed_time(a1) / reps
    nB = plan.nB.astype(np.int64)
    op_bytes = 8 * int((nB * nB).sum()) + 8 * (3 * int(nB.sum()) + n_vec)
    npn = pc.np_sub.astype(np.int64)
    nd = nB - npn
    slot_ng2 = int((plan.gsize[plan.sub_globs].astype(np.int64) ** 2).sum())
    # SURVEY 8(d) B_apply_local (dual LU, Phi/primal rows, (Q D) glob blocks at both
    # ends, vectors) + the coarse block-inverse operators read by the coarse solve
    pc_local_bytes = 8 * int((nd * nd).sum() + 2 * (nd * npn).sum() + 2 * slot_ng2) \
        + 8 * (6 * int(nB.sum()) + 4 * n_vec)
    coarse_bytes = pc.coarse_factor_bytes
    pc_bytes = pc_local_bytes + coarse_bytes
    coarse_ms = 0.0
    if pc.root:  # the coarse factor lives on rank 0 only
        a0.record()
        for _ in range(reps):
            pc.coarse_solve(pc.rp, pc.up)
        a1.record()
        torch.cuda.synchronize()
        coarse_ms = a0.elapsed_time(a1) / reps
    del keep, pc, op

    # e2e through the host API: the problem's inputs live in page-locked host
    # buffers (stage_inputs, outside the timed region, like a caller's own
    # data); every step: H2D of those buffers -> plan -> solve -> D2H of u
    from paper_2501_01676_b200.engine import stage_inputs, staged_bytes, upload_staged
    sysm = prob.system
    staged = stage_inputs(sysm, prob.partition, owned=owned)
    h2d = staged_bytes(staged)
    u_pinned = torch.empty(sysm.mesh.n_nodes, dtype=torch.float64, pin_memory=True)
    e2e_ms = []
    for i in range(args.e2e_steps + 1):  # the first (allocator warm-up) is not timed
        gc.collect()
        gc.disable()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        inp = upload_staged(staged)
        rr = pipeline.run(sysm, prob.partition, prob.globs, THETA, THETA, "new", inputs=inp,
                          comm=comm)
        u_pinned.copy_(rr.u)
        u_host = u_pinned.numpy()
        torch.cuda.synchronize()
        if i > 0:
            e2e_ms.append((time.perf_counter() - w0) * 1e3)
        gc.enable()
        del rr, inp
    e2e_step_ms = float(np.mean(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_step_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_step_ms = float(t.item())

    tflops, n_trail = trailing_flops(plan, dual_lu=True)
    tms = float(np.mean(trail_ms))
    if int(t_n.value) != n_trail * args.steps:
        raise RuntimeError(f"logged {t_n.value} trailing launches, expected {n_trail} x {args.steps}")
    peak, peak_src = fp64_peak()
    traffic, traffic_src = trailing_traffic()
    achieved = tflops / (tms * 1e-3) / 1e12
    hbm, hbm_src = hbm_peak()

    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_desc(cfg, n_cells, args.subs, prob, world),
        "roofline": {
            "kernel": "schur_trailing_kernel (batched trailing updates of the subdomain Schur "
                      "elimination and of the dual-block LU, DMMA m8n8k4)",
            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic,
            "traffic_source": traffic_src,
            "peak_source": peak_src,
            "algorithmic_flops_per_step": tflops, "launches_per_step": n_trail,
            "kernel_ms_per_step": tms,
            "share_of_step": tms / ms,
        },
        "apply": {
            "interface_operator_ms": op_ms, "interface_operator_GBps": op_bytes / (op_ms * 1e-3) / 1e9,
            "preconditioner_ms": pc_ms, "preconditioner_GBps": pc_bytes / (pc_ms * 1e-3) / 1e9,
            "hbm_peak_GBps": hbm, "hbm_peak_source": hbm_src,
            "interface_operator_frac": op_bytes / (op_ms * 1e-3) / 1e9 / hbm,
            "preconditioner_frac": pc_bytes / (pc_ms * 1e-3) / 1e9 / hbm,
            "preconditioner_bytes": pc_bytes,
            "coarse_solve_ms": coarse_ms, "coarse_operator_bytes": coarse_bytes,
            "bytes_formula": "SURVEY 8(d) B_apply_local + coarse block-inverse operator bytes; "
                             "B_op = 8 sum nB^2 + 8 (3 sum nB + n_hat)",
        },
        "phases_ms": phases, "ms_each_step": ms_each, "phases_each_step": per_step_phases,
        "iterations": res.iterations, "converged": bool(res.converged),
        "pnumF": res.pnumF, "pnumE": res.pnumE, "n_vertex": res.n_vertex, "n_c": res.n_c,
        "host_preprocessing_s": t_pre,
        "clocks": clk,
        "e2e": {"value": dofs / (e2e_step_ms * 1e-3), "unit": "DOF/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(u_host.nbytes),
                "ms_per_step": e2e_step_ms, "ms_each_step": [round(v, 3) for v in e2e_ms],
                "includes": "H2D from page-locked host buffers of the mesh nodes, connectivity, "
                            "viscosity table, partition and Dirichlet data; SUPG element blocks "
                            "built on the device; symbolic plan; full hot path; D2H of nodal u"},
        "gpu_launches": launches,
    }
    if rank == 0:
        line["parity"] = parity_check(cfg, args, res)
    if rank == 0 and not args.no_cpu_baseline:
        sp = cpu_sample_problem(cfg, args.cpu_sample_n, args.cpu_sample_subs)
        case, kind = cpu_case(sp)
        threads, t_best = best_threads(case)
        line["cpu_baseline"] = {
            "value": sp.n_dofs / t_best, "unit": "DOF/s", "cores": threads, "kind": kind,
            "sample": (f"{'unmodified reference (baseline/_ref)' if kind == 'reference' else 'oracle port'} "
                       f"hot path on {args.cpu_sample_n}^3 cells, {args.cpu_sample_subs}^3 subdomains, "
                       f"configs[{cfg - 1}] H/h/coefficients/thresholds, {sp.n_dofs} DOFs; best of 1 and "
                       f"{os.cpu_count()} BLAS threads"),
        }
        ref5 = reference_cfg5_timing()
        if ref5 is not None and cfg == 5 and args.n is None and args.subs is None:
            line["cpu_reference_same_config"] = ref5
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def spawn_ranks(args):
    """--gpus N outside torchrun: re-execute under torch.distributed.run with
    N ranks (one per GPU, rendezvous on 127.0.0.1)."""
    import socket

    if args.impl == "mine":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    rank, world, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
