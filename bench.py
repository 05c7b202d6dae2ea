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

``--impl reference``: the CPU oracle (restated reference algorithm, same
LAPACK/SuperLU calls) on a bounded sample of the same workload (same H/h,
coefficients and thresholds, 4^3 subdomains), on this host's cores.
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
    ap.add_argument("--sample-n", type=int, default=32)
    ap.add_argument("--sample-subs", type=int, default=4)
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
        "parallelism": ("subdomain batch on one GPU" if world == 1 else
                        f"subdomains sharded over {world} GPUs (contiguous blocks), glob eigenproblems by "
                        "first-sharer rank, NCCL sum-allreduce exchanges, coarse LU replicated"),
    }


# ---------------------------------------------------------------------------
# CPU oracle timing (reference arm and cpu_baseline)
# ---------------------------------------------------------------------------

def cpu_sample_problem(cfg, sample_n, sample_subs):
    from paper_2501_01676_b200 import configs
    return configs.build_problem(cfg, n=sample_n, subs=sample_subs)


def time_oracle(prob, threads):
    from threadpoolctl import threadpool_limits

    from oracle import bddc_oracle as O
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        res = O.run_pipeline(prob.system, prob.partition, prob.globs, THETA, THETA, "new")
        dt = time.perf_counter() - t0
    return dt, res


def best_threads(prob):
    ncpu = os.cpu_count() or 1
    t1, _ = time_oracle(prob, 1)
    if ncpu == 1:
        return 1, t1
    tn, _ = time_oracle(prob, ncpu)
    return (1, t1) if t1 <= tn else (ncpu, tn)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:  # under torchrun only rank 0 runs the CPU reference arm
        return
    prob = cpu_sample_problem(args.config, args.sample_n, args.sample_subs)
    threads, _ = best_threads(prob)
    for _ in range(max(args.warmup - 1, 0)):
        time_oracle(prob, threads)
    times = []
    for _ in range(args.steps):
        dt, res = time_oracle(prob, threads)
        times.append(dt)
    tstep = sum(times) / len(times)
    value = prob.n_dofs / tstep
    sample = (f"oracle (restated reference hot path, numpy/scipy LAPACK+SuperLU) on a "
              f"{args.sample_n}^3-cell, {args.sample_subs}^3-subdomain problem with configs[{args.config - 1}]'s "
              f"H/h, coefficients and thresholds ({prob.n_dofs} DOFs, {res['iterations']} iterations)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tstep * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(workload_desc(args.config, args.sample_n, args.sample_subs, prob),
                       parallelism=f"host CPU, {threads} BLAS thread(s) (no GPU)"),
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": threads, "kind": "port",
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
    prob = configs.build_problem(cfg, n=args.n, subs=args.subs)
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
    r = torch.randn(plan.n_hat, dtype=torch.float64, device="cuda")
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
    op_bytes = 8 * int((nB * nB).sum()) + 8 * (3 * int(nB.sum()) + plan.n_hat)
    npn = pc.np_sub.astype(np.int64)
    nd = nB - npn
    slot_ng2 = int((plan.gsize[plan.sub_globs].astype(np.int64) ** 2).sum())
    # SURVEY 8(d) B_apply_local (dual LU, Phi/primal rows, (Q D) glob blocks at both
    # ends, vectors) + the coarse block-inverse operators read by the coarse solve
    pc_local_bytes = 8 * int((nd * nd).sum() + 2 * (nd * npn).sum() + 2 * slot_ng2) \
        + 8 * (6 * int(nB.sum()) + 4 * plan.n_hat)
    coarse_bytes = pc.coarse_factor_bytes
    pc_bytes = pc_local_bytes + coarse_bytes
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
    if rank == 0 and not args.no_cpu_baseline:
        sp = cpu_sample_problem(cfg, args.sample_n, args.sample_subs)
        threads, t_best = best_threads(sp)
        line["cpu_baseline"] = {
            "value": sp.n_dofs / t_best, "unit": "DOF/s", "cores": threads, "kind": "port",
            "sample": (f"CPU oracle (restated reference hot path) on {args.sample_n}^3 cells, "
                       f"{args.sample_subs}^3 subdomains, configs[{cfg - 1}] H/h/coefficients/thresholds, "
                       f"{sp.n_dofs} DOFs; best of 1 and {os.cpu_count()} BLAS threads"),
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_mine(args)


if __name__ == "__main__":
    main()
