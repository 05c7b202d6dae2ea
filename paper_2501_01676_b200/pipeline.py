"""End-to-end hot path on the device, with per-phase CUDA-event timings.

Same phases as the reference harness (harness.py:250-292) plus interior
recovery: subdomain operators -> deluxe scaling -> Bsym^-1 -> adaptive
primal space -> preconditioner -> GMRES -> recover_interior.
"""

import time

import numpy as np
import torch

from .engine import (DeviceInterfaceOperator, DevicePreconditioner, DevicePrimalSpace,
                     DeviceScaling, LocalSystem, PhaseTimer, gmres_device, gmres_right_device,
                     _side_stream, device_element_blocks, recover_device, upload_inputs)
from .plan import Plan


class Result:
    pass


def run(system, partition, globs, theta_f, theta_e, variant="new", rel_tol=1e-8, max_iter=300,
        plan=None, inputs=None, timings=True, keep=False, kernel_timing=False,
        dplan=None, comm=None, side="left", restart=200, general=False):
    """Run the whole hot path; returns a Result with counts, solutions
    (device tensors) and phase times in ms (CUDA events).

    comm (dist.py): shard the subdomains over its ranks (each rank passes
    its own comm; results are replicated on every rank).
    general: face / edge eigenproblems by the reference algorithm verbatim
    (no certified fast paths)."""
    tm = PhaseTimer(timings)
    owned = None
    if comm is not None and comm.size > 1:
        owned = plan.owned if plan is not None else comm.owned(partition.n_subdomains)
    if inputs is None:
        inputs = upload_inputs(system, partition, owned=owned if plan is None or plan.on_device else None)
    if "Ke" not in inputs and "_supg" in inputs:
        # device element blocks first: the kernel runs while the host builds the plan
        if inputs.get("_late") is not None:
            # staged upload (engine.upload_staged): the nodes / viscosity table are
            # still in flight on the copy stream; the element kernel follows them
            # there, next to the plan's device work, and LocalSystem waits for it
            cur, aux = torch.cuda.current_stream(), _side_stream()
            inputs["conn"].record_stream(aux)
            with torch.cuda.stream(aux):
                Ke, Fe, ebad = device_element_blocks(inputs)
                for t in (Ke, Fe, ebad):
                    t.record_stream(cur)
                done = torch.cuda.Event()
                done.record(aux)
            inputs = {**inputs, "Ke": Ke, "Fe": Fe, "_ebad": ebad, "_late": done}
        else:
            Ke, Fe, ebad = device_element_blocks(inputs)
            inputs = {**inputs, "Ke": Ke, "Fe": Fe, "_ebad": ebad}
    if plan is None:
        tm.mark("symbolic_plan")
        plan = Plan(system, partition, globs, device_inputs=inputs, owned=owned)
    tm.mark("subdomain_ops")
    ls = LocalSystem(system, partition, globs, plan=plan, inputs=inputs,
                     kernel_timing=kernel_timing, dplan=dplan, comm=comm)
    inputs = None
    # the status checks of Bsym^-1 and of the scaling are read at the first
    # synchronisation of the GEP phase: the host keeps queueing meanwhile
    tm.mark("bsym_inverse")
    ls.bsym_inverse(check=False)
    tm.mark("scaling")
    sc = DeviceScaling(ls, check=False)
    tm.mark("gevp")
    ps = DevicePrimalSpace(ls, sc, theta_f, theta_e, variant, general=general)
    tm.mark("pc_setup")
    pc = DevicePreconditioner(ls, sc, ps.r_host, ps.Q, ps.d_q_off)
    op = DeviceInterfaceOperator(ls)
    tm.mark("gmres")
    rhs = op.rhs_local()
    if side == "left":  # the reference's full left-preconditioned GMRES
        it, conv, x, th, ph = gmres_device(op, rhs, pc, rel_tol, max_iter)
    else:  # right-preconditioned GMRES(restart), BASELINE.json's variant
        it, conv, x, th, ph = gmres_right_device(op, rhs, pc, rel_tol, max_iter, restart)
    tm.mark("recover")
    u = recover_device(ls, x)
    tm.mark("end")
    res = Result()
    kinds = plan.kind
    r = ps.r_host
    res.iterations, res.converged = it, conv
    res.solution, res.u = ls.layout.to_global(x), u  # solution: global, replicated on every rank
    res.solution_local = x
    res.true_hist, res.pre_hist = th, ph
    res.pnumF = int(r[kinds == 0].sum())
    res.pnumE = int(r[kinds == 1].sum())
    res.n_vertex = int(r[kinds == 2].sum())
    res.n_c = int(r.sum())
    res.n_primal = r
    res.n_sel = ps.n_sel_host
    res.times_ms = tm.result()
    res.trailing_ms = ls.trailing_ms
    if keep:
        res.ls, res.scaling, res.space, res.pc, res.op = ls, sc, ps, pc, op
    return res
