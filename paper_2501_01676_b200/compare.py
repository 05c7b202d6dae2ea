"""Old-vs-new edge-eigenproblem comparison (the paper's tables; reference
harness.py:186-201 ResultRow, :250-292 _run_problem, :310-361 emit_tables /
format_table / parse_results_csv), on the device path.

``compare_variants`` runs both primal-space variants on one problem with the
subdomain operators, Bsym^-1 and deluxe scaling shared (the reference charges
them to setup once, harness.py:259-263) and returns one ``ResultRow`` per
variant; ``format_table`` renders the side-by-side ``iters(pnumF,pnumE)``
table with the variant's eigenproblem + solve time, ``emit_tables`` writes
results.csv / results.txt in the reference's column layout.
"""

import csv
import time
from dataclasses import dataclass
from pathlib import Path

import torch

CSV_HEADER = ("case", "variant", "N", "m", "iters", "pnumF", "pnumE", "setup_s", "gevp_s",
              "solve_s", "converged")


@dataclass
class ResultRow:
    case: str
    variant: str
    N: int
    m: int
    iters: int
    pnumF: int
    pnumE: int
    setup_s: float
    gevp_s: float
    solve_s: float
    converged: bool

    def cell(self):
        return f"{self.iters}({self.pnumF},{self.pnumE})"


def compare_variants(system, partition, globs, theta_f, theta_e, label, m=0,
                     variants=("old", "new"), rel_tol=1e-8, max_iter=300):
    """Both variants on one problem; times are wall seconds with the device
    synchronised at each phase boundary."""
    from .engine import (DeviceInterfaceOperator, DevicePreconditioner, DevicePrimalSpace,
                         DeviceScaling, LocalSystem, gmres_device)

    def now():
        torch.cuda.synchronize()
        return time.perf_counter()

    t0 = now()
    ls = LocalSystem(system, partition, globs)
    ls.bsym_inverse()
    sc = DeviceScaling(ls)
    op = DeviceInterfaceOperator(ls)
    rhs = op.rhs_device()
    setup_s = now() - t0
    rows = []
    for v in variants:
        t1 = now()
        ps = DevicePrimalSpace(ls, sc, theta_f, theta_e, v)
        t2 = now()
        pc = DevicePreconditioner(ls, sc, ps.r_host, ps.Q, ps.d_q_off)
        it, conv, _, _, _ = gmres_device(op, rhs, pc, rel_tol, max_iter)
        t3 = now()
        kinds = ls.plan.kind
        r = ps.r_host
        rows.append(ResultRow(label, v, int(partition.n_subdomains), int(m), int(it),
                              int(r[kinds == 0].sum()), int(r[kinds == 1].sum()), setup_s,
                              t2 - t1, t3 - t2, bool(conv)))
        del pc, ps
    return rows


def format_table(rows):
    """One line per problem: iters(pnumF,pnumE) per variant and that variant's
    eigenproblem + solve time; unconverged cells are starred."""
    order, table = [], {}
    for r in rows:
        key = (r.case, r.N, r.m)
        if key not in table:
            order.append(key)
            table[key] = {}
        table[key][r.variant] = r
    head = ("case", "N", "m", "old", "t_old[s]", "new", "t_new[s]")
    body = []
    for key in order:
        cells = [key[0], str(key[1]), str(key[2])]
        for v in ("old", "new"):
            r = table[key].get(v)
            cells += (["-", "-"] if r is None else
                      [r.cell() + ("" if r.converged else "*"), f"{r.gevp_s + r.solve_s:.2f}"])
        body.append(cells)
    width = [max(len(line[i]) for line in [head, *body]) for i in range(len(head))]
    out = ["  ".join(c.ljust(w) for c, w in zip(line, width)).rstrip() for line in [head, *body]]
    text = "\n".join(out)
    if not all(r.converged for r in rows):
        text += "\n(* did not reach the residual tolerance)"
    return text + "\n"


def emit_tables(rows, out_dir):
    """results.csv + results.txt (reference column layout)."""
    if not rows:
        raise ValueError("no result rows to emit")
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    path = out / "results.csv"
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(CSV_HEADER)
        for r in rows:
            w.writerow([r.case, r.variant, r.N, r.m, r.iters, r.pnumF, r.pnumE, f"{r.setup_s:.3f}",
                        f"{r.gevp_s:.3f}", f"{r.solve_s:.3f}", "true" if r.converged else "false"])
    txt = out / "results.txt"
    txt.write_text(format_table(rows))
    return path, txt


def parse_results_csv(path):
    with open(path, newline="") as f:
        return [ResultRow(d["case"], d["variant"], int(d["N"]), int(d["m"]), int(d["iters"]),
                          int(d["pnumF"]), int(d["pnumE"]), float(d["setup_s"]), float(d["gevp_s"]),
                          float(d["solve_s"]), d["converged"] == "true")
                for d in csv.DictReader(f)]


__all__ = ["CSV_HEADER", "ResultRow", "compare_variants", "emit_tables", "format_table",
           "parse_results_csv"]
