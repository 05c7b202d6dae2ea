"""Stage-by-stage comparison of the CUDA path with golden fixtures (prints, no asserts)."""
import sys
import time
import traceback

import numpy as np
import torch

sys.path.insert(0, ".")
from tests.cases import gevp_values, golden, inputs, variants  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main(names):
    from paper_2501_01676_b200 import pipeline
    from paper_2501_01676_b200.substructuring import SubdomainOperator
    for name in names:
        g = golden(name)
        system, part, globs = inputs(name)
        for v in variants(g):
            try:
                t0 = time.time()
                res = pipeline.run(system, part, globs, float(g["theta_f"]), float(g["theta_e"]), v, keep=True)
                torch.cuda.synchronize()
                print(f"== {name} {v}: wall {time.time()-t0:.2f}s times {res.times_ms}")
                ls = res.ls
                for i in g["S_ids"].tolist()[:2]:
                    op = SubdomainOperator(ls, i)
                    print(f"  S[{i}] rel {rel(op.S, g[f'S_{i}']):.2e}  g {rel(op.g, g[f'g_{i}']):.2e}  Binv {rel(op.bsym_inverse(), g[f'Binv_{i}']):.2e}")
                print(f"  rhs {rel(res.op.rhs_device().cpu().numpy(), g['rhs']):.2e}  Sprobe {rel(res.op(g['probe']), g['Sprobe']):.2e}")
                ref_eig = gevp_values(g, v)
                mine = res.space.all_eigenvalues()
                worst, wk = 0.0, None
                for k, ev in ref_eig.items():
                    if mine.get(k) is None or mine[k].shape != ev.shape:
                        print("  shape mismatch", k); continue
                    fin = np.isfinite(ev)
                    e = np.max(np.abs(mine[k][fin] - ev[fin]) / np.maximum(np.abs(ev[fin]), 1e-300), initial=0)
                    if e > worst: worst, wk = e, k
                print(f"  eig worst rel {worst:.2e} at glob {wk}")
                bad = np.flatnonzero(res.n_primal != g[f"{v}_n_primal"])
                print(f"  n_primal mismatches {bad[:10]} (mine {res.n_primal[bad[:10]]} ref {g[f'{v}_n_primal'][bad[:10]]})")
                print(f"  counts mine {(res.pnumF, res.pnumE, res.n_vertex)} ref {(int(g[f'{v}_pnumF']), int(g[f'{v}_pnumE']), int(g[f'{v}_n_vertex']))}")
                print(f"  iters mine {res.iterations} ref {int(g[f'{v}_iterations'])}; pre_hist {res.pre_hist[-3:]} ref {g[f'{v}_pre_hist'][-3:]}")
                print(f"  Mprobe {rel(res.pc.apply(g['probe']), g[f'{v}_Mprobe']):.2e}")
                print(f"  solution {rel(res.solution.cpu().numpy(), g[f'{v}_solution']):.2e}  u {rel(res.u.cpu().numpy(), g[f'{v}_u']):.2e}")
            except Exception:
                traceback.print_exc()


if __name__ == "__main__":
    main(sys.argv[1:] or ["jump", "cfg1", "cfg1_lnH", "cfg4_small", "cfg5_small", "cfg2", "cfg2_lnH"])
