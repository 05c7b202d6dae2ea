import sys; sys.path.insert(0, '.')
import numpy as np, torch
from tests.cases import inputs, golden
from paper_2501_01676_b200 import pipeline
from paper_2501_01676_b200.dist import run_threads
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4_small"
size = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = golden(name); system, part, globs = inputs(name)
th_f, th_e = float(g["theta_f"]), float(g["theta_e"])
single = pipeline.run(system, part, globs, th_f, th_e, "new", keep=True)
p1 = single.ls.plan
S1 = single.ls.S.cpu().numpy(); B1 = single.ls.bsym_inverse().cpu().numpy(); g1 = single.ls.g.cpu().numpy()
e1 = single.space.all_eigenvalues()
def rank(comm):
    res = pipeline.run(system, part, globs, th_f, th_e, "new", keep=True, comm=comm)
    p = res.ls.plan
    return (p.owned, res.ls.S.cpu().numpy(), res.ls.bsym_inverse().cpu().numpy(), p.soff.copy(), p.nB.copy(), res.space.all_eigenvalues(), p.nDeep.copy(), p.nI.copy())
outs = run_threads(size, rank)
for owned, S, B, soff, nB, eig, nd, nI in outs:
    s0, s1 = owned
    for i in range(s1 - s0):
        n = int(nB[i]); a = int(soff[i]); b1 = int(p1.soff[s0 + i])
        dS = np.abs(S[a:a+n*n] - S1[b1:b1+n*n]).max() / np.abs(S1[b1:b1+n*n]).max()
        dB = np.abs(B[a:a+n*n] - B1[b1:b1+n*n]).max() / np.abs(B1[b1:b1+n*n]).max()
        if dS > 0 or dB > 0:
            print(f"sub {s0+i}: nB {n} nI {nI[i]} nDeep {nd[i]} (single nDeep {p1.nDeep[s0+i]}) dS {dS:.2e} dB {dB:.2e}")
eig = outs[0][5]
for k in e1:
    d = np.abs(eig[k] - e1[k]); f = np.isfinite(e1[k])
    if f.any() and (d[f] / np.maximum(np.abs(e1[k][f]), 1e-300)).max() > 1e-12:
        print("glob", k, "max rel eig diff", (d[f] / np.abs(e1[k][f])).max())
print("done")
