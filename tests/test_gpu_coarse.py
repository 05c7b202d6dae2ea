"""Coarse envelope LU and the solve kernels (grid-barrier, dataflow, block-inverse)
against a dense solve, on a coarse matrix with the structure the
preconditioner builds (subdomain cliques of primal dofs, reverse
Cuthill-McKee order, many 128-row super-panels)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_sub,seed", [(300, 0), (37, 1), (900, 2), (2000, 3)])
def test_coarse_solves_match_dense(n_sub, seed):
    import torch

    from paper_2501_01676_b200._lib import lib, stream
    from paper_2501_01676_b200.engine import (coarse_blockinv_layout, coarse_ordering, dev_i32,
                                              dev_i64)

    rng = np.random.default_rng(seed)
    # chain of subdomains, each sharing primal dofs with its neighbours
    per = rng.integers(3, 9, size=n_sub)
    starts = np.concatenate([[0], np.cumsum(per)])
    n = int(starts[-1]) + 5
    cliques = []
    for s in range(n_sub):
        own = list(range(starts[s], starts[s + 1]))
        nb = list(range(starts[s + 1], min(n, starts[s + 1] + 3)))
        far = list(rng.choice(n, size=2, replace=False)) if s % 50 == 0 else []
        cliques.append(np.unique(np.array(own + nb + far, dtype=np.int64)))
    np_sub = np.array([c.size for c in cliques])
    pgid = np.concatenate(cliques)
    order, new_id, lim, first = coarse_ordering(pgid, np_sub, n)
    C = np.zeros((n, n))
    for c in cliques:
        k = c.size
        B = rng.standard_normal((k, k)) * 0.3 + np.eye(k) * (k + 1.0)
        C[np.ix_(new_id[c], new_id[c])] += B
    C[np.arange(n), np.arange(n)] += 1.0  # dofs in no clique (the +5 tail)
    b = rng.standard_normal(n)
    x_ref = np.linalg.solve(C, b)

    Cd = torch.from_numpy(C.ravel().copy()).cuda()
    steps = (n + 63) // 64
    pinv = torch.empty(steps * 4096, dtype=torch.float64, device="cuda")
    piv = torch.zeros(n, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    lim_c = (ctypes.c_int * steps)(*lim.tolist())
    st = stream()
    lib.bddc_coarse_factor(Cd, dev_i64([0]), dev_i32([n]), dev_i32([n]), n,
                           ctypes.cast(lim_c, ctypes.c_void_p), pinv, piv, status, st)
    assert int(status.item()) == 0
    # grid-barrier solve
    rb = torch.from_numpy(b.copy()).cuda()
    x1 = torch.empty(n, dtype=torch.float64, device="cuda")
    lib.bddc_coarse_solve(Cd, n, n, pinv, 4096, dev_i32(lim), dev_i32(first), rb, x1, st)
    # dataflow solve, twice (epochs)
    nq = (n + 127) // 128
    l64 = lim.astype(np.int64)
    lsup = np.maximum.accumulate(np.array([l64[min(2 * q + 1, l64.size - 1)] for q in range(nq)]))
    q = np.arange(nq)
    jmin = np.minimum(np.searchsorted(lsup, 128 * q, side="right"), q)
    jmax = np.maximum((lsup - 1) // 128, q)
    flags = torch.zeros(2 * nq, dtype=torch.int32, device="cuda")
    for epoch in (1, 2):
        rb2 = torch.from_numpy(b.copy()).cuda()
        x2 = torch.empty(n, dtype=torch.float64, device="cuda")
        lib.bddc_coarse_solve_flow(Cd, n, n, pinv, 4096, dev_i32(jmin), dev_i32(jmax), rb2, x2,
                                   flags, epoch, st)
        torch.cuda.synchronize()
        e2 = np.linalg.norm(x2.cpu().numpy() - x_ref) / np.linalg.norm(x_ref)
        assert e2 <= 1e-12, e2
    e1 = np.linalg.norm(x1.cpu().numpy() - x_ref) / np.linalg.norm(x_ref)
    assert e1 <= 1e-12, e1
    # block-inverse operators (coarse.cu), three successive solves (epochs)
    lay = coarse_blockinv_layout(lim, n)
    F = torch.empty(int(lay["foff"][-1]), dtype=torch.float64, device="cuda")
    G = torch.empty(int(lay["goff"][-1]), dtype=torch.float64, device="cuda")
    cl, cu = dev_i32(lay["cl"]), dev_i32(lay["cu"])
    foff, goff = dev_i64(lay["foff"][:-1]), dev_i64(lay["goff"][:-1])
    assert lib.bddc_coarse_blockinv(Cd, n, n, pinv, 4096, lay["nD"], cl, cu, foff, goff,
                                    lay["max_ldf"], lay["max_ldg"], F, G, st) == 0
    cnt = torch.zeros(2 * lay["nD"], dtype=torch.int32, device="cuda")
    zb = torch.empty(n, dtype=torch.float64, device="cuda")
    for epoch in (1, 2, 3):
        rhs = rng.standard_normal(n)
        x3 = torch.empty(n, dtype=torch.float64, device="cuda")
        assert lib.bddc_coarse_solve_blockinv(F, G, n, lay["nD"], cl, cu, foff, goff,
                                              torch.from_numpy(rhs).cuda(), zb, x3, cnt, epoch,
                                              st) == 0
        torch.cuda.synchronize()
        xr = np.linalg.solve(C, rhs)
        e3 = np.linalg.norm(x3.cpu().numpy() - xr) / np.linalg.norm(xr)
        assert e3 <= 1e-12, (epoch, e3)
    # timing (informational)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    for _ in range(10):
        lib.bddc_coarse_solve(Cd, n, n, pinv, 4096, dev_i32(lim), dev_i32(first), rb, x1, st)
    ev[1].record()
    for e in range(10):
        lib.bddc_coarse_solve_flow(Cd, n, n, pinv, 4096, dev_i32(jmin), dev_i32(jmax), rb2, x2,
                                   flags, 10 + e, st)
    ev[2].record()
    for e in range(10):
        lib.bddc_coarse_solve_blockinv(F, G, n, lay["nD"], cl, cu, foff, goff, rb2, zb, x3, cnt,
                                       4 + e, st)
    ev[3].record()
    torch.cuda.synchronize()
    print(f"n={n} (nD={lay['nD']}, F+G {8 * (lay['foff'][-1] + lay['goff'][-1]) / 1e6:.1f} MB): "
          f"barrier solve {ev[0].elapsed_time(ev[1]) / 10:.3f} ms, "
          f"dataflow solve {ev[1].elapsed_time(ev[2]) / 10:.3f} ms, "
          f"block-inverse solve {ev[2].elapsed_time(ev[3]) / 10:.3f} ms")
