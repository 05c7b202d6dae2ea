"""Householder form of the change of basis (precond.cu): the reflector
products keep every glob's primal span, are orthogonal, and the reflector
transform Sbar = Q S Q^T equals the dense block product with the same Q."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_reflector_basis_and_transform():
    import torch

    from paper_2501_01676_b200 import configs, pipeline
    from paper_2501_01676_b200._lib import lib, stream
    from paper_2501_01676_b200.engine import dev_i32, dev_i64
    from paper_2501_01676_b200.plan import _excl

    # low thresholds: several face and edge constraints per glob
    prob = configs.build_problem(2, n=16, subs=2)
    res = pipeline.run(prob.system, prob.partition, prob.globs, 1.05, 1.05, "new", keep=True)
    ls, ps = res.ls, res.space
    p, d, st = ls.plan, ls.d, stream()
    r = ps.r_host
    assert (r[p.kind != 2] > 1).any()
    Q0 = ps.Q.clone()
    Q = ps.Q.clone()
    HV = torch.zeros_like(Q)
    w_sz = np.where(p.kind == 2, 0, p.gsize.astype(np.int64) * np.minimum(r, p.gsize))
    w_off = _excl(w_sz)
    W = torch.empty(max(int(w_off[-1]), 1), dtype=torch.float64, device="cuda")
    q_off = ps.d_q_off
    r_d = dev_i32(r)
    assert lib.bddc_pc_glob_reflectors(d.kind, d.gsize, r_d, Q, q_off, HV, W,
                                       dev_i64(w_off[:-1]), p.G, int(p.gsize.max()), st) == 0
    torch.cuda.synchronize()
    qh, q0, hv = Q.cpu().numpy(), Q0.cpu().numpy(), HV.cpu().numpy()
    for g in range(p.G):
        n, k = int(p.gsize[g]), int(r[g])
        o = int(ps.q_off[g])
        A, A0 = qh[o:o + n * n].reshape(n, n), q0[o:o + n * n].reshape(n, n)
        np.testing.assert_allclose(A @ A.T, np.eye(n), atol=1e-13)
        if k == 0 or p.kind[g] == 2:
            continue
        # same primal span: the leading rows of the old basis lie in span(A[:k])
        P = A[:k].T @ A[:k]
        np.testing.assert_allclose(A0[:k] @ P, A0[:k], atol=1e-12)
        if n > 1:  # A = H_k ... H_1 with H_j = I - w_j w_j^T
            H = np.eye(n)
            for j in range(min(k, n)):
                w = hv[o + j * n:o + (j + 1) * n]
                H = (np.eye(n) - np.outer(w, w)) @ H
            np.testing.assert_allclose(H, A, atol=1e-13)
    # reflector transform vs the dense DMMA block transform with the same Q
    S = ls.S
    Sb1 = torch.empty_like(S)
    assert lib.bddc_pc_transform_refl(d.nB, d.soff, d.sub_glob_start, d.sub_globs, d.sub_glob_boff,
                                      d.kind, d.gsize, r_d, HV, q_off, S, Sb1, p.N, st) == 0
    Sb2 = torch.empty_like(S)
    tmp = torch.empty_like(S)
    QT = torch.empty_like(Q)
    nbmax = int(p.nB.max())
    max_globs = int(np.diff(p.sub_glob_start).max())
    assert lib.bddc_pc_transform_schur(d.nB, d.soff, d.sub_glob_start, p.N, d.sub_globs,
                                       d.sub_glob_boff, d.sub_glob_sh, d.gsize, Q, q_off, QT, p.G,
                                       int(p.sub_globs.size), nbmax, int(p.gsize.max()),
                                       max_globs, S, tmp, Sb2, st) == 0
    torch.cuda.synchronize()
    a, b = Sb1.cpu().numpy(), Sb2.cpu().numpy()
    assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()


def test_fused_transform_embed_matches_two_pass():
    """bddc_pc_transform_embed (Sbar, embedded dual block Z, compact primal
    rows / columns in one pass) equals the two-pass reflector transform +
    dual embedding + extraction."""
    import torch

    from paper_2501_01676_b200 import configs, pipeline
    from paper_2501_01676_b200._lib import lib, stream
    from paper_2501_01676_b200.engine import dev_i32, dev_i64
    from paper_2501_01676_b200.plan import _excl, _ranges

    prob = configs.build_problem(2, n=16, subs=2)
    res = pipeline.run(prob.system, prob.partition, prob.globs, 1.05, 1.05, "new", keep=True)
    ls, ps = res.ls, res.space
    p, d, st = ls.plan, ls.d, stream()
    r = ps.r_host
    Q = ps.Q.clone()
    HV = torch.zeros_like(Q)
    w_sz = np.where(p.kind == 2, 0, p.gsize.astype(np.int64) * np.minimum(r, p.gsize))
    w_off = _excl(w_sz)
    W = torch.empty(max(int(w_off[-1]), 1), dtype=torch.float64, device="cuda")
    r_d = dev_i32(r)
    lib.bddc_pc_glob_reflectors(d.kind, d.gsize, r_d, Q, ps.d_q_off, HV, W, dev_i64(w_off[:-1]),
                                p.G, int(p.gsize.max()), st)
    cnt = r[p.sub_globs]
    np_sub = np.add.reduceat(cnt, p.sub_glob_start[:-1].astype(np.int64))
    pstart = _excl(np_sub)
    ppos = _ranges(p.sub_glob_boff, cnt)
    psub = np.repeat(np.arange(p.N), np_sub)
    pidx = np.full(int(p.voff[-1]), -1, dtype=np.int32)
    pidx[p.voff[psub] + ppos] = (np.arange(ppos.size) - pstart[psub]).astype(np.int32)
    mask = (pidx >= 0).astype(np.uint8)
    poff = _excl(np_sub * p.nB)
    npn = int(poff[-1])
    S = ls.S
    f64 = dict(dtype=torch.float64, device="cuda")
    # two-pass reference
    Sbar = torch.empty_like(S)
    lib.bddc_pc_transform_refl(d.nB, d.soff, d.sub_glob_start, d.sub_globs, d.sub_glob_boff,
                               d.kind, d.gsize, r_d, HV, ps.d_q_off, S, Sbar, p.N, st)
    Z0 = torch.empty_like(S)
    lib.bddc_pc_dual_embed(d.nB, d.soff, d.voff, torch.from_numpy(mask).cuda(), Sbar, Z0, None,
                           p.N, st)
    Sr0, Sc0 = torch.empty(npn, **f64), torch.empty(npn, **f64)
    lib.bddc_pc_primal_extract(d.nB, d.soff, d.voff, dev_i32(pidx), dev_i64(poff[:-1]), Sbar, Sr0,
                               Sc0, p.N, st)
    # fused: left reflectors per reflected glob block, then the row pass
    Z1 = torch.empty_like(S)
    Sr1, Sc1 = torch.empty(npn, **f64), torch.empty(npn, **f64)
    gk = p.sub_globs.astype(np.int64)
    ks = np.flatnonzero((p.kind[gk] != 2) & (p.gsize[gk] > 1) & (r[gk] > 0))
    sub_of_k = np.repeat(np.arange(p.N), np.diff(p.sub_glob_start))
    refl_start = np.searchsorted(ks, p.sub_glob_start.astype(np.int64))
    lib.bddc_pc_transform_embed(d.nB, d.soff, d.voff, d.pos2k, d.sub_globs, d.sub_glob_boff,
                                d.kind, d.gsize, r_d, HV, ps.d_q_off, dev_i32(refl_start),
                                dev_i32(ks), dev_i32(ks), dev_i32(sub_of_k[ks]), int(ks.size),
                                dev_i32(pidx), dev_i64(poff[:-1]), S, Z1, Sr1, Sc1, p.N,
                                int(p.nB.max()), st)
    torch.cuda.synchronize()
    for a, b in ((Z1, Z0), (Sr1, Sr0), (Sc1, Sc0)):
        a, b = a.cpu().numpy(), b.cpu().numpy()
        assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()
