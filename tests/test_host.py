"""CPU tests of the host side: C-ABI exports, symbolic plan, coarse ordering
and envelope (no GPU needed)."""

import ctypes
import subprocess

import numpy as np
import pytest

from tests.cases import inputs


def test_library_exports_header():
    from paper_2501_01676_b200 import build
    from paper_2501_01676_b200._lib import LIB_PATH, parse_header

    build.build()
    sigs = parse_header()
    assert len(sigs) >= 30
    dll = ctypes.CDLL(LIB_PATH)  # loads without a GPU
    out = subprocess.check_output(["nm", "-D", "--defined-only", LIB_PATH]).decode()
    exported = {ln.split()[-1] for ln in out.splitlines()}
    missing = [name for name in sigs if name not in exported]
    assert missing == []
    for name in sigs:
        getattr(dll, name)


def test_workspace_formulas_match_library():
    from paper_2501_01676_b200 import build, engine
    from paper_2501_01676_b200._lib import LIB_PATH

    build.build()
    dll = ctypes.CDLL(LIB_PATH)
    dll.bddc_ws_face.restype = ctypes.c_longlong
    dll.bddc_ws_face.argtypes = [ctypes.c_longlong]
    dll.bddc_ws_edge_new.restype = ctypes.c_longlong
    dll.bddc_ws_edge_new.argtypes = [ctypes.c_longlong] * 4
    dll.bddc_ws_face_fast.restype = ctypes.c_longlong
    dll.bddc_ws_face_fast.argtypes = [ctypes.c_longlong]
    for n in (1, 7, 49, 193):
        assert dll.bddc_ws_face(n) == int(engine._face_ws(n))
        assert dll.bddc_ws_face_fast(n) == int(engine._face_fast_ws(n))
    for ns, ne, wd, h in ((2, 7, 30, 8), (4, 7, 80, 14), (3, 20, 700, 150)):
        assert dll.bddc_ws_edge_new(ns, ne, wd, h) == int(engine._edge_new_ws(ns, ne, wd, h))


@pytest.mark.parametrize("name", ["jump", "cfg1", "cfg4_small"])
def test_plan_local_numbering(name):
    from paper_2501_01676_b200.plan import Plan

    system, part, globs = inputs(name)
    p = Plan(system, part, globs)
    el = system.mesh.elements
    for i in range(p.N):
        elems = np.flatnonzero(part.subdomain_of == i)
        nodes = np.unique(el[elems])
        free = system.node_to_free[nodes] >= 0
        iface = np.isin(nodes, globs.interface_nodes)
        ref_B = np.sort(nodes[free & iface])
        ref_I = nodes[free & ~iface]
        B = p.B_nodes[p.voff[i]:p.voff[i + 1]]
        assert np.array_equal(np.sort(B), ref_B)
        # interior: deep nodes (no element shared with an interface node) first,
        # each group in ascending node order; nDeep = even number of leading deep dofs
        I = p.I_nodes[p.ioff[i]:p.ioff[i + 1]]
        assert np.array_equal(np.sort(I), ref_I)
        touch = np.isin(el[elems], globs.interface_nodes).any(axis=1)
        shell = np.isin(I, np.unique(el[elems][touch]))
        n_deep = int((~shell).sum())
        assert not shell[:n_deep].any() and shell[n_deep:].all()
        assert np.array_equal(I[:n_deep], np.sort(I[:n_deep]))
        assert np.array_equal(I[n_deep:], np.sort(I[n_deep:]))
        assert p.nDeep[i] == n_deep - (n_deep & 1)
        ref_I = I
        # glob-major: every glob of the subdomain is one contiguous block
        for k in range(p.sub_glob_start[i], p.sub_glob_start[i + 1]):
            g = globs.globs[p.sub_globs[k]]
            bo = p.sub_glob_boff[k]
            assert np.array_equal(B[bo:bo + g.size], g.nodes)
        # element-local indices point at the right nodes
        e0, e1 = p.elem_start[i], p.elem_start[i + 1]
        ids = p.elem_ids[e0:e1]
        order = np.concatenate([ref_I, B])
        loc = p.loc4[ids]
        conn = el[ids]
        inside = loc < p.nL[i]
        assert np.array_equal(order[loc[inside]], conn[inside])
        assert np.all(system.node_to_free[conn[~inside]] < 0)
    # interface CSR covers every local interface entry once
    assert p.tstart[-1] == p.voff[-1]
    assert np.array_equal(np.sort(p.tsrc), np.arange(p.voff[-1]))


def _envelope_solve(C, lim, first):
    n = C.shape[0]
    A = C.copy()
    P = []
    for k in range(0, n, 64):
        w = min(64, n - k)
        L = min(n, lim[k // 64])
        Pk = np.linalg.inv(A[k:k + w, k:k + w])
        P.append(Pk)
        A[k:k + w, k + w:L] = Pk @ A[k:k + w, k + w:L]
        A[k + w:L, k + w:L] -= A[k + w:L, k:k + w] @ A[k:k + w, k + w:L]
        A[k + w:L, k:k + w] = A[k + w:L, k:k + w] @ Pk   # L' = A21 P_k (panel_scale_kernel)
    return A, P


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_coarse_envelope_exact(seed):
    """The coarse envelope LU / solve schedule (engine.coarse_ordering,
    csrc coarse_factor / coarse_solve) equals a dense solve."""
    from paper_2501_01676_b200.engine import coarse_ordering

    rng = np.random.default_rng(seed)
    N, n_c = 64, 300 + 70 * seed
    np_sub = rng.integers(3, 12, size=N)
    pgid = np.concatenate([rng.choice(n_c, size=k, replace=False) for k in np_sub])
    pgid = np.concatenate([pgid, np.arange(n_c)])
    np_sub = np.concatenate([np_sub, np.ones(n_c, dtype=np.int64)])
    C = np.zeros((n_c, n_c))
    off = 0
    for k in np_sub:
        g = pgid[off:off + k]
        off += k
        X = rng.standard_normal((k, k))
        C[np.ix_(g, g)] += X @ X.T + k * np.eye(k) + 0.3 * (X - X.T)
    order, new_id, lim, first = coarse_ordering(pgid, np_sub, n_c)
    assert np.array_equal(order[new_id], np.arange(n_c))
    Cn = C[np.ix_(order, order)]
    A, P = _envelope_solve(Cn, lim, first)
    b = rng.standard_normal(n_c)
    bb, t = b.copy(), np.zeros(n_c)
    for k in range(0, n_c, 64):      # forward with L' (coarse_solve_coop_kernel)
        w = min(64, n_c - k)
        L = min(n_c, lim[k // 64])
        bb[k + w:L] -= A[k + w:L, k:k + w] @ bb[k:k + w]
    for k in range(0, n_c, 64):      # t = blockdiag(P) b
        w = min(64, n_c - k)
        t[k:k + w] = P[k // 64] @ bb[k:k + w]
    for k in range(((n_c - 1) // 64) * 64, 0, -64):
        w = min(64, n_c - k)
        f = first[k // 64]
        t[f:k] -= A[f:k, k:k + w] @ t[k:k + w]
    x = np.linalg.solve(Cn, b)
    assert np.abs(t - x).max() <= 1e-12 * np.abs(x).max()


@pytest.mark.parametrize("config", [1, 2, 3, 4, 5])
def test_device_fields_reproduce_coefficient_callables(config):
    """The affine fields handed to the device element kernel evaluate to the
    same velocity / viscosity as the host callables of every BASELINE config."""
    from paper_2501_01676_b200 import configs

    n = 8
    prob = configs.build_problem(config, n=n, subs=2 if config != 4 else 16)
    c = prob.coeffs
    df = c.device_fields
    rng = np.random.default_rng(config)
    pts = rng.uniform(0.0, 1.0, size=(50, 3))
    a_host = np.asarray(c.velocity(pts), dtype=float)
    a_dev = pts @ np.asarray(df.velocity_matrix).T + np.asarray(df.velocity_offset)
    np.testing.assert_allclose(a_dev, a_host, rtol=0, atol=1e-15)
    assert np.all(np.asarray(c.reaction(pts)) == df.reaction)
    assert np.all(np.asarray(c.source(pts)) == df.source)
    m = prob.mesh.n_elements
    nu_dev = np.asarray(df.viscosity_table)[np.arange(m) % df.viscosity_period]
    np.testing.assert_array_equal(nu_dev, prob.system.viscosity)


@pytest.mark.parametrize("name", ["jump", "cfg1", "cfg4_small"])
def test_native_glob_tables_match_numpy(name, monkeypatch):
    """csrc/plan_host.cu (bddc_plan_glob_tables) builds the same glob tables as
    the numpy reference path of plan.py."""
    from paper_2501_01676_b200 import build
    from paper_2501_01676_b200 import plan as P

    build.build()
    system, part, globs = inputs(name)
    a = P.Plan(system, part, globs)
    monkeypatch.setattr(P, "NATIVE_GLOB_TABLES", False)
    b = P.Plan(system, part, globs)
    for k in ("sh_start", "sh_sub", "slot_glob", "sh_doff", "sub_globs", "sub_glob_sh",
              "sub_glob_start", "sub_glob_boff", "sh_boff", "nB", "voff", "_B_starts", "_B_counts",
              "B_nodes", "pos2k", "iface_perm", "loc4", "I_nodes"):
        assert np.array_equal(np.asarray(getattr(a, k)), np.asarray(getattr(b, k))), k
    assert a.d_total == b.d_total and a._B_range == b._B_range
