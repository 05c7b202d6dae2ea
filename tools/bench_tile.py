"""Microbenchmark of the batched Schur elimination (DMMA tile GEMM) on
cfg5-shaped matrices: 4096 x [729 x 730] (343 pivots), random diagonally
dominant.  Usage: python tools/bench_tile.py [lib.so ...]"""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_01676_b200 import _lib  # noqa: E402
import os  # noqa: E402
PANEL = int(os.environ.get("PANEL", "128"))


def run(path, N=4096, nI=343, nB=386, reps=3):
    dll = ctypes.CDLL(path)
    sigs = _lib.parse_header()
    f = dll.bddc_schur_eliminate_timed
    f.restype, f.argtypes = sigs["bddc_schur_eliminate_timed"]
    g = dll.bddc_gj_inverse
    g.restype, g.argtypes = sigs["bddc_gj_inverse"]
    nL = nI + nB
    ld = (nL + 2) // 2 * 2
    off = torch.arange(N, dtype=torch.int64, device="cuda") * nL * ld
    M0 = torch.rand(N, nL, ld, dtype=torch.float64, device="cuda")
    M0 += 4 * nL * torch.eye(nL, ld, dtype=torch.float64, device="cuda")
    i32 = lambda v: torch.full((N,), v, dtype=torch.int32, device="cuda")
    pinv = torch.empty(N * 4096, dtype=torch.float64, device="cuda")
    st = torch.zeros(N, dtype=torch.int32, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    flops = 0
    for k in range(0, nI, PANEL):
        w = min(PANEL, nI - k)
        flops += 2 * (nL - k - w) * (nL + 1 - k - w) * w * N
    best = 1e30
    for _ in range(reps):
        M = M0.clone()
        ms = ctypes.c_double(0)
        torch.cuda.synchronize()
        f(P(M), P(off), P(i32(ld)), P(i32(nI)), P(i32(nL)), P(i32(nL + 1)), N, nI, nL, nL + 1, PANEL,
          P(pinv), 4096, 0, P(st), 0, None, 0, None, None, stream, ctypes.cast(ctypes.pointer(ms), ctypes.c_void_p))
        torch.cuda.synchronize()
        best = min(best, ms.value)
    # GJ inverse of N x nB^2: general, and symmetric (SPD input)
    S0 = torch.rand(N, nB, nB, dtype=torch.float64, device="cuda") + 4 * nB * torch.eye(nB, dtype=torch.float64, device="cuda")
    soff = torch.arange(N, dtype=torch.int64, device="cuda") * nB * nB
    out = []
    for sym in (0, 1):
        A = 0.5 * (S0 + S0.transpose(1, 2)) if sym else S0
        gbest = 1e30
        for _ in range(reps):
            S = A.clone()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g(P(S), P(soff), P(i32(nB)), P(i32(nB)), N, nB, P(pinv), 4096, P(st), sym, sym, stream)
            e1.record()
            torch.cuda.synchronize()
            gbest = min(gbest, e0.elapsed_time(e1))
        ref = torch.linalg.inv(A[:4])
        err = ((S[:4] - ref).abs().max() / ref.abs().max()).item()
        asym = (S[:4] - S[:4].transpose(1, 2)).abs().max().item()
        out.append(f"GJ{'-sym' if sym else ''} {gbest:.2f} ms {2 * nB ** 3 * N / gbest / 1e9:.2f} TF/s-equiv err {err:.1e} asym {asym:.1e}")
    print(f"{path}: trailing {best:.2f} ms {flops / best / 1e9:.2f} TF/s | " + " | ".join(out), flush=True)


if __name__ == "__main__":
    for p in sys.argv[1:] or ["paper_2501_01676_b200/_bddc_b200.so"]:
        run(p)
