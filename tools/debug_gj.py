"""Batched GJ inverse of small matrices vs numpy (debug helper)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2501_01676_b200._lib import lib, stream

for n in (4, 8, 13, 64, 100):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)) + n * np.eye(n)
    M = torch.from_numpy(A.ravel().copy()).cuda()
    off = torch.zeros(1, dtype=torch.int64, device="cuda")
    nn = torch.full((1,), n, dtype=torch.int32, device="cuda")
    pinv = torch.zeros(4096, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.bddc_gj_inverse(M, off, nn, nn, 1, n, pinv, 4096, st, 0, 0, stream())
    X = M.cpu().numpy().reshape(n, n)
    E = X - np.linalg.inv(A)
    print(n, "status", int(st.item()), "err", np.abs(E).max())
    if not np.isfinite(E).all() or np.abs(E).max() > 1e-10:
        bad = np.argwhere(~np.isfinite(E) | (np.abs(E) > 1e-10))
        print(" first bad", bad[:10].tolist())
        P = pinv.cpu().numpy().reshape(64, 64)[:min(n, 64), :min(n, 64)]
        print(" pinv err", np.abs(P - np.linalg.inv(A[:min(n, 64), :min(n, 64)])).max())
