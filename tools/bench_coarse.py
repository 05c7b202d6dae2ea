"""Warm timing of the coarse envelope LU (bddc_coarse_factor) on a cfg5-sized
synthetic matrix: n = 12195, envelope half-width BW (default 1500), diagonally
dominant.  Prints the factor time and the time per 64-wide panel, to separate
the per-panel latency floor from the trailing-update work.
Usage: [BDDC_LIB=variant.so] python tools/bench_coarse.py [BW ...]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import os  # noqa: E402

from paper_2501_01676_b200 import _lib  # noqa: E402

if os.environ.get("BDDC_LIB"):  # a tuning / experiment variant of the library
    _lib.LIB_PATH = os.environ["BDDC_LIB"]
lib = _lib.lib


def run(bw, n=12195, reps=3):
    steps = (n + 63) // 64
    lim = np.minimum(n, (np.arange(steps) * 64 + 64 + bw)).astype(np.int32)
    lim_c = (ctypes.c_int * steps)(*lim.tolist())
    A0 = torch.rand(n, n, dtype=torch.float64, device="cuda")
    idx = torch.arange(n, device="cuda")
    band = (idx[:, None] - idx[None, :]).abs() <= bw
    A0 = torch.where(band, A0, torch.zeros((), dtype=torch.float64, device="cuda"))
    A0 += 4 * bw * torch.eye(n, dtype=torch.float64, device="cuda")
    pinv = torch.empty(steps * 4096, dtype=torch.float64, device="cuda")
    piv = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    off = torch.zeros(1, dtype=torch.int64, device="cuda")
    nv = torch.full((1,), n, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    best = 1e30
    for _ in range(reps):
        C = A0.clone().view(-1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.bddc_coarse_factor(C, off, nv, nv, n, ctypes.cast(lim_c, ctypes.c_void_p), pinv, piv, st,
                               ctypes.c_void_p(stream.cuda_stream))
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flops = sum(2.0 * (int(l) - k - 64) ** 2 * 64 for k, l in zip(range(0, n, 64), lim) if l > k + 64)
    print(f"bw {bw}: factor {best:.2f} ms, {best * 1e3 / steps:.1f} us/panel, "
          f"{flops / best / 1e9:.2f} TF/s, status {int(st.item())}", flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:] or ["1500"]:
        run(int(a))
