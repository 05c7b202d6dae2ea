"""Phase profile of the face / new-edge eigenproblem kernels (clock64 per
phase, summed over CTAs) on one hot-path step.

    python tools/prof_globs.py --build      # here: builds _bddc_b200_prof.so (-DBDDC_PROF)
    python tools/prof_globs.py [--config 5] # GPU box: one warm step, then the profile
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, ".")
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2501_01676_b200")
PROF_LIB = os.path.abspath(os.path.join(HERE, "_bddc_b200_prof.so"))

FACE = ["B_F gemms", "glob Schur x2", "parallel sum", "cholesky", "trsm L^-1", "whitening gemms",
        "tridiagonalize", "bisection", "eigvecs+rows", "row space basis"]
EDGE = ["J, M", "Bt assembly (X inverses)", "Btt (RR chol)", "pencil", "rows", "row space basis"]

ap = argparse.ArgumentParser()
ap.add_argument("--build", action="store_true")
ap.add_argument("--config", type=int, default=5)
args = ap.parse_args()
if args.build:
    from paper_2501_01676_b200 import build
    print(build.build(defines=("BDDC_PROF=1",), out=PROF_LIB))
    sys.exit(0)

os.environ["BDDC_LIB"] = PROF_LIB
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_01676_b200 import configs, pipeline  # noqa: E402
from paper_2501_01676_b200._lib import lib  # noqa: E402
from paper_2501_01676_b200.engine import upload_inputs  # noqa: E402

prob = configs.build_problem(args.config)
inputs = upload_inputs(prob.system, prob.partition)
read = lib.load().bddc_prof_read
read.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 64)()
for it in range(2):
    read(buf, 1)
    res = pipeline.run(prob.system, prob.partition, prob.globs, 10.0, 10.0, "new", inputs=inputs)
    torch.cuda.synchronize()
read(buf, 0)
v = np.array(buf[:], dtype=np.float64)
print(f"phases (ms) {res.times_ms}")
GJ = ["publish + barrier", "4x4 pivot chain", "U + barrier", "DMMA + pivot rows", "load", "store"]
for name, lo, labels in (("face_fast_kernel", 0, FACE), ("edge_new_kernel", 16, EDGE),
                         ("reg_gj64 (slot_schur / edge kernels)", 32, GJ)):
    tot = v[lo:lo + len(labels)].sum()
    print(f"\n{name}: total {tot:.3e} CTA-cycles")
    for i, lab in enumerate(labels):
        print(f"  {lab:28s} {v[lo + i]:.3e}  {100 * v[lo + i] / max(tot, 1):5.1f} %")
