"""GPU time per C-ABI entry point over one warm hot-path step (CUDA events
around every call; _lib.profile) -- a quick kernel-level breakdown without ncu.

    python tools/kernel_profile.py [--config 5] [--n N --subs S]
"""
import argparse
import sys

sys.path.insert(0, ".")

import torch  # noqa: E402

from paper_2501_01676_b200 import _lib, configs, pipeline  # noqa: E402
from paper_2501_01676_b200.engine import upload_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--subs", type=int, default=None)
args = ap.parse_args()
prob = configs.build_problem(args.config, n=args.n, subs=args.subs)
inputs = upload_inputs(prob.system, prob.partition)
for _ in range(2):
    res = pipeline.run(prob.system, prob.partition, prob.globs, 10.0, 10.0, "new", inputs=inputs)
torch.cuda.synchronize()
_lib.profile(True)
res = pipeline.run(prob.system, prob.partition, prob.globs, 10.0, 10.0, "new", inputs=inputs)
torch.cuda.synchronize()
rep = _lib.profile_report()
_lib.profile(False)
print("phases (ms):", {k: round(v, 2) for k, v in res.times_ms.items()})
tot = sum(t for _, t in rep.values())
print(f"{'entry point':40s} {'calls':>6s} {'ms':>9s} {'share':>6s}")
for name, (c, t) in sorted(rep.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:40s} {c:6d} {t:9.3f} {100 * t / tot:5.1f}%")
print(f"{'total (events)':40s} {'':6s} {tot:9.3f}")
