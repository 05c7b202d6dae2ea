"""One hot-path step on a config (for ncu launch lists / captures)."""
import argparse
import sys
import time

sys.path.insert(0, ".")

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--subs", type=int, default=None)
ap.add_argument("--steps", type=int, default=1)
args = ap.parse_args()

import torch  # noqa: E402

from paper_2501_01676_b200 import configs, pipeline  # noqa: E402
from paper_2501_01676_b200.engine import upload_inputs  # noqa: E402

prob = configs.build_problem(args.config, n=args.n, subs=args.subs)
inputs = upload_inputs(prob.system, prob.partition)
for _ in range(args.steps):
    t0 = time.time()
    res = pipeline.run(prob.system, prob.partition, prob.globs, 10.0, 10.0, "new", inputs=inputs)
    torch.cuda.synchronize()
    print(f"step {time.time() - t0:.3f}s iters {res.iterations} n_c {res.n_c} phases {res.times_ms}", flush=True)
