"""Sweep of the L2-group sizes of the batched factorisations (BDDC_*_GROUP):
each group of matrices goes through all its panel steps before the next one,
so a group that fits the L2 is read from DRAM once.  Prints the phase times."""
import os
import sys

sys.path.insert(0, ".")

import torch  # noqa: E402

from paper_2501_01676_b200 import configs, pipeline  # noqa: E402
from paper_2501_01676_b200.engine import upload_inputs  # noqa: E402

prob = configs.build_problem(5)
inputs = upload_inputs(prob.system, prob.partition)
sweep = [("BDDC_GJ_GROUP", g) for g in (0, 512, 128, 64, 32)]
sweep += [("BDDC_DUAL_GROUP", g) for g in (512, 128, 64, 32)]
sweep += [("BDDC_ELIM_GROUP_B", g) for g in (256, 64, 32, 16)]
sweep += [("BDDC_ELIM_GROUP_A", g) for g in (256, 64, 32)]
if len(sys.argv) > 1:
    sweep = [(a.split("=")[0], int(a.split("=")[1])) for a in sys.argv[1:]]
    for var, g in sweep:
        os.environ[var] = str(g)
    sweep = [("none", 0)]
for var, g in sweep:
    os.environ[var] = str(g)
    best = None
    for _ in range(4):
        res = pipeline.run(prob.system, prob.partition, prob.globs, 10.0, 10.0, "new", inputs=inputs)
        torch.cuda.synchronize()
        t = res.times_ms
        if best is None or sum(t.values()) < sum(best.values()):
            best = t
    print(f"{var}={g}: total {sum(best.values()):.2f} iters {res.iterations} "
          + " ".join(f"{k}={v:.2f}" for k, v in best.items()), flush=True)
    os.environ.pop(var, None)
