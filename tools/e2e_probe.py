"""Where the end-to-end step's extra time goes: staged upload alone, the step
with device-resident inputs, and the end-to-end step with / without the late
inputs on the copy stream."""
import gc
import sys
import time

sys.path.insert(0, ".")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_01676_b200 import configs, pipeline  # noqa: E402
from paper_2501_01676_b200.engine import stage_inputs, upload_inputs, upload_staged  # noqa: E402

prob = configs.build_problem(5)
s, part, globs = prob.system, prob.partition, prob.globs
staged = stage_inputs(s, part)
u_pinned = torch.empty(s.mesh.n_nodes, dtype=torch.float64, pin_memory=True)


def wall(f, n=5):
    out = []
    for i in range(n + 1):
        gc.collect(); gc.disable()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) * 1e3)
        gc.enable()
    return round(float(np.mean(out[1:])), 2), [round(x, 2) for x in out[1:]]


for ov in (False, True):
    print("upload only, overlap", ov, wall(lambda: upload_staged(staged, overlap=ov)))
dev = upload_inputs(s, part)
print("device-resident step", wall(lambda: pipeline.run(s, part, globs, 10.0, 10.0, "new", inputs=dev)))


def e2e(ov):
    inp = upload_staged(staged, overlap=ov)
    r = pipeline.run(s, part, globs, 10.0, 10.0, "new", inputs=inp)
    u_pinned.copy_(r.u)
    return r


for ov in (False, True, False, True):
    print("e2e, overlap", ov, wall(lambda: e2e(ov)))
r = e2e(True)
print("phases", {k: round(v, 2) for k, v in r.times_ms.items()})
r = e2e(False)
print("phases (no overlap)", {k: round(v, 2) for k, v in r.times_ms.items()})
