"""Small hot-path runs for compute-sanitizer (racecheck / synccheck / memcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py jump cfg1

Each named golden case runs the full device pipeline once (both variants for
the cases that have them) and checks the iteration count against the fixture.
"""
import sys

sys.path.insert(0, ".")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2501_01676_b200 import pipeline  # noqa: E402
from tests.cases import golden, inputs, variants  # noqa: E402

for name in sys.argv[1:] or ["jump"]:
    g = golden(name)
    system, part, globs = inputs(name)
    for v in variants(g):
        res = pipeline.run(system, part, globs, float(g["theta_f"]), float(g["theta_e"]), v)
        torch.cuda.synchronize()
        ok = abs(res.iterations - int(g[f"{v}_iterations"])) <= 1
        x = res.solution.cpu().numpy()
        rel = np.linalg.norm(x - g[f"{v}_solution"]) / np.linalg.norm(g[f"{v}_solution"])
        print(f"{name} {v}: iterations {res.iterations} (ref {int(g[f'{v}_iterations'])}) "
              f"solution rel {rel:.2e} {'ok' if ok and rel <= 1e-8 else 'MISMATCH'}", flush=True)
