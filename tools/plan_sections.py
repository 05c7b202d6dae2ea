"""Host wall time of the sections of the symbolic plan (cfg5), GPU drained at each boundary or not."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2501_01676_b200 import configs
from paper_2501_01676_b200.engine import DevicePlan, upload_inputs
from paper_2501_01676_b200 import plan as P

prob = configs.build_problem(5)
inputs = upload_inputs(prob.system, prob.partition)
names = ["_element_pre_torch", "_glob_part", "_restrict", "_interface_maps_torch", "_element_post_torch", "_layout"]
for drain in (False, True):
    acc = {}
    def wrap(name):
        f = getattr(P.Plan, name + "__orig", None) or getattr(P.Plan, name)
        setattr(P.Plan, name + "__orig", f)
        def g(self, *a, **k):
            t0 = time.perf_counter()
            r = f(self, *a, **k)
            if drain:
                torch.cuda.synchronize()
            acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
            return r
        setattr(P.Plan, name, g)
    for n in names:
        wrap(n)
    for _ in range(3):
        acc.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p = P.Plan(prob.system, prob.partition, prob.globs, device_inputs=inputs)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
    print("drain" if drain else "async", f"total {1e3*(t1-t0):.2f} ms:", {k: round(1e3*v, 2) for k, v in acc.items()})
