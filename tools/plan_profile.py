"""cProfile of the symbolic plan alone (host-bound phase): python tools/plan_profile.py"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2501_01676_b200 import configs  # noqa: E402
from paper_2501_01676_b200.engine import DevicePlan, upload_inputs  # noqa: E402
from paper_2501_01676_b200.plan import Plan  # noqa: E402

prob = configs.build_problem(5)
inputs = upload_inputs(prob.system, prob.partition)
for _ in range(3):
    p = Plan(prob.system, prob.partition, prob.globs, device_inputs=inputs)
    d = DevicePlan(p)
torch.cuda.synchronize()
t0 = time.perf_counter()
p = Plan(prob.system, prob.partition, prob.globs, device_inputs=inputs)
t1 = time.perf_counter()
d = DevicePlan(p)
t2 = time.perf_counter()
torch.cuda.synchronize()
t3 = time.perf_counter()
print(f"Plan host {1e3 * (t1 - t0):.2f} ms, DevicePlan host {1e3 * (t2 - t1):.2f} ms, drain {1e3 * (t3 - t2):.2f} ms")
pr = cProfile.Profile()
pr.enable()
p = Plan(prob.system, prob.partition, prob.globs, device_inputs=inputs)
d = DevicePlan(p)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
