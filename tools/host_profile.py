"""cProfile of hot-path steps (host-side overheads): python tools/host_profile.py [--config 5]"""
import argparse
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2501_01676_b200 import configs, pipeline  # noqa: E402
from paper_2501_01676_b200.engine import upload_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--subs", type=int, default=None)
a = ap.parse_args()
prob = configs.build_problem(a.config, n=a.n, subs=a.subs)
inputs = upload_inputs(prob.system, prob.partition)
run = lambda: pipeline.run(prob.system, prob.partition, prob.globs, 10.0, 10.0, "new", inputs=inputs)
run()
run()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
run()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(40)
