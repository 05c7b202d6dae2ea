"""Uninitialised-read hunt: torch.empty memory is NaN-filled, then every
device buffer of one pipeline run is checked for NaN."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
torch.use_deterministic_algorithms(True, warn_only=True)
import torch.utils.deterministic
torch.utils.deterministic.fill_uninitialized_memory = True
from tests.cases import inputs, golden
from paper_2501_01676_b200 import pipeline
name = sys.argv[1]
if len(sys.argv) > 2 and sys.argv[2] == "seq":
    os.environ["BDDC_NO_OVERLAP"] = "1"
g = golden(name)
system, part, globs = inputs(name)
r = pipeline.run(system, part, globs, float(g["theta_f"]), float(g["theta_e"]), "new", keep=True)
torch.cuda.synchronize()
print("iterations", r.iterations, "golden", int(g["new_iterations"]))
def chk(label, t):
    if isinstance(t, torch.Tensor) and t.is_floating_point():
        n = int(torch.isnan(t).sum().item())
        if n:
            print("NaN in", label, n, "of", t.numel())
for objname, obj in (("ls", r.ls), ("sc", r.scaling), ("ps", r.space), ("pc", r.pc), ("op", r.op)):
    for k, v in vars(obj).items():
        chk(f"{objname}.{k}", v)
chk("solution", r.solution)
print("done")
