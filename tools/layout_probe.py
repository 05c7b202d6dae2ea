"""Layout sensitivity probe: hold a dummy device allocation before a chosen
phase and check that the iteration count / solution do not change."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from tests.cases import inputs, golden
from paper_2501_01676_b200 import pipeline, engine
name = sys.argv[1]
g = golden(name)
system, part, globs = inputs(name)
hold = []
orig = {}
def wrap(cls, mb):
    init = cls.__init__
    def new_init(self, *a, **k):
        hold.append(torch.empty(int(mb * 2 ** 20), dtype=torch.uint8, device="cuda"))
        return init(self, *a, **k)
    orig[cls] = init
    cls.__init__ = new_init
base = None
for target in [None, "DeviceScaling", "DevicePrimalSpace", "DevicePreconditioner", "DeviceInterfaceOperator"]:
    for mb in ([0] if target is None else [1, 37, 300]):
        for c, f in orig.items():
            c.__init__ = f
        orig.clear()
        hold.clear()
        if target is not None:
            wrap(getattr(engine, target), mb)
        r = pipeline.run(system, part, globs, float(g["theta_f"]), float(g["theta_e"]), "new", keep=True)
        x = r.solution.cpu().numpy()
        if base is None:
            base = x
        print(target, mb, "iterations", r.iterations, "ph0 %.3e" % r.pre_hist[0],
              "x rel diff %.2e" % (np.linalg.norm(x - base) / np.linalg.norm(base)), flush=True)
