"""Bytes each rank moves per GMRES iteration on the sharded path,
from the host plans alone (no GPU): python tools/dist_bytes.py [--config 5] [--ranks 2 4 8]"""
import argparse
import sys

sys.path.insert(0, ".")

import numpy as np  # noqa: E402

from paper_2501_01676_b200 import configs  # noqa: E402
from paper_2501_01676_b200.dist import InterfaceLayout, SlotExchange, block_range  # noqa: E402
from paper_2501_01676_b200.plan import Plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
args = ap.parse_args()
prob = configs.build_problem(args.config)
n_hat = prob.globs.interface_nodes.size


class FakeComm:
    def __init__(self, rank, size):
        self.rank, self.size = rank, size


for R in args.ranks:
    halo, own, loc, slots = [], [], [], []
    for r in range(R):
        plan = Plan(prob.system, prob.partition, prob.globs,
                    owned=block_range(prob.partition.n_subdomains, R, r))
        lay = InterfaceLayout(plan, FakeComm(r, R))
        halo.append(lay.halo_bytes())
        own.append(lay.n_own)
        loc.append(lay.n_loc)
        sx = SlotExchange(plan, FakeComm(r, R))
        send, _ = sx._pairs("to_owner")
        sz = (plan.gsize[plan.slot_glob].astype(np.int64) ** 2)
        slots.append(8 * int(sum(sz[s].sum() for s in send.values())))
    print(f"R={R}: n_hat {n_hat}; per rank owned {min(own)}-{max(own)}, local {min(loc)}-{max(loc)}; "
          f"halo bytes out per interface-sum {min(halo)}-{max(halo)} "
          f"(x2 per iteration: S_hat and M^-1); Bsym slot blocks to glob owners "
          f"{min(slots)}-{max(slots)} bytes per buffer", flush=True)
