"""Per-kernel device times of each emulated y-strip (C5, G = 2 on one GPU),
for comparison with the single-grid step (tools/ab_kernels.py):

    python tools/strip_kernels.py [--coupling spike] [--steps 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1909_04153_b200 import stepper  # noqa: E402
from paper_1909_04153_b200.parallel import ShardedSimulator  # noqa: E402
from paper_1909_04153_b200.scenario import make_case  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--coupling", default="spike")
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
c2 = make_case("C5", gpus=2)
sim = ShardedSimulator(c2.bathy, c2.state.copy(), c2.boundaries,
                       stepper.TimeController(dt_init=c2.dt_init), phys=c2.phys, world=2,
                       coupling=a.coupling)
for _ in range(4):
    sim.advance()
dev = sim._dev
dev.set_timing(True)
acc = [dict() for _ in dev.strips]
for _ in range(a.steps):
    sim.advance()
    for k, r in enumerate(sorted(dev.strips)):
        for name, ms in dev.strips[r].kernel_times():
            acc[k][name] = acc[k].get(name, 0.0) + ms
torch.cuda.synchronize()
for k, d in enumerate(acc):
    print(json.dumps({"strip": k, "coupling": a.coupling, "sum_ms": round(sum(d.values()) / a.steps, 4),
                      **{n: round(v / a.steps, 4) for n, v in d.items()}}))
