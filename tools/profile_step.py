"""Run a few real steps of the bench workload (for ncu captures).

    python tools/profile_step.py [--scale S] [--steps N]

Three warm-up steps (Euler x2 + first AB3) then N AB3 steps; with ncu use
-s to skip the warm-up launches (6 kernels per step).
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1909_04153_b200 import stepper  # noqa: E402
from paper_1909_04153_b200.scenario import make_case  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=1)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--case", default="C4")
ap.add_argument("--precision", default="fp64")
ap.add_argument("--solver", default="thomas")
args = ap.parse_args()
case = make_case(args.case, scale=args.scale)
sim = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                        stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                        precision=args.precision, solver=args.solver)
for _ in range(3 + args.steps):
    rec = sim.advance()
torch.cuda.synchronize()
print("ok", rec)
