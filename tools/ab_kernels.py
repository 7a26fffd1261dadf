"""Per-kernel device times of the bench workload for A/B comparisons.

    BSQ_LIB=<variant.so> python tools/ab_kernels.py [--steps N] [--precision fp64]

Prints one JSON line: mean ms per kernel over N timed AB3 steps (CUDA events
on the library stream) and the mean step time.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1909_04153_b200 import _native as nat  # noqa: E402
from paper_1909_04153_b200 import stepper  # noqa: E402
from paper_1909_04153_b200.scenario import make_case  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--precision", default="fp64")
ap.add_argument("--case", default="C4")
ap.add_argument("--no-spec", action="store_true", help="do not queue the next stage early")
ap.add_argument("--solver", default="thomas")
a = ap.parse_args()
case = make_case(a.case)
sim = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                        stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                        precision=a.precision, solver=a.solver)
sim.speculate = not a.no_spec
for _ in range(4):
    sim.advance()
# whole-step device time without per-kernel events (they would split the
# launches PDL lets overlap)
st = sim._dev.stream
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
ev0.record(st)
for _ in range(a.steps):
    sim.advance()
ev1.record(st)
torch.cuda.synchronize()
step_dev = ev0.elapsed_time(ev1) / a.steps
sim._dev.set_timing(True)
acc, n = {}, 0
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.steps):
    sim.advance()
    for name, ms in sim._dev.kernel_times():
        acc[name] = acc.get(name, 0.0) + ms
    n += 1
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / n * 1e3
print(json.dumps({"lib": os.path.basename(nat.LIB_PATH), "spec": not a.no_spec,
                  "step_ms_dev": round(step_dev, 4), "step_ms_wall": round(wall, 4),
                  **{k: round(v / n, 4) for k, v in acc.items()}}))
