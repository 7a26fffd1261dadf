"""How far the SPIKE-coupled y-strips (ranks concurrent) drift from the
single-grid run over a long horizon: 512^2 rip channel, 4 emulated strips on
one GPU, eta rel-L2 and dt difference every 500 steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1909_04153_b200 import stepper  # noqa: E402
from paper_1909_04153_b200.parallel import ShardedSimulator  # noqa: E402
from paper_1909_04153_b200.scenario import make_case  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
world = int(sys.argv[2]) if len(sys.argv) > 2 else 4
case = make_case("C4", scale=8)
mk = lambda: stepper.TimeController(dt_init=case.dt_init)  # noqa: E731
one = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries, mk(), phys=case.phys)
sp = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries, mk(), phys=case.phys,
                      world=world, coupling="spike")
ii = case.bathy.grid.interior
rest = np.maximum(case.bathy.ws, case.bathy.bed_eff)[ii]
for k in range(1, steps + 1):
    a, b = one.advance(), sp.advance()
    if k % 500 == 0 or k == steps:
        ea, eb = one.state.w[ii] - rest, sp.state.w[ii] - rest
        r = np.linalg.norm(eb - ea) / np.linalg.norm(ea)
        print(f"step {k}: t={a.sim_time:.4f}  eta rel-L2 {r:.3e}  dt rel diff {abs(b.dt - a.dt) / a.dt:.3e}",
              flush=True)
