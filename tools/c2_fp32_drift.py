"""fp32 vs fp64 device runs of C2 (2048 x 64 runup): eta rel-L2 every 250 steps."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.scenario import make_case
case = make_case(sys.argv[1] if len(sys.argv) > 1 else "C2")
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6000
sims = [stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                          stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                          h_dry=case.h_dry, precision=p) for p in ("fp64", "fp32")]
b = case.bathy
ii = b.grid.interior
rest = np.maximum(b.ws, b.bed_eff)
for k in range(1, steps + 1):
    r = [s.advance() for s in sims]
    if k % 250 == 0:
        e = [(s.state.w - rest)[ii] for s in sims]
        rel = np.linalg.norm(e[1] - e[0]) / np.linalg.norm(e[0])
        m = [((s.state.w - b.bed_eff)[ii] > s.h_dry) for s in sims]
        print(f"step {k}: t64 {r[0].sim_time:.4f} t32 {r[1].sim_time:.4f} dt64 {r[0].dt:.3e} "
              f"dt32 {r[1].dt:.3e} eta rel-L2 {rel:.3e} mask diff {int((m[0] != m[1]).sum())}",
              flush=True)
