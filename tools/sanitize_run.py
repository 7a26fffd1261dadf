"""A few steps of small cases through every kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [fp64|fp32] [thomas|cr]

Runs the 128^2 shoal (maker, sponges) and a 70 x 37 odd-shaped wet/dry beach
with friction, 6 AB3 steps each (Euler bootstrap, speculation, both solves,
cross-correction, k_final), then 3 steps on two emulated y-strips.  Exits 0
when every step ran; the sanitizer's own exit code reports the findings.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1909_04153_b200 import boundary as bc  # noqa: E402
from paper_1909_04153_b200 import parallel, stepper  # noqa: E402
from paper_1909_04153_b200.grid import Grid, PhysParams, build_bathymetry, still_state  # noqa: E402
from paper_1909_04153_b200.scenario import make_case  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
solver = sys.argv[2] if len(sys.argv) > 2 else "thomas"


def beach():
    grid = Grid(70, 37, 0.1, 0.1)
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = build_bathymetry(grid, -0.3 + 0.06 * xc + 0.02 * np.sin(yc), ws=0.0)
    st = still_state(bathy)
    st.w += 0.02 * np.exp(-((np.pad(xc, 2, mode="edge") - 1.5) ** 2) / 0.2)
    bounds = bc.Boundaries(west=bc.Wall(), east=bc.Wall(), south=bc.Sponge(0.5, 10.0),
                           north=bc.Wall())
    return bathy, st, bounds, PhysParams(c_f=0.01)


def run(bathy, state, bounds, phys, dt_init, steps):
    sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(dt_init=dt_init),
                            phys=phys, precision=prec, solver=solver)
    for _ in range(steps):
        sim.advance()
    _ = sim.state.w.sum()


c = make_case("C3", scale=8)  # 128^2
run(c.bathy, c.state, c.boundaries, c.phys, c.dt_init, 6)
b, s, bo, ph = beach()
run(b, s, bo, ph, 0.005, 6)
if prec == "fp64" and solver == "thomas":
    sh = parallel.ShardedSimulator(c.bathy, c.state.copy(), c.boundaries,
                                   stepper.TimeController(dt_init=c.dt_init), phys=c.phys,
                                   world=2, coupling="spike")
    for _ in range(3):
        sh.advance()
print("sanitize_run ok", prec, solver)
