import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from test_gpu_random import _config
from oracle import oracle as orc
from paper_1909_04153_b200 import stepper
seed = int(sys.argv[1])
bathy, state, bounds, phys, ckw, skw = _config(seed)
nx, ny = bathy.grid.nx, bathy.grid.ny
print("P0 max", np.abs(state.p).max(), "kinds", [b.kind for b in (bounds.north, bounds.south, bounds.east, bounds.west)], skw, ckw)
sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw), phys=phys, **skw)
sim.speculate = False
ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(**ckw), phys=phys, **skw)
sim.advance(); ora.advance()
a, b = sim.state, ora.state
for name, A in (("dev", a), ("ora", b)):
    print(name, "P row2 cols nx..nx+3:", A.p[2, nx:nx + 4], " Q:", A.q[2, nx:nx + 4], " W:", A.w[2, nx:nx + 4])
    print(name, "P row2 cols 0..3:", A.p[2, 0:4])
