import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from test_gpu_random import _config
from paper_1909_04153_b200 import stepper, _native as nat
seed = int(sys.argv[1])
bathy, state, bounds, phys, ckw, skw = _config(seed)
nx, ny = bathy.grid.nx, bathy.grid.ny
sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw), phys=phys, **skw)
sim.speculate = False
c = sim.controller
pr = sim._fill_params(c.sim_time, c.dt, True)
dev = sim._dev
for ph in range(8):
    rc, res = dev.phase(ph, pr)
    if ph >= 1:
        w, p, q = dev.download(pending=True) if ph == 7 else [t.cpu().numpy() for t in (dev.rows(nat.ARR_W_NEW), dev.rows(nat.ARR_P_NEW), dev.rows(nat.ARR_Q_NEW))]
        print("phase", ph, "P_new row2 cols nx..nx+3", p[2, nx:nx + 4], " row 3:", p[3, nx:nx+4])
