"""Which kernel of the step differs on tiny momenta (test_gpu_tiny)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle import oracle as orc
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.grid import PhysParams
import test_gpu_tiny as T
rng = np.random.default_rng(5)
from paper_1909_04153_b200.grid import Grid, build_bathymetry, still_state
grid = Grid(70, 40, 0.25, 0.25)
xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
bathy = build_bathymetry(grid, -0.6 + 0.2 * np.exp(-((xc - 8) ** 2 + (yc - 5) ** 2) / 3.0), ws=0.0)
st = still_state(bathy)
shape = st.w.shape
st.w += 0.02 * np.exp(-((np.pad(xc, 2, mode="edge") - 4) ** 2) / 2.0)
st.p = 10.0 ** rng.uniform(-320, -290, shape) * rng.choice([-1.0, 1.0], shape)
st.q = 10.0 ** rng.uniform(-320, -290, shape) * rng.choice([-1.0, 1.0], shape)
st.p[rng.random(shape) < 0.3] = 0.0
phys = PhysParams()
sim = stepper.Simulator(bathy, st.copy(), T.walls(), stepper.TimeController(dt_init=0.01), phys=phys)
ex = sim._dev.speed_extrema()
eo = orc.speed_extrema(st, bathy, phys)
print("extrema", ex, eo, [a == b for a, b in zip(ex, eo)])
sr = sim._dev.stage_rates()
so = orc.stage_rates(st, bathy, phys)
names = ["e", "f", "g", "fs", "gs"]
for k in range(5):
    a, b = np.asarray(sr[k]), np.asarray(so[k])
    bad = a.view(np.uint64) != b.view(np.uint64)
    print(names[k], int(bad.sum()), a[bad][:3], b[bad][:3])

# step-by-step
sim = stepper.Simulator(bathy, st.copy(), T.walls(), stepper.TimeController(dt_init=0.01), phys=phys)
ora = orc.OracleSimulator(bathy, st.copy(), T.walls(), orc.OController(dt_init=0.01), phys=phys, threads=4)
for k in range(12):
    a, b = sim.advance(), ora.advance()
    rec_ok = (a.dt, a.max_cfl, a.max_speed, a.max_depth) == (b.dt, b.max_cfl, b.max_speed, b.max_depth)
    bad = {}
    for f in ("w", "p", "q"):
        x, y = getattr(sim.state, f), getattr(ora.state, f)
        m = x.view(np.uint64) != y.view(np.uint64)
        if m.any():
            idx = np.argwhere(m)[:3]
            bad[f] = (int(m.sum()), [(tuple(i), x[tuple(i)], y[tuple(i)]) for i in idx])
    print("step", k, "records ok" if rec_ok else f"records differ {a} {b}", bad if bad else "state ok")
    if bad or not rec_ok:
        break
