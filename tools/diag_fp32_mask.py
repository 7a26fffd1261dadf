import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import test_gpu_random as T
from oracle import oracle as orc
from paper_1909_04153_b200 import stepper
bathy, state, bounds, phys, ckw, skw = T._config(50)
ckw = dict(ckw, mode="fixed")
sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw), phys=phys, precision="fp32", **skw)
ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(**ckw), phys=phys, **skw)
for k in range(30):
    sim.advance(); ora.advance()
ii = bathy.grid.interior
h_dry = sim.h_dry
a = (sim.state.w - bathy.bed_eff)[ii]; b = (ora.state.w - bathy.bed_eff)[ii]
m = (a > h_dry) != (b > h_dry)
print("h_dry", h_dry, "skw", skw, "mismatches", int(m.sum()))
bed = bathy.bed_eff[ii]; w32 = sim.state.w[ii]; w64 = ora.state.w[ii]
for j, i in np.argwhere(m)[:10]:
    print(j, i, "h32", a[j, i], "h64", b[j, i], "bed", bed[j, i], "f32(bed)", float(np.float32(bed[j, i])), "w32", w32[j, i], "w64", w64[j, i])
