"""Time only the line-solve kernel of the bench workload (BSQ_LIB variants,
including timing experiments whose results are garbage): one real step to
set the state up, then bsq_solve_momentum seams are NOT used -- the phased
API runs SOLVE1F alone N times between CUDA events."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1909_04153_b200 import stepper, _native as nat
from paper_1909_04153_b200.scenario import make_case
case = make_case("C4")
sim = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                        stepper.TimeController(dt_init=case.dt_init), phys=case.phys)
sim.speculate = False
for _ in range(4):
    sim.advance()
dev = sim._dev
pr = sim._fill_params(sim.controller.sim_time, sim.controller.dt, False)
dev.phase(nat.PH_GHOST, pr); dev.phase(nat.PH_STAGE)
s = dev.stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    dev.phase(nat.PH_SOLVE1F)
torch.cuda.synchronize()
e0.record(s)
N = 20
for _ in range(N):
    dev.phase(nat.PH_SOLVE1F)
e1.record(s)
torch.cuda.synchronize()
print(json.dumps({"lib": os.path.basename(nat.LIB_PATH), "solve_ms": e0.elapsed_time(e1) / N}))
