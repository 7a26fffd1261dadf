import sys, os, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.scenario import make_case
case = make_case("C1")
sim = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries, stepper.TimeController(dt_init=case.dt_init), phys=case.phys)
for _ in range(20): sim.advance()
t0 = time.perf_counter()
for _ in range(500): sim.advance()
print("wall ms/step", (time.perf_counter() - t0) / 500 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(500): sim.advance()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(18)
