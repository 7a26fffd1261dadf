"""Weak-scaling cost of the strip path, emulated on one GPU: C5 with G=2
(global 4096 x 8192, two 4096 x 4096 strips run one after the other on the
same device).  Half the emulated step time is what one rank would spend per
step without NCCL latencies; compare with the single-grid 4096^2 step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1909_04153_b200 import stepper  # noqa: E402
from paper_1909_04153_b200.parallel import ShardedSimulator  # noqa: E402
from paper_1909_04153_b200.scenario import make_case  # noqa: E402


def timed(sim, n=10):
    for _ in range(4):
        sim.advance()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        sim.advance()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


c1 = make_case("C5", gpus=1)
one = stepper.Simulator(c1.bathy, c1.state.copy(), c1.boundaries,
                        stepper.TimeController(dt_init=c1.dt_init), phys=c1.phys)
print(f"one grid 4096^2: {timed(one):.3f} ms/step", flush=True)
one.close()
c2 = make_case("C5", gpus=2)
for coupling in ("spike", "pipeline"):
    for spec in (True, False):
        sp = ShardedSimulator(c2.bathy, c2.state.copy(), c2.boundaries,
                              stepper.TimeController(dt_init=c2.dt_init), phys=c2.phys,
                              world=2, coupling=coupling)
        sp.speculate = spec
        t = timed(sp)
        print(f"2 strips of 4096^2 ({coupling}, speculate={spec}): {t:.3f} ms/step on one GPU "
              f"= {t / 2:.3f} per strip", flush=True)
        sp.close()
