"""Per-step cost of the y-strip path against one grid, emulated on one GPU
(LocalComm: the strips run one after another on the same device, so this
measures the strip path's extra kernels and host work, not NCCL):
4096 x 4096 global, world strips, coupling "spike" (the bench's multi-GPU
mode) and "pipeline"."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1909_04153_b200 import stepper  # noqa: E402
from paper_1909_04153_b200.parallel import ShardedSimulator  # noqa: E402
from paper_1909_04153_b200.scenario import make_case  # noqa: E402

case = make_case("C5", gpus=1)
mk = lambda: stepper.TimeController(dt_init=case.dt_init)  # noqa: E731


def timed(sim, n=10):
    for _ in range(4):
        sim.advance()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        sim.advance()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


one = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries, mk(), phys=case.phys)
print(f"one grid: {timed(one):.3f} ms/step", flush=True)
one.speculate = False
print(f"one grid, no speculation: {timed(one):.3f} ms/step", flush=True)
one.close()
for coupling in ("spike", "pipeline"):
    sp = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries, mk(), phys=case.phys,
                          world=1, coupling=coupling)
    print(f"1 strip (phased path) {coupling}: {timed(sp):.3f} ms/step", flush=True)
    del sp
for world in (2, 4):
    for coupling in ("spike", "pipeline"):
        sp = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries, mk(), phys=case.phys,
                              world=world, coupling=coupling)
        print(f"{world} strips {coupling}: {timed(sp):.3f} ms/step (all strips, one GPU)", flush=True)
        del sp

# per-kernel device times of strip 0 (2 strips, spike) and the step's wall time
sp = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries, mk(), phys=case.phys,
                      world=2, coupling="spike")
for _ in range(4):
    sp.advance()
sp._dev.set_timing(True)
acc = {}
for _ in range(5):
    sp.advance()
    for name, ms in sp._dev.kernel_times():
        acc[name] = acc.get(name, 0.0) + ms / 5
print("strip 0 kernels (ms):", {k: round(v, 4) for k, v in acc.items()},
      "sum", round(sum(acc.values()), 3), flush=True)
