"""Where the bench's e2e time goes: state upload, each advance(), download
(wall clock with a device sync after each part; one GPU, bench workload)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1909_04153_b200 import stepper  # noqa: E402
from paper_1909_04153_b200.grid import FieldState  # noqa: E402
from paper_1909_04153_b200.scenario import make_case  # noqa: E402

case = make_case("C5", gpus=1)
pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
       for a in (case.state.w, case.state.p, case.state.q)]
pin_out = [torch.empty(a.shape, dtype=torch.float64).pin_memory().numpy() for a in pin]
for rep in range(2):
    sim = stepper.Simulator(case.bathy, FieldState(*pin), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys)
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    sim.state = FieldState(*pin)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    steps = []
    for _ in range(20):
        s0 = time.perf_counter()
        sim.advance()
        steps.append((time.perf_counter() - s0) * 1e3)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    sim.download_state(out=pin_out)
    t.append(time.perf_counter())
    print(f"rep {rep}: upload {1e3 * (t[1] - t[0]):.2f} ms, 20 steps {1e3 * (t[2] - t[1]):.2f} ms, "
          f"download {1e3 * (t[3] - t[2]):.2f} ms; per step " + " ".join(f"{x:.2f}" for x in steps))
    sim.close()
