"""A few steps of the emulated C5 G = 2 y-strip run (for an ncu launch list):
    ncu --metrics gpu__time_duration.sum --csv python tools/strip_step.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1909_04153_b200 import stepper  # noqa: E402
from paper_1909_04153_b200.parallel import ShardedSimulator  # noqa: E402
from paper_1909_04153_b200.scenario import make_case  # noqa: E402

coupling = sys.argv[1] if len(sys.argv) > 1 else "spike"
c2 = make_case("C5", gpus=2)
sim = ShardedSimulator(c2.bathy, c2.state.copy(), c2.boundaries,
                       stepper.TimeController(dt_init=c2.dt_init), phys=c2.phys, world=2,
                       coupling=coupling)
for _ in range(6):
    sim.advance()
torch.cuda.synchronize()
print("strip_step ok")
