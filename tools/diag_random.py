"""Where do device and oracle states differ on the randomized configs
(tests/test_gpu_random.py)?  Prints per field: #cells, #interior cells."""
import sys
sys.path.insert(0, 'tests')
sys.path.insert(0, '.')
import numpy as np  # noqa: E402
from test_gpu_random import _config  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1909_04153_b200 import stepper  # noqa: E402

seeds = [int(s) for s in sys.argv[1].split(",")] if len(sys.argv) > 1 else range(24)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for seed in seeds:
    for spec in (True, False):
        bathy, state, bounds, phys, ckw, skw = _config(seed)
        sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw), phys=phys, **skw)
        sim.speculate = spec
        ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(**ckw), phys=phys, **skw)
        first = None
        try:
            for k in range(steps):
                a = sim.advance(); b = ora.advance()
                if first is None:
                    sa, sb = sim.state, ora.state
                    for f in "wpq":
                        A, B = getattr(sa, f), getattr(sb, f)
                        bad = ~((A == B) | (np.isnan(A) & np.isnan(B)))
                        if bad.any():
                            ny, nx = A.shape
                            inter = bad[2:ny - 2, 2:nx - 2].sum()
                            first = (k, f, int(bad.sum()), int(inter), np.argwhere(bad)[:3].tolist())
                            break
        except Exception as e:
            first = (first, "EXC", str(e)[:80])
        kinds = [bb.kind for bb in (bounds.north, bounds.south, bounds.east, bounds.west)]
        print(seed, "spec" if spec else "nospec", bathy.grid.nx, bathy.grid.ny, kinds, skw, ckw["mode"], first)
