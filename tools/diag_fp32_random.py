"""fp32 vs the fp64 oracle on random configurations (tests/test_gpu_random.py
_config): eta rel-L2 after each step, and whether the operator lost diagonal
dominance.  Run on a B200:  python tools/diag_fp32_random.py 58 118 2"""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import test_gpu_random as T  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_1909_04153_b200 import stepper  # noqa: E402

for seed in [int(a) for a in sys.argv[1:]]:
    bathy, state, bounds, phys, ckw, skw = T._config(seed)
    ckw = dict(ckw, mode="fixed")
    with warnings.catch_warnings(record=True) as wl:
        warnings.simplefilter("always")
        sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw),
                                phys=phys, precision="fp32", **skw)
    ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(**ckw), phys=phys, **skw)
    ii = bathy.grid.interior
    rels, cfl = [], []
    try:
        for k in range(30):
            r = sim.advance()
            ora.advance()
            cfl.append(r.max_cfl)
            a = sim.state.w[ii] - bathy.ws
            b = ora.state.w[ii] - bathy.ws
            rels.append(float(np.linalg.norm(a - b) / np.linalg.norm(b)))
    except Exception as e:  # noqa: BLE001
        rels.append(f"abort: {str(e)[:60]}")
    print(seed, bathy.grid.nx, bathy.grid.ny, skw, "dominance warnings:", len(wl),
          "max cfl %.3f" % max(cfl) if cfl else "", "rel-L2 every 5 steps:",
          [x if isinstance(x, str) else float("%.2e" % x) for x in rels[4::5]] + rels[-1:])
