"""Long-horizon parity (north_star: identical dt sequence and 1e-9 after 1000
steps): the rip-channel bench geometry at 512^2 (irregular maker, friction,
wet/dry beach) for 4000 adaptive steps with speculation on, every record and
the final state bit for bit against the CPU oracle.  Any single-bit
difference on the way would be amplified by the breaking wave field."""

import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.scenario import make_case

pytestmark = pytest.mark.gpu
II = (slice(2, -2), slice(2, -2))


def test_rip_512_4000_steps_bitwise():
    case = make_case("C4", scale=8)
    sim = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                            h_dry=case.h_dry)
    ora = orc.OracleSimulator(case.bathy, case.state.copy(), case.boundaries,
                              orc.OController(dt_init=case.dt_init), phys=case.phys,
                              h_dry=case.h_dry, threads=os.cpu_count() or 8)
    for k in range(4000):
        a, b = sim.advance(), ora.advance()
        assert (a.dt, a.max_cfl, a.max_speed, a.max_depth) == \
            (b.dt, b.max_cfl, b.max_speed, b.max_depth), k
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(sim.state, f)[II], getattr(ora.state, f)[II]), f
    assert sim.clamped_volume == pytest.approx(ora.clamped_volume, rel=1e-12, abs=1e-300)
    print(f"4000 steps bitwise, t = {sim.controller.sim_time:.4f} s")


def test_rip_512_spike_strips_2000_steps_stay_within_1e12():
    """4 SPIKE-coupled y-strips (the multi-GPU bench mode, emulated on one
    GPU) against the single grid over 2000 adaptive steps: the coupling's
    rounding does not grow (measured ~5e-15 on eta after 4000 steps,
    tools/spike_drift.py)."""
    from paper_1909_04153_b200.parallel import ShardedSimulator
    case = make_case("C4", scale=8)
    one = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys)
    sp = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries,
                          stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                          world=4, coupling="spike")
    for k in range(2000):
        a, b = one.advance(), sp.advance()
        assert b.dt == pytest.approx(a.dt, rel=1e-12), k
    ii = case.bathy.grid.interior
    rest = np.maximum(case.bathy.ws, case.bathy.bed_eff)[ii]
    ea, eb = one.state.w[ii] - rest, sp.state.w[ii] - rest
    assert np.linalg.norm(eb - ea) / np.linalg.norm(ea) <= 1e-12
    scale = max(np.linalg.norm(one.state.p[ii]), np.linalg.norm(one.state.q[ii]))
    for f in ("p", "q"):
        d = getattr(sp.state, f)[ii] - getattr(one.state, f)[ii]
        assert np.linalg.norm(d) / scale <= 1e-11, f
