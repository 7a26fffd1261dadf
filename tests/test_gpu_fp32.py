"""fp32 mode (north_star): device storage and arithmetic in float, checked
against the fp64 reference on identical inputs.  Bar: rel-L2 of the surface
deviation eta <= 1e-4 and an identical wet/dry mask ``w - bed_eff > h_dry``."""

import numpy as np
import pytest

import golden_cases as gc
from oracle import oracle as orc
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.scenario import make_case

pytestmark = pytest.mark.gpu
II = (slice(2, -2), slice(2, -2))
ETA_TOL = 1e-4  # north_star fp32 bound


def eta(w, bathy):
    rest = np.maximum(bathy.ws, bathy.bed_eff)
    return (w - rest)[II]


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def mask(w, bathy, h_dry, fp32=False):
    """Wet cells, w - bed_eff > h_dry.  An fp32 run is judged against its own
    float-rounded bed: its dry cells hold w == float(bed_eff) exactly."""
    bed = bathy.bed_eff.astype(np.float32).astype(np.float64) if fp32 else bathy.bed_eff
    return (w - bed)[II] > h_dry


@pytest.mark.parametrize("name", ["c1", "runup", "maker_sponge", "rip_irregular"])
def test_fp32_golden_run(name):
    """Full golden runs (C1: 1000 adaptive steps) in fp32 vs the reference."""
    z = gc.load(name)
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    sim = stepper.Simulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys,
                            precision="fp32", **skw)
    for _ in range(int(z["steps"])):
        sim.advance()
    w = sim.state.w
    e32, e64 = eta(w, bathy), eta(z["w"], bathy)
    r = rel(e32, e64)
    print(f"{name}: fp32 eta rel-L2 {r:.3e}, dt[-1] {sim.records[-1].dt:.6e} "
          f"vs {z['records'][-1, 2]:.6e}")
    assert r <= ETA_TOL
    h_dry = sim.h_dry
    assert np.array_equal(mask(w, bathy, h_dry, fp32=True), mask(z["w"], bathy, h_dry))
    # the adaptive dt sequence stays close to the fp64 one
    np.testing.assert_allclose([rc.dt for rc in sim.records], z["records"][:, 2], rtol=1e-3)


def test_fp32_rip_512_vs_oracle():
    case = make_case("C4", scale=8)
    sim = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                            precision="fp32")
    ora = orc.OracleSimulator(case.bathy, case.state.copy(), case.boundaries,
                              orc.OController(dt_init=case.dt_init), phys=case.phys, threads=8)
    for _ in range(200):
        sim.advance()
        ora.advance()
    w32, w64 = sim.state.w, ora.state.w
    r = rel(eta(w32, case.bathy), eta(w64, case.bathy))
    print(f"rip 512^2 200 steps: fp32 eta rel-L2 {r:.3e}")
    assert r <= ETA_TOL
    h = sim.h_dry
    m32, m64 = mask(w32, case.bathy, h, fp32=True), mask(w64, case.bathy, h)
    assert np.array_equal(m32, m64), int((m32 != m64).sum())
