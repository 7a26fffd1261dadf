"""Tiny numerators end to end: bitwise parity where Markstein's quotient step
alone is not exact (|x| < 2^-970; tests/test_gpu_quotients.py shows the
helpers miss IEEE by an ulp there), with Simulator(exact_subnormal=True): the
stage detects such inputs per tile and divides exactly; the line solves and
k_final divide with the IEEE division (bsq_device.cuh "Tiny numerators"):

  - momenta of 1e-300 down to subnormals everywhere;
  - a coarse shallow channel whose implicit operator couples neighbours so
    weakly that a line solve's far field decays by ~1e-3 per cell into the
    subnormal range and to zero (the solve's per-chunk check).
"""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1909_04153_b200 import boundary as bc
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.grid import Grid, PhysParams, build_bathymetry, still_state

pytestmark = pytest.mark.gpu


def walls():
    return bc.Boundaries(west=bc.Wall(), east=bc.Wall(), south=bc.Wall(), north=bc.Wall())


def run_both(bathy, state, bounds, steps, phys=None, dt_init=0.01, **kw):
    phys = phys or PhysParams()
    sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(dt_init=dt_init),
                            phys=phys, exact_subnormal=True, **kw)
    ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(dt_init=dt_init),
                              phys=phys, threads=4, **kw)
    for k in range(steps):
        a, b = sim.advance(), ora.advance()
        assert (a.dt, a.max_cfl, a.max_speed, a.max_depth) == \
            (b.dt, b.max_cfl, b.max_speed, b.max_depth), k
    for f in ("w", "p", "q"):
        got, want = getattr(sim.state, f), getattr(ora.state, f)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), f
    return sim.state


def test_tiny_and_subnormal_momenta_bitwise():
    rng = np.random.default_rng(5)
    grid = Grid(70, 40, 0.25, 0.25)
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = build_bathymetry(grid, -0.6 + 0.2 * np.exp(-((xc - 8) ** 2 + (yc - 5) ** 2) / 3.0),
                             ws=0.0)
    st = still_state(bathy)
    shape = st.w.shape
    st.w += 0.02 * np.exp(-((np.pad(xc, 2, mode="edge") - 4) ** 2) / 2.0)
    mag = 10.0 ** rng.uniform(-320, -290, shape)  # normal tiny and subnormal
    st.p = mag * rng.choice([-1.0, 1.0], shape)
    st.q = 10.0 ** rng.uniform(-320, -290, shape) * rng.choice([-1.0, 1.0], shape)
    st.p[rng.random(shape) < 0.3] = 0.0
    assert ((st.p != 0) & (np.abs(st.p) < 2.0 ** -970)).any()  # the class is exercised
    run_both(bathy, st, walls(), 12, dt_init=0.01)


def test_far_field_underflow_in_line_solves_bitwise():
    # coarse cells over shallow water: (B + 1/3) d^2 / dx^2 ~ 4e-3, so each
    # Thomas step scales the far field by ~4e-3 -- 1e-300 within ~130 cells
    grid = Grid(600, 6, 0.5, 0.5)
    xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = build_bathymetry(grid, np.full((6, 600), -0.05), ws=0.0)
    st = still_state(bathy)
    st.w += 0.004 * np.exp(-((np.pad(xc, 2, mode="edge") - 10.0) ** 2) / 8.0)
    final = run_both(bathy, st, walls(), 30, dt_init=0.02)
    p = final.p[2:-2, 2:-2]
    assert ((np.abs(p) > 0) & (np.abs(p) < 2.0 ** -970)).any()  # subnormals reached


def test_default_mode_normal_range_bitwise():
    """Default mode on the far-field case: every cell whose reference value
    is 0 or at least 2^-900 in magnitude is bitwise equal; cells below may
    differ by the Markstein quotient's ulp (and what follows from it)."""
    grid = Grid(600, 6, 0.5, 0.5)
    xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = build_bathymetry(grid, np.full((6, 600), -0.05), ws=0.0)
    st = still_state(bathy)
    st.w += 0.004 * np.exp(-((np.pad(xc, 2, mode="edge") - 10.0) ** 2) / 8.0)
    phys = PhysParams()
    sim = stepper.Simulator(bathy, st.copy(), walls(), stepper.TimeController(dt_init=0.02),
                            phys=phys)
    ora = orc.OracleSimulator(bathy, st.copy(), walls(), orc.OController(dt_init=0.02),
                              phys=phys, threads=4)
    for _ in range(30):
        a, b = sim.advance(), ora.advance()
        assert (a.dt, a.max_cfl, a.max_speed, a.max_depth) == \
            (b.dt, b.max_cfl, b.max_speed, b.max_depth)
    for f in ("w", "p", "q"):
        got, want = getattr(sim.state, f), getattr(ora.state, f)
        big = (want == 0) | (np.abs(want) >= 2.0 ** -900)
        assert np.array_equal(got[big].view(np.uint64), want[big].view(np.uint64)), f
        small = ~big
        if small.any():
            assert np.all(np.abs(got[small]) < 2.0 ** -800), f


def test_tiny_momenta_on_y_strips_bitwise():
    """Emulated y-strips (pipeline coupling, bitwise = one grid): tiny
    momenta in halo rows that arrive from another strip are detected by the
    receiving strip's stage tiles too."""
    from paper_1909_04153_b200 import parallel
    rng = np.random.default_rng(11)
    grid = Grid(64, 48, 0.25, 0.25)
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = build_bathymetry(grid, -0.6 + 0.2 * np.exp(-((xc - 8) ** 2 + (yc - 6) ** 2) / 3.0),
                             ws=0.0)
    st = still_state(bathy)
    shape = st.w.shape
    st.w += 0.02 * np.exp(-((np.pad(xc, 2, mode="edge") - 4) ** 2) / 2.0)
    st.p = 10.0 ** rng.uniform(-320, -290, shape) * rng.choice([-1.0, 1.0], shape)
    st.q = 10.0 ** rng.uniform(-320, -290, shape) * rng.choice([-1.0, 1.0], shape)
    phys = PhysParams()
    sim = parallel.ShardedSimulator(bathy, st.copy(), walls(), stepper.TimeController(dt_init=0.01),
                                    phys=phys, exact_subnormal=True, world=3, coupling="pipeline")
    ora = orc.OracleSimulator(bathy, st.copy(), walls(), orc.OController(dt_init=0.01), phys=phys,
                              threads=4)
    for k in range(8):
        a, b = sim.advance(), ora.advance()
        assert (a.dt, a.max_cfl, a.max_speed, a.max_depth) == \
            (b.dt, b.max_cfl, b.max_speed, b.max_depth), k
    for f in ("w", "p", "q"):
        got, want = getattr(sim.state, f), getattr(ora.state, f)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), f


@pytest.mark.parametrize("nx,ny", [(4099, 5), (5000, 6), (1500, 257)])
def test_long_x_lines_paths_bitwise(nx, ny):
    """Few long x lines: the warp-per-line solve up to the shared-memory limit
    (4099 cells: the line's dw on chip), the TMA ring beyond it (5000 cells)
    and above the line-count threshold (257 lines) -- all bitwise vs the
    oracle, ghosts folded at both ends of every line."""
    grid = Grid(nx, ny, 0.05, 0.05)
    xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = build_bathymetry(grid, -0.3 - 0.05 * np.sin(0.01 * xc), ws=0.0)
    st = still_state(bathy)
    st.w += 0.01 * np.exp(-((np.pad(xc, 2, mode="edge") - 0.3 * nx * 0.05) ** 2) / 4.0)
    run_both(bathy, st, walls(), 6, dt_init=0.004)
