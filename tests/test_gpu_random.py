"""Randomized parity (the reference's property-test style):
seeded random configurations -- grid shapes that are not multiples of any
tile size, beds with emergent islands and beaches, every side policy
(wall, sine maker, irregular maker, sponge), friction, film cutoff, cross
correction on/off, both solvers, adaptive and fixed dt, fp64 -- each run
40 steps on the device and on the CPU oracle and compared bit for bit:
records (dt, CFL, speed, depth), the padded state and the clamped volume."""

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1909_04153_b200 import boundary as bc
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.grid import Grid, PhysParams, build_bathymetry, still_state

pytestmark = pytest.mark.gpu
SEEDS = list(range(int(__import__("os").environ.get("BSQ_RANDOM_SEEDS", "40"))))


def _config(seed):
    rng = np.random.default_rng(1000 + seed)
    nx, ny = int(rng.integers(5, 90)), int(rng.integers(5, 70))
    dx, dy = float(rng.uniform(0.1, 0.6)), float(rng.uniform(0.1, 0.6))
    grid = Grid(nx, ny, dx, dy, x0=float(rng.uniform(-3, 3)), y0=float(rng.uniform(-3, 3)))
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    depth0 = float(rng.uniform(0.3, 1.5))
    bed = -depth0 + 0.15 * np.sin(rng.uniform(0.2, 1.0) * xc + rng.uniform(0, 6))
    if rng.random() < 0.5:  # an emergent island
        cx = grid.x0 + rng.uniform(0.3, 0.7) * nx * dx
        cy = grid.y0 + rng.uniform(0.3, 0.7) * ny * dy
        bed = bed + (depth0 + 0.3) * np.exp(-((xc - cx) ** 2 + (yc - cy) ** 2)
                                            / rng.uniform(0.5, 3.0))
    if rng.random() < 0.3:  # a beach on the east
        bed = np.maximum(bed, -depth0 + 0.8 * (xc - grid.x0 - 0.6 * nx * dx))
    bathy = build_bathymetry(grid, bed, ws=0.0)
    state = still_state(bathy)
    # a hump of water where it is wet
    r2 = ((xc - xc.mean()) ** 2 + (yc - yc.mean()) ** 2) / max(dx * nx, dy * ny) ** 2
    hump = float(rng.uniform(0.0, 0.05)) * np.exp(-20 * r2)
    ii = grid.interior
    wet = state.w[ii] > bathy.bed_eff[ii]
    state.w[ii] = np.where(wet, state.w[ii] + hump, state.w[ii])

    g = 2
    edge = {"west": bathy.depth[g:-g, g], "east": bathy.depth[g:-g, -g - 1],
            "south": bathy.depth[g, g:-g], "north": bathy.depth[-g - 1, g:-g]}
    pols = {}
    for side in bc.SIDES:
        cell = dx if side in ("west", "east") else dy
        n_cells = nx if side in ("west", "east") else ny
        choices = ["wall", "sponge"] if 2.0 * cell < 0.5 * n_cells * cell else ["wall"]
        if edge[side].min() > 0.05:
            choices += ["sine", "irregular"]
        kind = choices[int(rng.integers(len(choices)))]
        if kind == "wall":
            pols[side] = bc.Wall()
        elif kind == "sponge":
            pols[side] = bc.Sponge(float(rng.uniform(2.0 * cell, 0.4 * n_cells * cell)),
                                   float(rng.uniform(1.0, 12.0)))
        elif kind == "sine":
            pols[side] = bc.SineMaker((bc.sine_component(float(rng.uniform(0.002, 0.02)),
                                                         float(rng.uniform(0.8, 2.5)),
                                                         float(edge[side].min())),))
        else:
            spec = bc.SpectrumSpec(float(rng.uniform(0.01, 0.04)), float(rng.uniform(1.0, 2.0)),
                                   int(rng.integers(4, 20)), 0.02, int(rng.integers(100)))
            pols[side] = bc.IrregularMaker(tuple(bc.jonswap_components(spec,
                                                                       float(edge[side].min()))))
    bounds = bc.Boundaries(**pols)
    phys = PhysParams(c_f=float(rng.choice([0.0, 0.002, 0.01])))
    skw = dict(cross_correction=bool(rng.random() < 0.8),
               solver="cr" if rng.random() < 0.25 else "thomas",
               h_dry=float(rng.choice([0.0, 1e-4, 1e-3])) if rng.random() < 0.5 else None)
    mode = "fixed" if rng.random() < 0.2 else "adaptive"
    ckw = dict(dt_init=float(rng.uniform(0.002, 0.01)), mode=mode)
    return bathy, state, bounds, phys, ckw, skw


@pytest.mark.parametrize("seed", SEEDS)
def test_random_configuration_bitwise_vs_oracle(seed):
    bathy, state, bounds, phys, ckw, skw = _config(seed)
    sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw),
                            phys=phys, **skw)
    ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(**ckw), phys=phys,
                              **skw)
    err_a = err_b = None
    for k in range(40):
        try:
            a = sim.advance()
        except (stepper.InstabilityError, ZeroDivisionError) as e:
            err_a = (type(e).__name__, str(e))
        try:
            b = ora.advance()
        except (orc.OracleInstability, ZeroDivisionError) as e:
            err_b = (type(e).__name__.replace("OracleInstability", "InstabilityError"), str(e))
        assert (err_a is None) == (err_b is None), (k, err_a, err_b)
        if err_a:
            assert err_a == err_b
            return
        assert (a.dt, a.max_cfl, a.max_speed, a.max_depth) == \
            (b.dt, b.max_cfl, b.max_speed, b.max_depth), k
    sa, sb = sim.state, ora.state
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(sa, f), getattr(sb, f)), f
    assert sim.clamped_volume == pytest.approx(ora.clamped_volume, rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("seed", [s for s in SEEDS if s % 3 == 0])
def test_random_configuration_sharded_bitwise_vs_oracle(seed):
    """The same configurations on 2-3 emulated y-strips (rank-pipelined
    column solves): still the oracle's bits."""
    from paper_1909_04153_b200.parallel import ShardedSimulator
    bathy, state, bounds, phys, ckw, skw = _config(seed)
    if skw["solver"] == "cr":
        skw["solver"] = "thomas"  # strips run the Thomas pipeline
    world = 3 if bathy.grid.ny >= 15 else 2
    if bathy.grid.ny < 5 * world:
        pytest.skip("too few rows for the strips")
    sim = ShardedSimulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw),
                           phys=phys, world=world, **skw)
    ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(**ckw), phys=phys,
                              **skw)
    for k in range(30):
        try:
            a = sim.advance()
        except stepper.InstabilityError:
            with pytest.raises(orc.OracleInstability):
                ora.advance()
            return
        b = ora.advance()
        assert (a.dt, a.max_cfl, a.max_speed, a.max_depth) == \
            (b.dt, b.max_cfl, b.max_speed, b.max_depth), k
    ii = bathy.grid.interior
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(sim.state, f)[ii], getattr(ora.state, f)[ii]), f


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("seed", [s for s in SEEDS if s % 4 == 1])
def test_random_configuration_spike_strips_vs_oracle(seed):
    """coupling="spike" on random configurations: <= 1e-12 relative to the
    oracle after 30 steps (same dt sequence to 1e-12)."""
    from paper_1909_04153_b200.parallel import ShardedSimulator
    bathy, state, bounds, phys, ckw, skw = _config(seed)
    skw["solver"] = "thomas"
    world = 3 if bathy.grid.ny >= 15 else 2
    if bathy.grid.ny < 5 * world:
        pytest.skip("too few rows for the strips")
    sim = ShardedSimulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw),
                           phys=phys, world=world, coupling="spike", **skw)
    ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(**ckw), phys=phys,
                              **skw)
    for k in range(30):
        try:
            a = sim.advance()
        except stepper.InstabilityError:
            # the coupled strips agree with one grid to ~1e-15: the oracle
            # must abort at the same step
            with pytest.raises(orc.OracleInstability):
                ora.advance()
            return
        b = ora.advance()
        assert a.dt == pytest.approx(b.dt, rel=1e-12), k
    ii = bathy.grid.interior
    sa, sb = sim.state, ora.state
    assert _rel(sa.w[ii], sb.w[ii]) <= 1e-12
    scale = max(np.linalg.norm(sb.p[ii]), np.linalg.norm(sb.q[ii]), 1e-300)
    for f in ("p", "q"):
        assert np.linalg.norm(getattr(sa, f)[ii] - getattr(sb, f)[ii]) / scale <= 1e-10, f


@pytest.mark.parametrize("seed", [s for s in SEEDS if s % 4 == 2])
def test_random_configuration_fp32_vs_oracle(seed):
    """precision="fp32" on random configurations: eta rel-L2 <= 1e-4 against
    the fp64 oracle after 30 steps (fixed dt, so both take the same steps),
    both solvers, and an identical wet mask w - bed_eff > h_dry.  A device
    abort must be an oracle abort within a step or two (fp32 rounding can
    move a blow-up across the bound one step earlier or later)."""
    bathy, state, bounds, phys, ckw, skw = _config(seed)
    ckw = dict(ckw, mode="fixed")
    sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw),
                            phys=phys, precision="fp32", **skw)
    ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(**ckw), phys=phys,
                              **skw)
    for k in range(30):
        try:
            sim.advance()
        except stepper.InstabilityError:
            with pytest.raises(orc.OracleInstability):
                for _ in range(3):
                    ora.advance()
            return
        try:
            ora.advance()
        except orc.OracleInstability:
            # the oracle blew up first: the device must follow within a step
            with pytest.raises(stepper.InstabilityError):
                for _ in range(2):
                    sim.advance()
            return
    ii = bathy.grid.interior
    eta_a = sim.state.w[ii] - bathy.ws
    eta_b = ora.state.w[ii] - bathy.ws
    r = _rel(eta_a, eta_b)
    print(f"seed {seed} ({skw['solver']}): fp32 eta rel-L2 {r:.3e}")
    assert r <= 1e-4
    # the fp32 run's wetness is judged against its own (float-rounded) bed:
    # a dry cell holds w == float(bed_eff) exactly, which sits a rounding
    # step above or below the fp64 bed (tools/diag_fp32_mask.py, seed 50)
    h_dry = sim.h_dry
    bed32 = bathy.bed_eff.astype(np.float32).astype(np.float64)
    assert np.array_equal((sim.state.w - bed32)[ii] > h_dry,
                          (ora.state.w - bathy.bed_eff)[ii] > h_dry)
