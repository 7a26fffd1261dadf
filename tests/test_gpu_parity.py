"""Parity of the B200 step (through the C ABI) against the reference.

Bar: bitwise.  The fp64 build reproduces the reference's arithmetic
operation for operation, so every StepRecord (the whole adaptive dt
sequence) and the final eta/P/Q must equal the reference's bit for bit --
far inside north_star's 1e-9 rel-L2 tolerance, which is asserted too.
"""

import math

import numpy as np
import pytest

import golden_cases as gc
from oracle import oracle as orc
from paper_1909_04153_b200 import boundary as bc
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.grid import GHOST, Bathymetry, FieldState, Grid, PhysParams
from paper_1909_04153_b200.scenario import make_case

pytestmark = pytest.mark.gpu
II = (slice(2, -2), slice(2, -2))
REL_L2_TOL = 1e-9  # north_star fp64 bound (BASELINE.json)


def rel_l2(a, b):
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / den if den > 0 else np.linalg.norm(a - b)


def run_sim(sim, steps, err_type=stepper.InstabilityError):
    recs, abort = [], None
    for _ in range(steps):
        try:
            r = sim.advance()
        except err_type as err:
            abort = (err.step_index, err.sim_time, str(err))
            break
        recs.append((r.step_index, r.sim_time, r.dt, r.max_cfl, r.max_speed, r.max_depth))
    return np.array(recs, dtype=np.float64).reshape(-1, 6), abort


@pytest.mark.parametrize("name", gc.RUNS)
def test_golden_run_bitwise(name):
    z = gc.load(name)
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    sim = stepper.Simulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys, **skw)
    recs, abort = run_sim(sim, int(z["steps"]))
    ref = z["records"]
    assert recs.shape == ref.shape
    # identical adaptive dt sequence, step for step
    assert np.array_equal(recs[:, 2], ref[:, 2])
    assert np.array_equal(recs, ref)
    st = sim.state
    for f in ("w", "p", "q"):
        got, want = getattr(st, f)[II], z[f][II]
        assert rel_l2(got, want) <= REL_L2_TOL
        assert np.array_equal(got, want), f
        # the padded arrays a caller sees, ghost frame included
        assert np.array_equal(getattr(st, f), z[f]), f + " (padded)"
    assert sim.clamped_volume == pytest.approx(float(z["clamped_volume"]), rel=1e-12, abs=1e-300)
    if int(z["abort_step"]) >= 0:
        assert abort == (int(z["abort_step"]), float(z["abort_time"]), str(z["abort_msg"]))
    else:
        assert abort is None


def _kernel_setup():
    z = np.load(gc.GOLDEN + "/kernels.npz")
    grid = Grid(int(z["nx"]), int(z["ny"]), float(z["dx"]), float(z["dy"]))
    bathy = Bathymetry(grid=grid, ws=float(z["ws"]), bed=None, bed_eff=z["bed_eff"],
                       depth=z["depth"], depth_dx=z["depth_dx"], depth_dy=z["depth_dy"],
                       bed_face_x=z["bed_face_x"], bed_face_y=z["bed_face_y"],
                       h_eps=float(z["h_eps"]))
    st = FieldState(z["w"].copy(), z["p"].copy(), z["q"].copy())
    phys = PhysParams(g=float(z["g"]), b_disp=float(z["b_disp"]), c_f=float(z["c_f"]))
    walls = bc.Boundaries(west=bc.Wall(), east=bc.Wall(), south=bc.Wall(), north=bc.Wall())
    sim = stepper.Simulator(bathy, st, walls, stepper.TimeController(dt_init=0.01), phys=phys)
    return z, sim


def test_stage_kernel_bitwise_vs_reference_kernels():
    z, sim = _kernel_setup()
    e, f, g, fs, gs = sim._dev.stage_rates()
    for name, got in (("e", e), ("f", f), ("gg", g), ("fstar", fs), ("gstar", gs)):
        assert np.array_equal(got, z[name]), name


def test_speed_extrema_bitwise_vs_reference():
    z, sim = _kernel_setup()
    assert np.array_equal(np.array(sim._dev.speed_extrema()), z["extrema"])
    assert np.array_equal(np.array(sim._extrema), z["extrema"])


def test_line_solves_bitwise_vs_reference():
    z, sim = _kernel_setup()
    p, q = sim._dev.solve_momentum(z["rhs"], z["rhs"], z["gw"], z["ge"], z["gs"], z["gn"])
    assert np.array_equal(p, z["px"])
    assert np.array_equal(q, z["qy"])


@pytest.mark.parametrize("kinds", [("wall", "wall", "wall", "wall"),
                                   ("maker", "sponge", "wall", "maker"),
                                   ("sponge", "maker", "maker", "wall"),
                                   ("maker", "maker", "maker", "maker")])
def test_ghost_fill_matches_oracle_policies(kinds):
    """Corner ownership and every policy combination (boundary.py:316-323)."""
    rng = np.random.default_rng(3)
    grid = Grid(11, 9, 0.3, 0.3)
    from paper_1909_04153_b200.grid import build_bathymetry
    bathy = build_bathymetry(grid, np.full((9, 11), -1.0), ws=0.0)
    comp = bc.WaveComponent(0.01, 2.0, 1.5, 0.3)
    pols = {}
    for side, k in zip(bc.SIDES, kinds):
        pols[side] = {"wall": bc.Wall(), "sponge": bc.Sponge(1.0, 2.0),
                      "maker": bc.SineMaker((comp,))}[k]
    bounds = bc.Boundaries(**pols)
    st = FieldState(rng.normal(size=grid.shape_padded) * 0.01, rng.normal(size=grid.shape_padded),
                    rng.normal(size=grid.shape_padded))
    sim = stepper.Simulator(bathy, st, bounds, stepper.TimeController(dt_init=0.01))
    eta, flux = np.zeros(4), np.zeros(4)
    t = 0.37
    for k, pol in enumerate(sim._policies):
        if bc.policy_kind(pol) == "maker":
            eta[k], flux[k] = bc.maker_surface_flux(pol.components, t)
    sim._dev.fill_ghosts(eta, flux)
    got = sim.state
    ref_state = orc.OState(st.w.copy(), st.p.copy(), st.q.copy())
    # oracle ghost fill through a zero-length run is not exposed; rebuild the
    # reference rule directly (boundary.py:206-261, order N, S, E, W)
    w, p, q = ref_state.w, ref_state.p, ref_state.q
    g = GHOST
    for k, side in enumerate(bc.SIDES):
        if kinds[k] == "maker":
            wv = bathy.ws + eta[k]
            if side == "west":
                w[:, :g], p[:, :g], q[:, :g] = wv, flux[k], 0.0
            elif side == "east":
                w[:, -g:], p[:, -g:], q[:, -g:] = wv, -flux[k], 0.0
            elif side == "south":
                w[:g, :], q[:g, :], p[:g, :] = wv, flux[k], 0.0
            else:
                w[-g:, :], q[-g:, :], p[-g:, :] = wv, -flux[k], 0.0
        else:
            if side in ("west", "east"):
                trip = ((w, 1.0), (q, 1.0), (p, -1.0))
            else:
                trip = ((w, 1.0), (p, 1.0), (q, -1.0))
            for arr, s in trip:
                if side == "west":
                    arr[:, g - 1] = s * arr[:, g]
                    arr[:, g - 2] = s * arr[:, g + 1]
                elif side == "east":
                    arr[:, -g] = s * arr[:, -g - 1]
                    arr[:, -g + 1] = s * arr[:, -g - 2]
                elif side == "south":
                    arr[g - 1, :] = s * arr[g, :]
                    arr[g - 2, :] = s * arr[g + 1, :]
                else:
                    arr[-g, :] = s * arr[-g - 1, :]
                    arr[-g + 1, :] = s * arr[-g - 2, :]
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(got, f), getattr(ref_state, f)), f


def _vs_oracle(case, steps, threads=8, solver="thomas"):
    sim = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                            h_dry=case.h_dry, solver=solver)
    ora = orc.OracleSimulator(case.bathy, case.state.copy(), case.boundaries,
                              orc.OController(dt_init=case.dt_init), phys=case.phys,
                              h_dry=case.h_dry, threads=threads, solver=solver)
    for k in range(steps):
        a, b = sim.advance(), ora.advance()
        assert (a.dt, a.max_cfl, a.max_speed, a.max_depth) == \
            (b.dt, b.max_cfl, b.max_speed, b.max_depth), k
    sa, sb = sim.state, ora.state
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(sa, f)[II], getattr(sb, f)[II]), f
    return sim


def test_shoal_sponges_maker_256_vs_oracle_bitwise():
    _vs_oracle(make_case("C3", scale=4), 60)


def test_rip_irregular_friction_512_vs_oracle_bitwise():
    _vs_oracle(make_case("C4", scale=8), 40)


def test_cyclic_reduction_solver_256_vs_oracle_bitwise():
    """solver="cr" (cyclic_reduction_batch, _kernels.py:384-451), 256^2 with
    sponges and a maker; non-power-of-two lines exercise the identity padding."""
    _vs_oracle(make_case("C3", scale=4), 30, solver="cr")
    _vs_oracle(make_case("C4", scale=12), 10, solver="cr")


def test_rip_4096_full_size_vs_oracle_bitwise():
    """Full north_star size (4096^2, the bench workload), bit for bit over
    the 3 Euler bootstrap steps and 50 AB3 steps (speculative stage on)."""
    import os
    _vs_oracle(make_case("C4"), 53, threads=len(os.sched_getaffinity(0)) or 8)


def test_lake_at_rest_full_size_is_fixed_point():
    """Well-balance at 4096^2 (size-independent property, the reference's
    test_stepper.py:265-275 scaled up): a lake at rest over a submerged
    bump with walls stays at rest."""
    from paper_1909_04153_b200.grid import build_bathymetry, still_state
    n = 4096
    grid = Grid(n, n, 30.0 / n, 24.0 / n)
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = build_bathymetry(grid, -2.0 + 0.8 * np.exp(-0.2 * ((xc - 12) ** 2 + (yc - 8) ** 2)),
                             ws=0.0)
    state = still_state(bathy)
    walls = bc.Boundaries(west=bc.Wall(), east=bc.Wall(), south=bc.Wall(), north=bc.Wall())
    sim = stepper.Simulator(bathy, state.copy(), walls, stepper.TimeController(dt_init=0.002))
    for _ in range(10):
        sim.advance()
    st = sim.state
    assert np.max(np.abs(st.w[II] - state.w[II])) <= 1e-12
    assert np.max(np.abs(st.p[II])) <= 1e-12 and np.max(np.abs(st.q[II])) <= 1e-12


def test_nonfinite_state_aborts_with_location():
    z = gc.load("hump")
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    sim = stepper.Simulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys)
    ora = orc.OracleSimulator(bathy, gc.inputs(z)[1], bounds, orc.OController(**ckw), phys=phys)
    sim.advance()
    ora.advance()
    sim.state.p[GHOST + 2, GHOST + 3] = np.inf   # edit the host copy, as the reference test does
    st = ora.state
    st.p[GHOST + 2, GHOST + 3] = np.inf
    ora.set_state(st)
    with pytest.raises(orc.OracleInstability) as want:
        ora.advance()
    with pytest.raises(stepper.InstabilityError) as got:
        sim.advance()
    # the first non-finite stage cell in row-major order, as the reference reports it
    assert str(got.value) == str(want.value)
    assert got.value.step_index == want.value.step_index == 2


def test_singular_operator_raises_zero_division():
    grid = Grid(8, 6, 1.0, 1.0)
    from paper_1909_04153_b200.grid import build_bathymetry
    bathy = build_bathymetry(grid, np.full((6, 8), -1.0), ws=0.0)
    # b = 1 + 2 (B + 1/3) d^2/dx^2 is exactly 0 for this B (d = dx = 1)
    phys = PhysParams(b_disp=-0.8333333333333334)
    walls = bc.Boundaries(west=bc.Wall(), east=bc.Wall(), south=bc.Wall(), north=bc.Wall())
    with pytest.warns(UserWarning):
        sim = stepper.Simulator(bathy, FieldState(*[a.copy() for a in (
            np.maximum(0.0, bathy.bed_eff), np.zeros(grid.shape_padded),
            np.zeros(grid.shape_padded))]), walls, stepper.TimeController(dt_init=0.01),
            phys=phys)
    with pytest.raises(ZeroDivisionError):
        sim.advance()


def test_singular_operator_cr_reports_reduction():
    """solver="cr" raises the reference's reduction-phase message
    (_kernels.py:419), like the oracle on the same inputs."""
    grid = Grid(8, 6, 1.0, 1.0)
    from paper_1909_04153_b200.grid import build_bathymetry
    bathy = build_bathymetry(grid, np.full((6, 8), -1.0), ws=0.0)
    phys = PhysParams(b_disp=-0.8333333333333334)
    walls = bc.Boundaries(west=bc.Wall(), east=bc.Wall(), south=bc.Wall(), north=bc.Wall())
    mk = lambda: FieldState(np.maximum(0.0, bathy.bed_eff), np.zeros(grid.shape_padded),
                            np.zeros(grid.shape_padded))
    with pytest.warns(UserWarning):
        sim = stepper.Simulator(bathy, mk(), walls, stepper.TimeController(dt_init=0.01),
                                phys=phys, solver="cr")
    ora = orc.OracleSimulator(bathy, mk(), walls, orc.OController(dt_init=0.01), phys=phys,
                              solver="cr")
    with pytest.raises(ZeroDivisionError) as want:
        ora.advance()
    with pytest.raises(ZeroDivisionError) as got:
        sim.advance()
    assert str(got.value) == str(want.value) == "singular tridiagonal system in reduction"


def test_pending_rollback_keeps_committed_state():
    """A step that raises is not committed (reference: self.state unchanged)."""
    z = gc.load("blowup")
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    sim = stepper.Simulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys, **skw)
    abort_step = int(z["abort_step"])
    for _ in range(abort_step - 1):
        sim.advance()
    before = sim.state
    w0 = before.w.copy()
    with pytest.raises(stepper.InstabilityError) as exc:
        sim.advance()
    assert exc.value.step_index == abort_step
    assert np.array_equal(sim.state.w[II], w0[II])
    assert math.isfinite(sim.controller.dt)
