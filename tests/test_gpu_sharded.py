"""y-strip sharding on one GPU: ranks emulated in one
process (LocalComm), so the multi-rank exchange logic runs for real.  Bar:
bitwise equal to the reference golden runs / the single-GPU path -- the
sharded step performs the single-GPU operation sequence exactly."""

import numpy as np
import pytest

import golden_cases as gc
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.parallel import ShardedSimulator, split_rows, strip_band
from paper_1909_04153_b200.scenario import make_case

pytestmark = pytest.mark.gpu
II = (slice(2, -2), slice(2, -2))


@pytest.mark.parametrize("name,world", [("hump", 2), ("maker_sponge", 3), ("maker_sponge", 4),
                                        ("rip_irregular", 2), ("rip_irregular", 5),
                                        ("lake", 2), ("dry_clamp", 2), ("blowup", 2)])
def test_sharded_golden_run_bitwise(name, world):
    z = gc.load(name)
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    sim = ShardedSimulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys,
                           world=world, **skw)
    recs, abort = [], None
    for _ in range(int(z["steps"])):
        try:
            r = sim.advance()
        except stepper.InstabilityError as err:
            abort = (err.step_index, err.sim_time, str(err))
            break
        recs.append((r.step_index, r.sim_time, r.dt, r.max_cfl, r.max_speed, r.max_depth))
    recs = np.array(recs, dtype=np.float64).reshape(-1, 6)
    assert np.array_equal(recs, z["records"])
    st = sim.state
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(st, f)[II], z[f][II]), f
    assert sim.clamped_volume == pytest.approx(float(z["clamped_volume"]), rel=1e-12, abs=1e-300)
    if int(z["abort_step"]) >= 0:
        assert abort == (int(z["abort_step"]), float(z["abort_time"]), str(z["abort_msg"]))


def test_sharded_rip_512_matches_single_gpu_bitwise():
    case = make_case("C4", scale=8)
    one = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys)
    four = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys, world=4)
    for _ in range(30):
        a, b = one.advance(), four.advance()
        assert a == b
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(one.state, f), getattr(four.state, f)), f


def test_split_rows_and_bands():
    assert split_rows(10, 2) == [(0, 5), (5, 5)]
    assert split_rows(11, 2) == [(0, 6), (6, 5)]
    with pytest.raises(ValueError):
        split_rows(9, 2)
    # a 6-row north band over strips of 5 rows at rows 0, 5, 10 (ny = 15): rows 9..14
    assert strip_band(9, 6, 10, 5) == (0, 5, 1)
    assert strip_band(9, 6, 5, 5) == (4, 1, 0)
    assert strip_band(9, 6, 0, 5) == (0, 0, 0)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_spike_coupled_strips_match_single_gpu(world):
    """coupling="spike" (partitioned y-solves, ranks concurrent): the same
    solution up to rounding.  Bar: <= 1e-12 relative after 30
    adaptive steps, and the same dt sequence to 1e-12."""
    case = make_case("C4", scale=8)
    one = stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                            stepper.TimeController(dt_init=case.dt_init), phys=case.phys)
    sp = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries,
                          stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                          world=world, coupling="spike")
    for _ in range(30):
        a, b = one.advance(), sp.advance()
        assert b.dt == pytest.approx(a.dt, rel=1e-12)
        assert b.max_speed == pytest.approx(a.max_speed, rel=1e-12)
    sa, sb = one.state, sp.state
    assert _rel(sb.w[II], sa.w[II]) <= 1e-12
    # momenta against the larger of the two fields (Q is ~0 in 1-D-like parts)
    scale = max(np.linalg.norm(sa.p[II]), np.linalg.norm(sa.q[II]))
    for f in ("p", "q"):
        assert np.linalg.norm(getattr(sb, f)[II] - getattr(sa, f)[II]) / scale <= 1e-12, f


def test_spike_coupled_strips_golden_maker_sponge():
    """Sponges on N/S rows split across strips, maker on the west edge: the
    reference's own run to <= 1e-12 after 200 steps, same step count."""
    z = gc.load("maker_sponge")
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    sim = ShardedSimulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys,
                           world=4, coupling="spike", **skw)
    dts = [sim.advance().dt for _ in range(int(z["steps"]))]
    assert np.allclose(dts, z["records"][:, 2], rtol=1e-12, atol=0)
    st = sim.state
    assert _rel(st.w[II], z["w"][II]) <= 1e-12
    scale = max(np.linalg.norm(z["p"][II]), np.linalg.norm(z["q"][II]))
    for f in ("p", "q"):
        assert np.linalg.norm(getattr(st, f)[II] - z[f][II]) / scale <= 1e-12, f


@pytest.mark.parametrize("coupling,world", [("pipeline", 3), ("spike", 2)])
def test_fp32_strips_match_single_grid_fp32(coupling, world):
    """precision="fp32" on y-strips (the fp32 line of the multi-GPU bench):
    the rank pipeline performs the one-grid fp32 operations exactly (bitwise
    against the single-grid fp32 run), the spike coupling within fp32
    rounding of it; and the strip run stays within the fp32 contract of the
    fp64 one-grid reference (eta rel-L2 <= 1e-4, same wet mask)."""
    case = make_case("C4", scale=8)

    def mk(cls=stepper.Simulator, precision="fp32", **kw):
        return cls(case.bathy, case.state.copy(), case.boundaries,
                   stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                   precision=precision, **kw)
    one32, one64 = mk(), mk(precision="fp64")
    sp = mk(ShardedSimulator, world=world, coupling=coupling)
    for _ in range(30):
        a, b = one32.advance(), sp.advance()
        one64.advance()
        if coupling == "pipeline":
            assert (a.dt, a.max_cfl, a.max_speed) == (b.dt, b.max_cfl, b.max_speed)
    sa, sb, s64 = one32.state, sp.state, one64.state
    if coupling == "pipeline":
        for f in ("w", "p", "q"):
            assert np.array_equal(getattr(sa, f), getattr(sb, f)), f
    else:
        assert _rel(sb.w[II], sa.w[II]) <= 1e-6
    rest = np.maximum(case.bathy.ws, case.bathy.bed_eff)
    assert _rel((sb.w - rest)[II], (s64.w - rest)[II]) <= 1e-4
    bed32 = case.bathy.bed_eff.astype(np.float32).astype(np.float64)
    h = sp.h_dry
    assert np.array_equal((sb.w - bed32)[II] > h, (s64.w - case.bathy.bed_eff)[II] > h)


@pytest.mark.parametrize("coupling,world", [("pipeline", 3), ("spike", 2)])
def test_strip_speculation_changes_no_bit(coupling, world):
    """Strips queue the next step's ghosts and inner stage rows on the rank-
    reduced CFL rate (BSQ_PH_FINAL_LAUNCH); the run with speculation equals the
    run without it bit for bit, with state reads (ghost frame restores) and an
    in-place edit in between."""
    case = make_case("C4", scale=8)

    def run(spec):
        sim = ShardedSimulator(case.bathy, case.state.copy(), case.boundaries,
                               stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                               world=world, coupling=coupling)
        sim.speculate = spec
        recs = []
        for k in range(24):
            recs.append(sim.advance())
            if k in (5, 11):
                st = sim.state
                _ = st.w.sum()
            if k == 15:
                sim.state.p[200:210, 300:310] *= 0.5
        out = (recs, [getattr(sim.state, f).copy() for f in ("w", "p", "q")])
        sim.close()
        return out

    r1, s1 = run(True)
    r0, s0 = run(False)
    assert r1 == r0
    for a, b in zip(s1, s0):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
