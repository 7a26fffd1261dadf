"""Pin the CPU oracle (oracle/bsq_oracle.c + oracle/oracle.py) to the
reference: bitwise against every golden fixture the unmodified reference
produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import golden_cases as gc
from oracle import oracle as orc

II = (slice(2, -2), slice(2, -2))


def _run_oracle(name, threads=None):
    z = gc.load(name)
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    ctrl = orc.OController(**ckw)
    sim = orc.OracleSimulator(bathy, state, bounds, ctrl, phys=phys, threads=threads, **skw)
    recs, abort = [], None
    for _ in range(int(z["steps"])):
        try:
            r = sim.advance()
        except orc.OracleInstability as err:
            abort = (err.step_index, err.sim_time, str(err))
            break
        recs.append((r.step_index, r.sim_time, r.dt, r.max_cfl, r.max_speed, r.max_depth))
    return z, sim, np.array(recs, dtype=np.float64).reshape(-1, 6), abort


@pytest.mark.parametrize("name", gc.RUNS)
def test_oracle_matches_reference_run_bitwise(name):
    z, sim, recs, abort = _run_oracle(name)
    # the whole dt sequence and every record, bit for bit
    assert recs.shape == z["records"].shape
    assert np.array_equal(recs, z["records"])
    st = sim.state
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(st, f)[II], z[f][II]), f
        assert np.array_equal(getattr(st, f), z[f]), f + " (padded, ghost frame included)"
    assert sim.clamped_volume == pytest.approx(float(z["clamped_volume"]), rel=1e-12, abs=1e-300)
    if int(z["abort_step"]) >= 0:
        assert abort is not None and abort[0] == int(z["abort_step"])
        assert abort[1] == float(z["abort_time"])
        assert abort[2] == str(z["abort_msg"])
    else:
        assert abort is None


def test_oracle_thread_count_does_not_change_bits():
    _, a, ra, _ = _run_oracle("maker_sponge", threads=1)
    _, b, rb, _ = _run_oracle("maker_sponge", threads=4)
    assert np.array_equal(ra, rb)
    for f in ("w", "p", "q"):
        assert np.array_equal(getattr(a.state, f), getattr(b.state, f))


def _kernel_inputs():
    z = np.load(gc.GOLDEN + "/kernels.npz")
    from paper_1909_04153_b200.grid import Bathymetry, FieldState, Grid, PhysParams
    grid = Grid(int(z["nx"]), int(z["ny"]), float(z["dx"]), float(z["dy"]))
    bathy = Bathymetry(grid=grid, ws=float(z["ws"]), bed=None, bed_eff=z["bed_eff"],
                       depth=z["depth"], depth_dx=z["depth_dx"], depth_dy=z["depth_dy"],
                       bed_face_x=z["bed_face_x"], bed_face_y=z["bed_face_y"],
                       h_eps=float(z["h_eps"]))
    st = FieldState(z["w"], z["p"], z["q"])
    phys = PhysParams(g=float(z["g"]), b_disp=float(z["b_disp"]), c_f=float(z["c_f"]))
    return z, bathy, st, phys


def test_oracle_stage_kernels_match_reference_bitwise():
    z, bathy, st, phys = _kernel_inputs()
    e, f, g, fs, gs = orc.stage_rates(st, bathy, phys)
    for name, got in (("e", e), ("f", f), ("gg", g), ("fstar", fs), ("gstar", gs)):
        assert np.array_equal(got, z[name]), name


def test_oracle_speed_extrema_match_reference_bitwise():
    z, bathy, st, phys = _kernel_inputs()
    assert np.array_equal(np.array(orc.speed_extrema(st, bathy, phys)), z["extrema"])


def test_oracle_tridiagonal_solvers_match_reference_bitwise():
    z = np.load(gc.GOLDEN + "/kernels.npz")
    assert np.array_equal(orc.thomas_batch(z["dl"], z["dd"], z["du"], z["r"]), z["thomas"])
    assert np.array_equal(orc.cr_batch(z["dl"], z["dd"], z["du"], z["r"]), z["cr"])


def test_oracle_weights_match_reference_bitwise():
    rows = np.load(gc.GOLDEN + "/weights.npz")["rows"]
    for r in rows:
        w = orc.ab3_weights(*r[:3])
        s = orc.increment_weights(*r[:3])
        assert tuple(w) == tuple(r[3:6])
        assert tuple(s) == tuple(r[6:9])


def test_oracle_zero_pivot_raises():
    dl = np.zeros((1, 3))
    dd = np.array([[1.0, 0.0, 1.0]])
    with pytest.raises(ZeroDivisionError):
        orc.thomas_batch(dl, dd, np.zeros((1, 3)), np.ones((1, 3)))


@pytest.mark.parametrize("dl,dd,du,msg", [
    # messages as the reference's cyclic_reduction_batch raises them on these
    # inputs (_kernels.py:419, :439; checked against the reference run here)
    (np.zeros((2, 4)), np.array([[1.0, 1, 1, 1], [0.0, 1, 1, 1]]), np.zeros((2, 4)),
     "singular tridiagonal system in reduction"),
    (np.array([[0.0, 1.0]]), np.array([[1.0, 1.0]]), np.array([[1.0, 0.0]]),
     "singular tridiagonal system: zero core determinant"),
])
def test_oracle_cr_singular_messages(dl, dd, du, msg):
    with pytest.raises(ZeroDivisionError) as exc:
        orc.cr_batch(dl, dd, du, np.ones(dd.shape))
    assert str(exc.value) == msg
