"""Speculative next-stage launch (bsq_step_params.spec): bsq_step queues the
next step's ghost + stage kernels behind its finalize, with dt and weights
from a device copy of the controller, and the next step uses them only if
they match the host's own values bit for bit.  Whatever the path, results
(including the ghost frame a caller sees on ``sim.state``) must be exactly
those of the non-speculative step."""

import numpy as np
import pytest

import golden_cases as gc
from paper_1909_04153_b200 import stepper
from paper_1909_04153_b200.scenario import make_case

pytestmark = pytest.mark.gpu


def _pair(z_or_case, **extra):
    sims = []
    for spec in (True, False):
        if isinstance(z_or_case, str):
            z = gc.load(z_or_case)
            bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
            sim = stepper.Simulator(bathy, state, bounds, stepper.TimeController(**ckw),
                                    phys=phys, **skw, **extra)
        else:
            c = z_or_case
            sim = stepper.Simulator(c.bathy, c.state.copy(), c.boundaries,
                                    stepper.TimeController(dt_init=c.dt_init), phys=c.phys,
                                    h_dry=c.h_dry, **extra)
        sim.speculate = spec
        sims.append(sim)
    return sims


def _same_full_state(a, b):
    sa, sb = a.state, b.state
    for f in ("w", "p", "q"):
        x, y = getattr(sa, f), getattr(sb, f)
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64)), f


@pytest.mark.parametrize("name", ["maker_sponge", "rip_irregular", "fixed_single_pass", "runup"])
def test_speculation_is_invisible(name):
    """Same records and the same padded state (ghost frame included, bit
    patterns compared) with and without speculation."""
    a, b = _pair(name)
    z = gc.load(name)
    for _ in range(min(int(z["steps"]), 400)):
        assert a.advance() == b.advance()
    _same_full_state(a, b)


def test_state_reads_between_steps_and_run_truncation():
    """Reading sim.state between steps (lazy ghost restore), a run() whose
    last step is truncated (speculated dt rejected), and a caller-given dt."""
    a, b = _pair(make_case("C3", scale=8))
    for k in range(12):
        ra, rb = a.advance(), b.advance()
        assert ra == rb
        if k % 3 == 0:
            _same_full_state(a, b)
    t_end = a.controller.sim_time + 2.5 * a.controller.dt
    assert a.run(t_end) == b.run(t_end)
    _same_full_state(a, b)
    assert a.advance(0.7 * a.controller.dt) == b.advance(0.7 * b.controller.dt)
    for _ in range(5):
        assert a.advance() == b.advance()
    _same_full_state(a, b)


def test_speculated_parameters_are_used():
    """On a plain adaptive run the device controller agrees with the host:
    the stage kernel is not relaunched (its event disappears from the
    step's kernel list)."""
    c = make_case("C3", scale=8)
    sim = stepper.Simulator(c.bathy, c.state.copy(), c.boundaries,
                            stepper.TimeController(dt_init=c.dt_init), phys=c.phys)
    for _ in range(6):
        sim.advance()
    sim._dev.set_timing(True)
    sim.advance()
    sim.advance()
    names = [n for n, _ in sim._dev.kernel_times()]
    # the queued ghost + stage ran behind the previous step's finalize
    assert names[:2] == ["ghost_t", "stage"], names
    assert names.count("stage") == 1


def test_stage_error_after_speculation_reports_like_no_speculation():
    z = gc.load("hump")
    errs = []
    for spec in (True, False):
        bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
        sim = stepper.Simulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys)
        sim.speculate = spec
        for _ in range(5):
            sim.advance()
        st = sim.state
        st.p[4, 5] = np.inf  # host edit: uploaded before the next step (spec rejected)
        with pytest.raises(stepper.InstabilityError) as e:
            sim.advance()
        errs.append((str(e.value), e.value.state))
    assert errs[0][0] == errs[1][0]
    for f in ("w", "p", "q"):
        x, y = getattr(errs[0][1], f), getattr(errs[1][1], f)
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64)), f


def test_blowup_after_speculation_same_error_state():
    z = gc.load("blowup")
    errs = []
    for spec in (True, False):
        bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
        sim = stepper.Simulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys,
                                **skw)
        sim.speculate = spec
        with pytest.raises(stepper.InstabilityError) as e:
            for _ in range(int(z["steps"])):
                sim.advance()
        errs.append((str(e.value), e.value.state, sim.state))
    assert errs[0][0] == errs[1][0]
    for k in (1, 2):
        for f in ("w", "p", "q"):
            x, y = getattr(errs[0][k], f), getattr(errs[1][k], f)
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64)), (k, f)


def test_rejected_speculation_then_plain_steps_keep_ghosts():
    """A speculation rejected by a caller-given dt, followed by steps that
    queue none: every later state read (its ghost frame included) is the
    non-speculative one -- the frame saved for the rejected speculation
    must not come back when the buffers cycle round to the same slots."""
    for read_each in (False, True):
        a, b = _pair(make_case("C3", scale=8))
        for _ in range(6):
            assert a.advance() == b.advance()
        assert a.advance(0.9 * a.controller.dt) == b.advance(0.9 * b.controller.dt)
        a.speculate = False
        for k in range(1, 10):
            assert a.advance() == b.advance()
            if read_each or k % 6 == 0 or k == 9:
                _same_full_state(a, b)
        a.speculate = True
        for _ in range(4):
            assert a.advance() == b.advance()
            _same_full_state(a, b)


@pytest.mark.parametrize("track_bytes", [64 << 20, 0])
def test_in_place_state_edits_take_effect(track_bytes, monkeypatch):
    """The reference semantics of editing ``sim.state`` in place between
    steps hold on both paths: a pristine copy and a diff (small grids), or
    the write-back of the handed-out arrays (grids above EDIT_TRACK_BYTES,
    forced here with a zero threshold)."""
    from oracle import oracle as orc
    monkeypatch.setattr(stepper.Simulator, "EDIT_TRACK_BYTES", track_bytes)
    z = gc.load("maker_sponge")
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    sim = stepper.Simulator(bathy, state.copy(), bounds, stepper.TimeController(**ckw),
                            phys=phys, **skw)
    ora = orc.OracleSimulator(bathy, state.copy(), bounds, orc.OController(**ckw), phys=phys,
                              **skw)
    for k in range(12):
        if k in (4, 9):
            for s in (sim, ora):
                st = s.state  # the oracle hands out a copy: its edit is set back below
                st.w[10:14, 8:20] += 0.003 * (k + 1)
                st.p[12, 5:9] = -0.001
                if s is ora:
                    ora.set_state(st)
        a, b = sim.advance(), ora.advance()
        assert (a.dt, a.max_cfl, a.max_speed, a.max_depth) == \
            (b.dt, b.max_cfl, b.max_speed, b.max_depth), k
    for f in ("w", "p", "q"):
        x, y = getattr(sim.state, f), getattr(ora.state, f)
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64)), f
