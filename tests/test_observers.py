"""Per-step observers and artifact formats.

CPU: the host paths of observers.py driven by the oracle reproduce the
reference run loop's gauge series and running max (tests/golden/
observers.npz, made by the reference), and the artifact writers produce the
reference's bytes.  GPU: the device observers (gauges sampled by k_final,
max folded by the stage kernel) give the same series and maxima bit for bit.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import golden_cases as gc
from oracle import oracle as orc
from paper_1909_04153_b200 import artifacts as art
from paper_1909_04153_b200 import observers as obs
from paper_1909_04153_b200 import stepper

GAUGES = [("g_west", 1.1, 4.0, 0.0), ("g_shore", 5.0, 4.1, 0.05),
          ("g_dry", 6.0, 4.0, 0.0), ("g_sponge", 9.4, 6.3, 0.2)]


def _fixture():
    return np.load(os.path.join(gc.GOLDEN, "observers.npz"), allow_pickle=False)


def _island():
    z = gc.load("island")
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    return z, bathy, state, bounds, phys, ckw, skw


def _specs():
    return [obs.GaugeSpec(g, x, y, iv) for g, x, y, iv in GAUGES]


def _bytes(z, name):
    return z["file_" + name].tobytes()


def test_gauge_cells_match_reference():
    z = _fixture()
    _, bathy, *_ = _island()
    cells = [obs.gauge_cell(bathy.grid, x, y) for _, x, y, _ in GAUGES]
    assert np.array_equal(np.array(cells), z["cells"])
    with pytest.raises(ValueError):
        obs.gauge_cell(bathy.grid, -5.0, 1.0)
    with pytest.raises(ValueError):
        obs.GaugeSpec("bad", 0.0, 0.0, -1.0)


def test_host_observers_on_oracle_match_reference_run_loop():
    """GaugeRecorder / MaxSurfaceTracker host paths, fed by the oracle."""
    z = _fixture()
    zr, bathy, state, bounds, phys, ckw, skw = _island()
    sim = orc.OracleSimulator(bathy, state, bounds, orc.OController(**ckw), phys=phys)
    rec = obs.GaugeRecorder(bathy, _specs())
    tr = obs.MaxSurfaceTracker(bathy)
    rec.record(sim.state, 0.0)
    tr.update(sim.state)
    for _ in range(int(zr["steps"])):
        r = sim.advance()
        rec.record(sim.state, r.sim_time)
        tr.update(sim.state)
    for g, *_ in GAUGES:
        assert np.array_equal(rec.series(g), z[f"series_{g}"]), g
    assert np.array_equal(tr.max_w, z["max_w"])


def test_ascii_raster_bytes_match_reference(tmp_path):
    z = _fixture()
    art.write_ascii_grid(tmp_path / "special.asc", z["special"], 0.05, xll=-1.5, yll=2.0)
    assert (tmp_path / "special.asc").read_bytes() == _bytes(z, "special.asc")
    art.write_ascii_grid(tmp_path / "max_w.asc", z["max_w"], 0.25)
    assert (tmp_path / "max_w.asc").read_bytes() == _bytes(z, "max_w.asc")
    back = art.load_ascii_grid(tmp_path / "max_w.asc")
    assert np.array_equal(back.values, z["max_w"]) and back.cellsize == 0.25
    # a strided view formats like its contiguous copy
    v = np.arange(60.0).reshape(6, 10) / 7.0
    art.write_ascii_grid(tmp_path / "a.asc", v[:, 2:9], 1.0)
    art.write_ascii_grid(tmp_path / "b.asc", np.ascontiguousarray(v[:, 2:9]), 1.0)
    assert (tmp_path / "a.asc").read_bytes() == (tmp_path / "b.asc").read_bytes()


def test_ascii_loader_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.asc"
    p.write_text("ncols 2\nnrows 2\nxllcorner 0\nyllcorner 0\ncellsize 1\n1 2\n3\n")
    with pytest.raises(ValueError):
        art.load_ascii_grid(p)
    p.write_text("ncols 2\nnrows 1\nxllcorner 0\nyllcorner 0\ncellsize 1\nNODATA_value -9\n1 -9\n")
    with pytest.raises(ValueError):
        art.load_ascii_grid(p)
    p.write_text("ncols 2\nnrows 1\nxllcorner 0\ncellsize 1\n1 2\n")
    with pytest.raises(ValueError):
        art.load_ascii_grid(p)


def test_dt_history_and_gauge_csv_bytes(tmp_path):
    """Writers fed with the reference's own records / series."""
    z = _fixture()
    zr = gc.load("island")
    recs = [stepper.StepRecord(step_index=int(r[0]), sim_time=r[1], dt=r[2], max_cfl=r[3],
                               max_speed=r[4], max_depth=r[5]) for r in zr["records"]]
    art.write_dt_history(str(tmp_path), recs)
    assert (tmp_path / "dt_history.csv").read_bytes() == _bytes(z, "dt_history.csv")
    _, bathy, *_ = _island()
    rec = obs.GaugeRecorder(bathy, _specs())
    for g, *_ in GAUGES:
        rec.samples[g] = [tuple(row) for row in z[f"series_{g}"]]
    rec.write_csv(str(tmp_path))
    for g, *_ in GAUGES:
        assert (tmp_path / f"gauge_{g}.csv").read_bytes() == _bytes(z, f"gauge_{g}.csv"), g


# ---------------------------------------------------------------------------- GPU


def _run_device(sim_factory):
    z = _fixture()
    zr, bathy, state, bounds, phys, ckw, skw = _island()
    sim = sim_factory(bathy, state, bounds, stepper.TimeController(**ckw), phys)
    rec = obs.GaugeRecorder(bathy, _specs())
    tr = obs.MaxSurfaceTracker(bathy)
    rec.record(sim, 0.0)
    tr.update(sim)
    for _ in range(int(zr["steps"])):
        r = sim.advance()
        rec.record(sim, r.sim_time)
        tr.update(sim)
    for g, *_ in GAUGES:
        assert np.array_equal(rec.series(g), z[f"series_{g}"]), g
    assert np.array_equal(tr.max_w, z["max_w"])
    return sim, rec, tr


@pytest.mark.gpu
def test_device_observers_match_reference_run_loop():
    _run_device(lambda b, s, bd, c, ph: stepper.Simulator(b, s, bd, c, phys=ph))


@pytest.mark.gpu
def test_device_observers_sharded_strips():
    from paper_1909_04153_b200.parallel import ShardedSimulator
    _run_device(lambda b, s, bd, c, ph: ShardedSimulator(b, s, bd, c, phys=ph, world=3))


@pytest.mark.gpu
def test_device_max_skips_aborted_step_and_state_edits_count():
    """The tracker folds committed states only: a step that raises is not
    folded (the reference's on_step never runs for it)."""
    z = gc.load("blowup")
    bathy, state, bounds, phys, ckw, skw = gc.inputs(z)
    sim = stepper.Simulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys, **skw)
    tr = obs.MaxSurfaceTracker(bathy)
    host = np.full((bathy.grid.ny, bathy.grid.nx), -np.inf)
    ii = (slice(2, -2), slice(2, -2))
    tr.update(sim)
    np.maximum(host, sim.state.w[ii], out=host)
    with pytest.raises(stepper.InstabilityError):
        for _ in range(int(z["steps"])):
            sim.advance()
            tr.update(sim)
            np.maximum(host, sim.state.w[ii], out=host)
    assert np.array_equal(tr.max_w, host)


@pytest.mark.gpu
def test_snapshots_from_device(tmp_path):
    zr, bathy, state, bounds, phys, ckw, skw = _island()
    sim = stepper.Simulator(bathy, state, bounds, stepper.TimeController(**ckw), phys=phys)
    tr = obs.MaxSurfaceTracker(bathy)
    tr.update(sim)
    for _ in range(20):
        sim.advance()
        tr.update(sim)
    paths = art.write_snapshots(str(tmp_path), art.SNAPSHOT_FIELDS, sim, tr,
                                sim.controller.sim_time)
    assert [os.path.basename(p)[:2] for p in paths] == ["w_", "P_", "Q_", "ma"]
    g = art.load_ascii_grid(paths[0])
    assert np.array_equal(g.values, sim.state.w[2:-2, 2:-2])
    assert np.array_equal(art.load_ascii_grid(paths[3]).values, tr.max_w)
