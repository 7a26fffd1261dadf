"""Drop-in fidelity against the reference package's own objects (CPU).

The GPU box has no boussim; these run in the build container, where the
unmodified reference imports from /root/reference (numba, lazily compiled),
and are skipped elsewhere:

  - a Simulator built from boussim's Grid / Bathymetry / FieldState /
    Boundaries / TimeController / PhysParams hands the device exactly the
    descriptor, static fields, initial state and per-side forcing it gets
    from this package's own objects (the device itself is replaced by a
    recorder, so no GPU is needed -- the GPU suite proves those inputs give
    the reference's bits);
  - with boussim importable, InstabilityError is a subclass of
    boussim.stepper.InstabilityError, so cli.py:654's except clause catches
    it after INTEGRATION.md's one-line swap.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


class _Recorder:
    """Stands in for DeviceStep: records what the Simulator hands the device."""

    def __init__(self, desc, bathy):
        self.desc = bytes(memoryview(desc))
        self.static = {k: np.array(getattr(bathy, k), copy=True)
                       for k in ("bed_eff", "depth", "depth_dx", "depth_dy", "bed_face_x",
                                 "bed_face_y")}
        self.workspace = None
        self.uploads = []

    def upload(self, w, p, q):
        self.uploads.append(tuple(np.array(a, copy=True) for a in (w, p, q)))

    def speed_extrema(self):
        return (0.0, 0.0, 0.0)

    def __getattr__(self, name):  # anything else the constructor touches
        return lambda *a, **k: None


def _build(mod_grid, mod_bc, mod_stepper_ctrl, case):
    """One case from either package: (bathy, state, boundaries, controller, phys, kw)."""
    g = mod_grid
    if case == "maker_sponge":
        grid = g.Grid(40, 32, 0.25, 0.25, x0=0.0, y0=0.0)
        xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
        bathy = g.build_bathymetry(grid, -0.6 + 0.25 * np.exp(-((xc - 5.5) ** 2 + (yc - 4.0) ** 2)
                                                               / 2.0), ws=0.0)
        d_west = float(bathy.depth[2:-2, 2].min())
        b = mod_bc.Boundaries(west=mod_bc.SineMaker((mod_bc.sine_component(0.01, 1.2, d_west),)),
                              east=mod_bc.Sponge(2.0, 8.0), south=mod_bc.Sponge(1.0, 5.0),
                              north=mod_bc.Wall())
        return bathy, g.still_state(bathy), b, mod_stepper_ctrl(dt_init=0.01), g.PhysParams(), {}
    if case == "jonswap_beach":
        grid = g.Grid(48, 24, 0.5, 0.5)
        xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
        bathy = g.build_bathymetry(grid, -0.8 + 0.03 * xc, ws=0.0)
        d_west = float(bathy.depth[2:-2, 2].min())
        comps = mod_bc.jonswap_components(mod_bc.SpectrumSpec(0.05, 1.6, 16, 0.02, 3), d_west)
        b = mod_bc.Boundaries(west=mod_bc.IrregularMaker(tuple(comps)), east=mod_bc.Wall(),
                              south=mod_bc.Sponge(2.0, 6.0), north=mod_bc.Wall())
        return (bathy, g.still_state(bathy), b, mod_stepper_ctrl(dt_init=0.005, cfl_target=0.2),
                g.PhysParams(c_f=0.003), dict(h_dry=1e-3, cross_correction=False))
    raise ValueError(case)


@pytest.mark.parametrize("case", ["maker_sponge", "jonswap_beach"])
def test_boussim_objects_give_identical_device_inputs(case, monkeypatch):
    sys.path.insert(0, REF)
    try:
        from boussim import boundary as rb, grid as rg, stepper as rstep
    finally:
        sys.path.remove(REF)
    from paper_1909_04153_b200 import boundary as bc, grid as og, stepper

    recs = []
    monkeypatch.setattr(stepper.Simulator, "_make_device",
                        lambda self, desc, bathy, device: recs.append(_Recorder(desc, bathy))
                        or recs[-1])
    sims = []
    for mg, mb, ctrl in ((rg, rb, rstep.TimeController), (og, bc, stepper.TimeController)):
        bathy, st, b, c, phys, kw = _build(mg, mb, ctrl, case)
        sims.append(stepper.Simulator(bathy, st, b, c, phys=phys, **kw))
    ref, own = recs
    assert ref.desc == own.desc
    for k in ref.static:
        assert np.array_equal(ref.static[k].view(np.uint64), own.static[k].view(np.uint64)), k
    for a, b in zip(ref.uploads[0], own.uploads[0]):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    s_ref, s_own = sims
    assert s_ref.blowup_bound == s_own.blowup_bound and s_ref._chain == s_own._chain
    for r1, r2 in zip(s_ref._maker_rows, s_own._maker_rows):
        assert (r1 is None) == (r2 is None)
        if r1 is not None:
            assert np.array_equal(r1, r2)
    for b1, b2 in zip(s_ref._bands, s_own._bands):
        assert (b1 is None) == (b2 is None)
        if b1 is not None:
            assert np.array_equal(b1[0], b2[0]) and b1[1:] == b2[1:]
    # the per-step forcing the host sends: wavemaker sums and sponge factors
    for sim in sims:
        sim.controller.dt_prev, sim.controller.dt_prev2 = 0.0045, 0.005
        sim._fill_params(0.37, 0.004, euler=False)
    p1, p2 = (bytes(memoryview(s._params)) for s in sims)
    f1 = [s._fac_keep for s in sims]
    for k in range(4):
        assert (f1[0][k] is None) == (f1[1][k] is None)
        if f1[0][k] is not None:
            assert np.array_equal(f1[0][k], f1[1][k])
    # sponge factor pointers differ between the two; everything else is equal
    n_ptr = 4 * ctypes.sizeof(ctypes.c_void_p)
    from paper_1909_04153_b200 import _native as nat
    off = nat.StepParams.sponge_fac.offset
    assert p1[:off] == p2[:off] and p1[off + n_ptr:] == p2[off + n_ptr:]


def test_instability_error_is_boussims_when_importable():
    code = (
        "import boussim.stepper as r\n"
        "from paper_1909_04153_b200 import stepper as s\n"
        "assert issubclass(s.InstabilityError, r.InstabilityError)\n"
        "try:\n"
        "    raise s.InstabilityError('x', step_index=3, sim_time=0.5)\n"
        "except r.InstabilityError as e:\n"
        "    assert (e.step_index, e.sim_time, e.state) == (3, 0.5, None)\n"
        "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]),
               NUMBA_CACHE_DIR="/tmp/numba_cache")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr[-2000:]
