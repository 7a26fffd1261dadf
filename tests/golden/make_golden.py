"""Generate tests/golden/*.npz by running the UNMODIFIED reference solver.

Run in the build container only (needs /root/reference and numba):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Each fixture stores the run's full inputs (static fields, initial state,
boundary specs, controller settings) plus the reference's outputs (final
padded state, every StepRecord, clamped volume, any abort), so tests on the
GPU box -- where /root/reference does not exist -- can rebuild the exact
inputs and compare bit for bit.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from boussim import boundary as rb  # noqa: E402
from boussim import dispersion, hydro, implicit, stepper  # noqa: E402
from boussim import _kernels as rk  # noqa: E402
from boussim import grid as rg  # noqa: E402
from boussim import scenario as rs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SIDES = ("north", "south", "east", "west")


def walls():
    return rb.Boundaries(west=rb.Wall(), east=rb.Wall(), south=rb.Wall(), north=rb.Wall())


def hump(grid, bathy, amp, x0, y0, width):
    st = rg.still_state(bathy)
    xp, yp = grid.x_centers_padded(), grid.y_centers_padded()
    st.w += amp * np.exp(-((xp[None, :] - x0) ** 2 + (yp[:, None] - y0) ** 2) / width ** 2)
    return st


# --------------------------------------------------------------------------
# cases: name -> (bathy, state, boundaries, phys, controller kwargs, sim kwargs, steps)


def case_c1():
    grid = rg.Grid(1024, 5, 0.05, 0.05)
    bathy = rg.build_bathymetry(grid, np.full((5, 1024), -0.32), ws=0.0)
    st = rs.solitary_wave_ic(rs.SolitaryWaveSpec(0.0576, 0.32, crest_x=15.0), bathy)
    return bathy, st, walls(), rg.PhysParams(), dict(dt_init=0.002), {}, 1000


def case_hump(solver="thomas"):
    grid = rg.Grid(26, 18, 0.5, 0.5)
    xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = rg.build_bathymetry(grid, -1.5 - 0.3 * np.sin(0.4 * xc), ws=0.0)
    st = hump(grid, bathy, 0.04, 6.5, 4.5, 1.5)
    return bathy, st, walls(), rg.PhysParams(), dict(dt_init=0.015), dict(solver=solver), 150


def case_maker_sponge():
    grid = rg.Grid(40, 32, 0.25, 0.25, x0=0.0, y0=0.0)
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    bed = -0.6 + 0.25 * np.exp(-((xc - 5.5) ** 2 + (yc - 4.0) ** 2) / 2.0)
    bathy = rg.build_bathymetry(grid, bed, ws=0.0)
    d_west = float(bathy.depth[2:-2, 2].min())
    b = rb.Boundaries(west=rb.SineMaker((rb.sine_component(0.01, 1.2, d_west),)),
                      east=rb.Sponge(2.0, 8.0), south=rb.Sponge(1.0, 5.0), north=rb.Wall())
    return bathy, rg.still_state(bathy), b, rg.PhysParams(), dict(dt_init=0.01), {}, 200


def case_rip_irregular():
    grid = rg.Grid(64, 48, 20.48 / 64, 30.0 / 48, x0=0.0, y0=-15.0)
    bathy = rs.rip_channel_bathymetry(grid)
    d_west = float(bathy.depth[2:-2, 2].min())
    comps = rb.jonswap_components(rb.SpectrumSpec(0.13, 1.6, 68, 0.01, 7), d_west)
    b = rb.Boundaries(west=rb.IrregularMaker(tuple(comps)), east=rb.Wall(), south=rb.Wall(),
                      north=rb.Wall())
    return bathy, rg.still_state(bathy), b, rg.PhysParams(c_f=0.0025), dict(dt_init=0.001), {}, 300


def case_runup():
    grid = rg.Grid(400, 6, 0.05, 0.05)
    xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
    bed = np.where(xc < 12.0, -0.32, -0.32 + (xc - 12.0) / 20.0)
    bathy = rg.build_bathymetry(grid, bed, ws=0.0)
    st = rs.solitary_wave_ic(rs.SolitaryWaveSpec(0.0576, 0.32, crest_x=8.0), bathy)
    return bathy, st, walls(), rg.PhysParams(c_f=0.001), dict(dt_init=0.002), dict(h_dry=1e-3), 3000


def case_dry_clamp():
    grid = rg.Grid(40, 10, 0.5, 0.5)
    xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = rg.build_bathymetry(grid, -1.0 + 0.12 * xc, ws=0.0)
    return bathy, rg.still_state(bathy), walls(), rg.PhysParams(), dict(dt_init=0.01), {}, 120


def case_blowup():
    b = case_hump()
    return b[0], b[1], b[2], b[3], b[4], dict(cross_correction=False), 60


def case_fixed_single_pass():
    grid = rg.Grid(26, 18, 0.5, 0.5)
    xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
    bathy = rg.build_bathymetry(grid, -1.5 - 0.3 * np.sin(0.4 * xc), ws=0.0)
    st = hump(grid, bathy, 0.04, 6.5, 4.5, 1.5)
    return bathy, st, walls(), rg.PhysParams(), dict(dt_init=0.015, mode="fixed"), \
        dict(cross_correction=False), 25


def case_lake():
    grid = rg.Grid(30, 24, 0.5, 0.5)
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    bed = -2.0 + 0.8 * np.exp(-0.2 * ((xc - 6) ** 2 + (yc - 4) ** 2))
    bathy = rg.build_bathymetry(grid, bed, ws=0.0)
    return bathy, rg.still_state(bathy), walls(), rg.PhysParams(), dict(dt_init=0.02), {}, 200


CASES = {
    "c1": case_c1,
    "hump": case_hump,
    "hump_cr": lambda: case_hump("cr"),
    "maker_sponge": case_maker_sponge,
    "rip_irregular": case_rip_irregular,
    "runup": case_runup,
    "dry_clamp": case_dry_clamp,
    "blowup": case_blowup,
    "fixed_single_pass": case_fixed_single_pass,
    "lake": case_lake,
}


def case_island():
    """Maker-driven waves around an emergent island: wet/dry gauges."""
    grid = rg.Grid(40, 32, 0.25, 0.25)
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    bed = -0.6 + 0.9 * np.exp(-((xc - 6.0) ** 2 + (yc - 4.0) ** 2) / 1.5)
    bathy = rg.build_bathymetry(grid, bed, ws=0.0)
    d_west = float(bathy.depth[2:-2, 2].min())
    b = rb.Boundaries(west=rb.SineMaker((rb.sine_component(0.02, 1.0, d_west),)),
                      east=rb.Sponge(2.0, 8.0), south=rb.Wall(), north=rb.Wall())
    return bathy, rg.still_state(bathy), b, rg.PhysParams(), dict(dt_init=0.01), {}, 250


CASES["island"] = case_island

# gauges of the observers fixture: (id, x, y, record_interval); g_dry sits on
# the island (dry), g_shore at its edge, g_sponge inside the east sponge
GAUGES = [("g_west", 1.1, 4.0, 0.0), ("g_shore", 5.0, 4.1, 0.05),
          ("g_dry", 6.0, 4.0, 0.0), ("g_sponge", 9.4, 6.3, 0.2)]


def encode_boundaries(b):
    kinds, comps, sponges = [], [], []
    for k, side in enumerate(SIDES):
        pol = getattr(b, side)
        kinds.append(pol.kind)
        if pol.kind in ("sine", "irregular"):
            for c in pol.components:
                comps.append((k, c.amplitude, c.omega, c.k, c.phase))
        if pol.kind == "sponge":
            sponges.append((k, pol.width, pol.lambda_max))
    return (np.array(kinds), np.array(comps, dtype=np.float64).reshape(-1, 5),
            np.array(sponges, dtype=np.float64).reshape(-1, 3))


def run_case(name):
    bathy, st, b, phys, ckw, skw, steps = CASES[name]()
    init = st.copy()
    ctrl = stepper.TimeController(**ckw)
    sim = stepper.Simulator(bathy, st, b, ctrl, phys=phys, **skw)
    recs, abort = [], None
    for _ in range(steps):
        try:
            r = sim.advance()
        except stepper.InstabilityError as err:
            abort = (err.step_index, err.sim_time, str(err))
            break
        recs.append((r.step_index, r.sim_time, r.dt, r.max_cfl, r.max_speed, r.max_depth))
    kinds, comps, sponges = encode_boundaries(b)
    g = bathy.grid
    out = dict(
        nx=g.nx, ny=g.ny, dx=g.dx, dy=g.dy, x0=g.x0, y0=g.y0, ws=bathy.ws, h_eps=bathy.h_eps,
        bed=bathy.bed[2:-2, 2:-2], bed_eff=bathy.bed_eff, depth=bathy.depth,
        depth_dx=bathy.depth_dx, depth_dy=bathy.depth_dy, bed_face_x=bathy.bed_face_x,
        bed_face_y=bathy.bed_face_y,
        w0=init.w, p0=init.p, q0=init.q,
        side_kinds=kinds, maker_comps=comps, sponges=sponges,
        g=phys.g, b_disp=phys.b_disp, c_f=phys.c_f,
        dt_init=ckw["dt_init"], mode=ckw.get("mode", "adaptive"),
        solver=skw.get("solver", "thomas"), cross_correction=skw.get("cross_correction", True),
        h_dry=skw.get("h_dry", np.nan), steps=steps,
        records=np.array(recs, dtype=np.float64).reshape(-1, 6),
        w=sim.state.w, p=sim.state.p, q=sim.state.q,
        clamped_volume=sim.clamped_volume,
        abort_step=abort[0] if abort else -1, abort_time=abort[1] if abort else np.nan,
        abort_msg=abort[2] if abort else "",
    )
    np.savez_compressed(os.path.join(OUT, f"run_{name}.npz"), **out)
    print(f"{name}: {len(recs)} steps, abort={abort is not None}, "
          f"dt[-1]={recs[-1][2] if recs else None}")


def kernels_fixture():
    """Per-kernel outputs of the reference on random wet/dry states."""
    rng = np.random.default_rng(20261018)
    grid = rg.Grid(23, 17, 0.3, 0.4)
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    bed = -0.8 + 0.9 * np.exp(-((xc - 3.0) ** 2 + (yc - 3.5) ** 2) / 4.0)  # emergent island
    bathy = rg.build_bathymetry(grid, bed, ws=0.0)
    st = rg.still_state(bathy)
    shape = st.w.shape
    st.w = np.maximum(bathy.bed_eff, st.w + 0.05 * rng.standard_normal(shape))
    st.p = 0.1 * rng.standard_normal(shape)
    st.q = 0.1 * rng.standard_normal(shape)
    phys = rg.PhysParams(c_f=0.003)
    stage = dispersion.compute_stages(st, bathy, hydro.NumericsParams(), phys)
    us, vs = dispersion.compute_ustar_vstar(st, bathy, phys)
    ext = hydro.speed_extrema(st, bathy, phys)
    # tridiagonal batches: the implicit operator plus random dominant systems
    coef = implicit.assemble(bathy, phys)
    rhs = rng.standard_normal((grid.ny, grid.nx))
    gw, ge = rng.standard_normal(grid.ny), rng.standard_normal(grid.ny)
    gs, gn = rng.standard_normal(grid.nx), rng.standard_normal(grid.nx)
    px = implicit.solve_x(coef, rhs, gw, ge)
    qy = implicit.solve_y(coef, rhs, gs, gn)
    m, n = 9, 37
    dl = rng.uniform(-1, 1, (m, n))
    du = rng.uniform(-1, 1, (m, n))
    dd = (np.abs(dl) + np.abs(du) + rng.uniform(0.5, 2.0, (m, n))) * rng.choice([-1.0, 1.0], (m, n))
    r = rng.uniform(-5, 5, (m, n))
    th, cr = np.empty((m, n)), np.empty((m, n))
    rk.thomas_batch(dl, dd, du, r, th)
    rk.cyclic_reduction_batch(dl, dd, du, r, cr)
    np.savez_compressed(
        os.path.join(OUT, "kernels.npz"),
        nx=grid.nx, ny=grid.ny, dx=grid.dx, dy=grid.dy, ws=bathy.ws, h_eps=bathy.h_eps,
        bed=bed, bed_eff=bathy.bed_eff, depth=bathy.depth, depth_dx=bathy.depth_dx,
        depth_dy=bathy.depth_dy, bed_face_x=bathy.bed_face_x, bed_face_y=bathy.bed_face_y,
        w=st.w, p=st.p, q=st.q, g=phys.g, b_disp=phys.b_disp, c_f=phys.c_f,
        e=stage.e, f=stage.f, gg=stage.g, fstar=stage.fstar, gstar=stage.gstar,
        ustar=us, vstar=vs, extrema=np.array(ext),
        ax=coef.ax, bx=coef.bx, cx=coef.cx, ay_t=coef.ay_t, by_t=coef.by_t, cy_t=coef.cy_t,
        rhs=rhs, gw=gw, ge=ge, gs=gs, gn=gn, px=px, qy=qy,
        dl=dl, dd=dd, du=du, r=r, thomas=th, cr=cr)
    print("kernels fixture written")


def observers_fixture():
    """The reference run loop's observers (cli.py:621-647): a GaugeRecorder
    and a MaxSurfaceTracker updated before the run and after every step, plus
    the artifact bytes its writers produce (ASCII rasters, dt_history.csv,
    gauge CSVs)."""
    import io
    import tempfile
    from boussim import cli as rc
    bathy, st, b, phys, ckw, skw, steps = case_island()
    sim = stepper.Simulator(bathy, st, b, stepper.TimeController(**ckw), phys=phys, **skw)
    specs = [rs.GaugeSpec(g, x, y, iv) for g, x, y, iv in GAUGES]
    rec = rs.GaugeRecorder(bathy, specs)
    tr = rs.MaxSurfaceTracker(bathy)
    rec.record(sim.state, 0.0)
    tr.update(sim.state)
    for _ in range(steps):
        r = sim.advance()
        rec.record(sim.state, r.sim_time)
        tr.update(sim.state)
    out = {f"series_{g}": rec.series(g) for g, *_ in GAUGES}
    out["cells"] = np.array([rs.gauge_cell(bathy.grid, x, y) for _, x, y, _ in GAUGES])
    out["max_w"] = tr.max_w
    tmp = tempfile.mkdtemp()
    g = bathy.grid
    rg.write_ascii_grid(os.path.join(tmp, "w.asc"), sim.state.w[2:-2, 2:-2], cellsize=g.dx,
                        xll=g.x0, yll=g.y0)
    rg.write_ascii_grid(os.path.join(tmp, "max_w.asc"), tr.max_w, cellsize=g.dx, xll=g.x0,
                        yll=g.y0)
    rc._write_dt_history(tmp, sim.records)
    rec.write_csv(tmp)
    for name in ["w.asc", "max_w.asc", "dt_history.csv"] + [f"gauge_{g}.csv" for g, *_ in GAUGES]:
        with open(os.path.join(tmp, name), "rb") as fh:
            out["file_" + name] = np.frombuffer(fh.read(), dtype=np.uint8)
    # a raster of special values (formatting edge cases)
    rng = np.random.default_rng(11)
    v = rng.standard_normal((7, 9)) * 10.0 ** rng.integers(-320, 300, size=(7, 9))
    v[0, :7] = [np.nan, -np.nan, np.inf, -np.inf, -0.0, 0.0, 5e-324]
    v[1, :3] = [1e16, 123456.0, 0.1]
    rg.write_ascii_grid(os.path.join(tmp, "special.asc"), v, 0.05, xll=-1.5, yll=2.0)
    out["special"] = v
    with open(os.path.join(tmp, "special.asc"), "rb") as fh:
        out["file_special.asc"] = np.frombuffer(fh.read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "observers.npz"), **out)
    print("observers fixture written", {k: v.shape for k, v in out.items() if k.startswith("series")})


def weights_fixture():
    """ab3/increment weights for a spread of step triples (incl. clamped)."""
    from boussim import multistep as rm
    rng = np.random.default_rng(7)
    triples = [(1.0, 2.0, 2.0), (0.01, 0.01, 0.01), (0.002, 0.0028, 0.0021),
               (1.0, 20.0, 0.5), (0.5, 0.01, 3.0)]
    triples += [tuple(rng.uniform(1e-4, 1e-2, 3)) for _ in range(200)]
    rows = []
    for t in triples:
        st = rm.StepTriple(*t)
        w = rm.ab3_weights(st, ratio_policy="clamp")
        s = rm.increment_weights(st, ratio_policy="clamp")
        rows.append(t + w.as_tuple() + tuple(s))
    np.savez_compressed(os.path.join(OUT, "weights.npz"), rows=np.array(rows))
    print("weights fixture written")


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        run_case(nm)
    kernels_fixture()
    weights_fixture()
    observers_fixture()
