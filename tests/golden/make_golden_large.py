"""Goldens of the BASELINE configurations at their stated sizes, from the
UNMODIFIED reference solver (build container only: needs /root/reference and
numba):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_large.py [c2 c3 c3j]

  c2   C2: 2048 x 64 plane-beach runup, h_dry = 1e-3, 6000 adaptive steps
       (BASELINE configs[1])
  c3   C3: 1024 x 1024 elliptic shoal, sine maker + sponges, 400 steps
  c3j  C3 with the irregular (JONSWAP) maker, 400 steps

The inputs are rebuilt on the GPU box by paper_1909_04153_b200.scenario
.make_case (whose generators are pinned bitwise to the reference's by
tests/test_abi_host.py and the test below re-checks a digest of them), so a
fixture stores only outputs: every StepRecord, the SHA-256 of the final
padded w, P, Q (ghost frame included) -- the bitwise check -- and, for C2,
the final surface deviation eta in float32 plus the wet mask for the fp32-mode
check.
The reference objects are built with the reference's own API and the same
expressions as scenario.make_case.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from boussim import boundary as rb  # noqa: E402
from boussim import grid as rg  # noqa: E402
from boussim import scenario as rs  # noqa: E402
from boussim import stepper  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def walls():
    return rb.Boundaries(west=rb.Wall(), east=rb.Wall(), south=rb.Wall(), north=rb.Wall())


def case_c2():
    grid = rg.Grid(2048, 64, 0.05, 0.05)
    xc, _ = np.meshgrid(grid.x_centers(), grid.y_centers())
    bed = np.where(xc < 40.0, -0.32, -0.32 + (xc - 40.0) / 20.0)
    bathy = rg.build_bathymetry(grid, bed, ws=0.0)
    st = rs.solitary_wave_ic(rs.SolitaryWaveSpec(0.0576, 0.32, crest_x=33.0), bathy)
    return bathy, st, walls(), rg.PhysParams(), 0.002, dict(h_dry=1e-3), 6000


def berkhoff_bed(grid, ws=0.0):
    xc, yc = np.meshgrid(grid.x_centers(), grid.y_centers())
    xs = grid.x0 + 0.5 * grid.nx * grid.dx
    ys = grid.y0 + 0.5 * grid.ny * grid.dy
    th = math.radians(20.0)
    xr = (yc - ys) * math.cos(th) - (xc - xs) * math.sin(th)
    yr = (yc - ys) * math.sin(th) + (xc - xs) * math.cos(th)
    d = np.where(yr < -5.82, 0.45, np.maximum(0.10, 0.45 - 0.02 * (5.82 + yr)))
    inside = (xr / 4.0) ** 2 + (yr / 3.0) ** 2 < 1.0
    lift = -0.3 + 0.5 * np.sqrt(np.maximum(0.0, 1.0 - (xr / 5.0) ** 2 - (yr / 3.75) ** 2))
    d = np.where(inside, d - lift, d)
    return ws - d


def case_c3(irregular=False):
    grid = rg.Grid(1024, 1024, 0.025, 0.025)
    bathy = rg.build_bathymetry(grid, berkhoff_bed(grid), ws=0.0)
    d_west = float(bathy.depth[2:-2, 2].min())
    if irregular:
        west = rb.IrregularMaker(tuple(rb.jonswap_components(
            rb.SpectrumSpec(0.05, 1.0, 64, 2.0 / 64, 0), d_west)))
    else:
        west = rb.SineMaker((rb.sine_component(0.0232, 1.0, d_west),))
    b = rb.Boundaries(west=west, east=rb.Sponge(2.0, 10.0), south=rb.Sponge(1.0, 10.0),
                      north=rb.Sponge(1.0, 10.0))
    return bathy, rg.still_state(bathy), b, rg.PhysParams(), 0.002, {}, 400


CASES = {"c2": case_c2, "c3": case_c3, "c3j": lambda: case_c3(True)}


def run(name):
    bathy, st, b, phys, dt_init, skw, steps = CASES[name]()
    inputs = digest(np.concatenate([bathy.bed_eff.ravel(), bathy.depth.ravel(),
                                    bathy.depth_dx.ravel(), bathy.depth_dy.ravel(),
                                    bathy.bed_face_x.ravel(), bathy.bed_face_y.ravel(),
                                    st.w.ravel(), st.p.ravel(), st.q.ravel()]))
    sim = stepper.Simulator(bathy, st, b, stepper.TimeController(dt_init=dt_init), phys=phys,
                            **skw)
    t0 = time.perf_counter()
    recs = []
    for _ in range(steps):
        r = sim.advance()
        recs.append((r.step_index, r.sim_time, r.dt, r.max_cfl, r.max_speed, r.max_depth))
    wall = time.perf_counter() - t0
    s = sim.state
    out = dict(steps=steps, records=np.array(recs, dtype=np.float64), inputs_sha=inputs,
               w_sha=digest(s.w), p_sha=digest(s.p), q_sha=digest(s.q),
               clamped_volume=sim.clamped_volume, ref_seconds=wall)
    if name == "c2":  # fp32-mode check: eta (rel-L2) and the wet mask w - bed_eff > h_dry
        ii = bathy.grid.interior
        out["eta32"] = (s.w - np.maximum(bathy.ws, bathy.bed_eff))[ii].astype(np.float32)
        out["wet"] = np.packbits((s.w - bathy.bed_eff)[ii] > sim.h_dry)
    np.savez_compressed(os.path.join(OUT, f"large_{name}.npz"), **out)
    print(f"{name}: {steps} steps in {wall:.1f} s, dt[-1]={recs[-1][2]:.6g}", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(CASES):
        run(nm)
