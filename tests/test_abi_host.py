"""CPU-side checks: the C-ABI library loads and exports every symbol
include/bsq.h declares (no compute without a GPU), and the host data model
and per-step host scalars are bitwise the reference's (golden fixtures)."""

import ctypes
import os
import re

import numpy as np
import pytest

import golden_cases as gc
from paper_1909_04153_b200 import _native as nat
from paper_1909_04153_b200 import boundary as bc
from paper_1909_04153_b200 import multistep
from paper_1909_04153_b200.grid import Grid, build_bathymetry, still_state
from paper_1909_04153_b200.scenario import SolitaryWaveSpec, rip_channel_bathymetry, solitary_wave_ic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "bsq.h")).read()
    return sorted(set(re.findall(r"\b(bsq_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(nat.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    # the ctypes binding declares exactly the header's entry points
    assert sorted(n for n, _, _ in nat.SIGNATURES) == syms


def test_struct_layouts_match_header_sizes():
    # sizes computed from the C declarations (x86-64 natural alignment)
    assert ctypes.sizeof(nat.Desc) == 72 + 12 * 8 + 24  # 17 int32 + pad, 12 doubles, 6 int32
    assert ctypes.sizeof(nat.Static) == 7 * 8
    assert ctypes.sizeof(nat.StepResult) == 5 * 8 + 8 * 8
    assert ctypes.sizeof(nat.StepParams) == 16 + 8 + 48 + 128 + 32 + 8 + 8 + 8 * 8


def test_workspace_query_needs_no_gpu():
    d = nat.Desc()
    d.nx, d.ny, d.dx, d.dy = 64, 48, 0.1, 0.1
    n = nat.lib().bsq_workspace_bytes(ctypes.byref(d))
    assert n > 48 * 52 * 64 * 8
    d.nx = 3
    assert nat.lib().bsq_workspace_bytes(ctypes.byref(d)) == 0


@pytest.mark.parametrize("name", ["c1", "runup", "rip_irregular", "dry_clamp", "lake"])
def test_build_bathymetry_bitwise(name):
    z = gc.load(name)
    grid = Grid(int(z["nx"]), int(z["ny"]), float(z["dx"]), float(z["dy"]), float(z["x0"]),
                float(z["y0"]))
    b = build_bathymetry(grid, z["bed"], ws=float(z["ws"]))
    for f in ("bed_eff", "depth", "depth_dx", "depth_dy", "bed_face_x", "bed_face_y"):
        assert np.array_equal(getattr(b, f), z[f]), f
    assert b.h_eps == float(z["h_eps"])


def test_rip_bathymetry_and_jonswap_bitwise():
    z = gc.load("rip_irregular")
    grid = Grid(64, 48, 20.48 / 64, 30.0 / 48, x0=0.0, y0=-15.0)
    b = rip_channel_bathymetry(grid)
    assert np.array_equal(b.bed_eff, z["bed_eff"])
    d_west = float(b.depth[2:-2, 2].min())
    comps = bc.jonswap_components(bc.SpectrumSpec(0.13, 1.6, 68, 0.01, 7), d_west)
    got = np.array([(3, c.amplitude, c.omega, c.k, c.phase) for c in comps])
    assert np.array_equal(got, z["maker_comps"])


def test_solitary_ic_bitwise():
    z = gc.load("c1")
    grid = Grid(1024, 5, 0.05, 0.05)
    b = build_bathymetry(grid, np.full((5, 1024), -0.32), ws=0.0)
    st = solitary_wave_ic(SolitaryWaveSpec(0.0576, 0.32, crest_x=15.0), b)
    assert np.array_equal(st.w, z["w0"]) and np.array_equal(st.p, z["p0"])


def test_weights_bitwise():
    rows = np.load(gc.GOLDEN + "/weights.npz")["rows"]
    for r in rows:
        st = multistep.StepTriple(*r[:3])
        assert multistep.ab3_weights(st, ratio_policy="clamp").as_tuple() == tuple(r[3:6])
        assert tuple(multistep.increment_weights(st, ratio_policy="clamp")) == tuple(r[6:9])


def test_frozen_weights():
    w = multistep.ab3_weights(multistep.StepTriple(1.0, 2.0, 2.0))
    assert (w.w_cur, w.w_prev, w.w_prev2) == pytest.approx((17 / 12, -7 / 12, 1 / 6), rel=1e-15)
    v = multistep.vfd_weights("newest", 1.0, 2.0)
    assert v.as_tuple() == pytest.approx((4 / 3, -3 / 2, 1 / 6), rel=1e-15)
    assert multistep.increment_weights(multistep.StepTriple(0.1, 0.1, 0.1)) == (2.0, -3.0, 1.0)


def test_sponge_factors_match_reference_expression():
    grid = Grid(40, 32, 0.25, 0.25)
    lo, s = bc.sponge_band(grid, "east", 2.0, 8.0)
    assert lo == 32 and s.size == 8
    fac = bc.sponge_factors(s, 2.0, 8.0, 0.01)
    sref = ((np.arange(40) + 0.5) * 0.25)[::-1]
    inb = sref < 2.0
    assert np.array_equal(fac, np.exp(-(8.0 * ((2.0 - sref[inb]) / 2.0) ** 2) * 0.01))
    assert bc.sponge_band(grid, "west", 2.0, 0.0) is None


def test_maker_values_sum_in_order():
    comps = [bc.WaveComponent(0.01, 2.0, 1.1, 0.2), bc.WaveComponent(0.02, 3.0, 2.1, 1.0)]
    eta, flux = bc.maker_surface_flux(comps, 0.7)
    s0 = 0.01 * np.sin(2.0 * 0.7 + 0.2)
    s1 = 0.02 * np.sin(3.0 * 0.7 + 1.0)
    assert eta == pytest.approx(s0 + s1, rel=1e-15)
    assert flux == pytest.approx(s0 * (2.0 / 1.1) + s1 * (3.0 / 2.1), rel=1e-15)


def test_native_maker_sums_bitwise():
    """bsq_maker_sums (host C, libm sin) == boundary.maker_surface_flux, the
    reference's math.sin loop, on the C4 JONSWAP spectrum (68 components)."""
    from paper_1909_04153_b200.scenario import make_case
    comps = make_case("C4", scale=16).boundaries.west.components
    rows = np.ascontiguousarray([(c.amplitude, c.omega, c.k, c.phase) for c in comps])
    out = np.zeros(2)
    for t in np.concatenate([np.random.default_rng(5).uniform(0, 200, 3000),
                             np.arange(0.0, 3.0, 0.00137)]):
        assert nat.lib().bsq_maker_sums(nat.ptr(rows), len(comps), float(t), nat.ptr(out)) == 0
        assert (out[0], out[1]) == bc.maker_surface_flux(comps, float(t))


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1909_04153_b200 import stepper
    grid = Grid(8, 6, 1.0, 1.0)
    b = build_bathymetry(grid, np.full((6, 8), -1.0), ws=0.0)
    walls = bc.Boundaries(west=bc.Wall(), east=bc.Wall(), south=bc.Wall(), north=bc.Wall())
    with pytest.raises(RuntimeError, match="CUDA"):
        stepper.Simulator(b, still_state(b), walls, stepper.TimeController(dt_init=0.01))
