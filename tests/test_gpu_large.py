"""BASELINE configurations at their stated sizes against the unmodified
reference (goldens from tests/golden/make_golden_large.py):

  C2  2048 x 64 plane-beach runup, h_dry = 1e-3, 6000 adaptive steps
  C3  1024 x 1024 elliptic shoal with sponges, sine maker, 400 steps
  C3J the same shoal with the irregular (JONSWAP) maker, 400 steps

Bar: bitwise -- every StepRecord and the SHA-256 of the final padded w, P, Q
(ghost frame included) equal the reference's.  fp32 mode on C2: eta rel-L2
<= 1e-4 and an identical wet mask (north_star).  The inputs are rebuilt by
scenario.make_case; a CPU test pins them to the digest of the reference's.
"""

import hashlib
import os

import numpy as np
import pytest

from paper_1909_04153_b200.scenario import make_case

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
II = (slice(2, -2), slice(2, -2))
CASES = {"c2": "C2", "c3": "C3", "c3j": "C3J"}


def load(name):
    return np.load(os.path.join(GOLDEN, f"large_{name}.npz"), allow_pickle=False)


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def inputs_digest(case):
    b, s = case.bathy, case.state
    return digest(np.concatenate([b.bed_eff.ravel(), b.depth.ravel(), b.depth_dx.ravel(),
                                  b.depth_dy.ravel(), b.bed_face_x.ravel(), b.bed_face_y.ravel(),
                                  s.w.ravel(), s.p.ravel(), s.q.ravel()]))


@pytest.mark.parametrize("name", sorted(CASES))
def test_large_inputs_match_reference(name):
    """make_case rebuilds exactly the reference's static fields and state."""
    z = load(name)
    assert inputs_digest(make_case(CASES[name])) == str(z["inputs_sha"])


def _sim(case, **kw):
    from paper_1909_04153_b200 import stepper
    return stepper.Simulator(case.bathy, case.state.copy(), case.boundaries,
                             stepper.TimeController(dt_init=case.dt_init), phys=case.phys,
                             h_dry=case.h_dry, **kw)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_large_run_bitwise(name):
    z = load(name)
    case = make_case(CASES[name])
    sim = _sim(case)
    recs = []
    for _ in range(int(z["steps"])):
        r = sim.advance()
        recs.append((r.step_index, r.sim_time, r.dt, r.max_cfl, r.max_speed, r.max_depth))
    recs = np.array(recs, dtype=np.float64)
    ref = z["records"]
    assert np.array_equal(recs[:, 2], ref[:, 2]), "adaptive dt sequence"
    assert np.array_equal(recs, ref)
    st = sim.state
    for f in ("w", "p", "q"):
        assert digest(getattr(st, f)) == str(z[f + "_sha"]), f + " (padded, bitwise)"
    assert sim.clamped_volume == pytest.approx(float(z["clamped_volume"]), rel=1e-12, abs=1e-300)
    sim.close()


@pytest.mark.gpu
def test_c2_fp32_eta_and_mask():
    """fp32 mode on the 6000-step C2 runup (wet/dry front, h_dry = 1e-3)."""
    z = load("c2")
    case = make_case("C2")
    sim = _sim(case, precision="fp32")
    for _ in range(int(z["steps"])):
        sim.advance()
    b = case.bathy
    w = sim.state.w
    eta = (w - np.maximum(b.ws, b.bed_eff))[II]
    ref = z["eta32"].astype(np.float64)
    rel = float(np.linalg.norm(eta - ref) / np.linalg.norm(ref))
    print(f"C2 fp32: eta rel-L2 {rel:.3e}")
    assert rel <= 1e-4
    wet = (w - b.bed_eff)[II] > sim.h_dry
    ref_wet = np.unpackbits(z["wet"])[:wet.size].reshape(wet.shape).astype(bool)
    assert np.array_equal(wet, ref_wet)
    sim.close()
