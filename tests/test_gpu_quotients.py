"""The step's quotient helpers (bsq_device.cuh) against IEEE x / d, bit for
bit, on the device, through the bsq_check_quotients seam.

Every division of the reference (numba, IEEE binary64) is computed on the
B200 as a Markstein quotient from a correctly rounded reciprocal, so parity
rests on these helpers returning exactly x / d over the inputs each call site
can see: normal and subnormal numerators (sponge damping drives momenta
towards zero geometrically), signed zeros, and -- where the non-finite scans
must see the reference's cells -- infinities and NaN.
"""

import ctypes

import numpy as np
import pytest

from paper_1909_04153_b200 import _native as nat

pytestmark = pytest.mark.gpu

OPS = {"div_static": 0, "div_pos": 1, "div_rcp": 2, "div_rcp_pos": 3, "div_nonneg": 4,
       "div_static_pos": 5}


def run(op, x, d):
    x = np.ascontiguousarray(x, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    out = np.empty_like(x)
    rc = nat.lib().bsq_check_quotients(op, nat.ptr(x), nat.ptr(d), ctypes.c_long(x.size),
                                       nat.ptr(out))
    assert rc == 0, nat.lib().bsq_last_error()
    return out


def same(a, b):
    """Bitwise equal, NaN matching any NaN."""
    ab, bb = a.view(np.uint64), b.view(np.uint64)
    return (ab == bb) | (np.isnan(a) & np.isnan(b))


def numerators(rng, n):
    mant = rng.integers(1, 2 ** 52, n, dtype=np.uint64)
    sub = mant.view(np.float64) * rng.choice([-1.0, 1.0], n)  # subnormals
    norm = rng.standard_normal(n) * 10.0 ** rng.uniform(-300, 300, n)
    tiny = rng.standard_normal(n) * 10.0 ** rng.uniform(-307, -300, n)  # near the subnormal range
    return {"normal": norm, "tiny_normal": tiny, "subnormal": sub}


# divisor range each call site guarantees
DIVISORS = {
    "div_static": lambda rng, n: 10.0 ** rng.uniform(-4, 4, n),   # 2dx, dx^2, 3, 6
    "div_pos": lambda rng, n: 10.0 ** rng.uniform(-4, 4, n),
    "div_rcp": lambda rng, n: 10.0 ** rng.uniform(-12, 4, n),     # friction h*^2
    "div_rcp_pos": lambda rng, n: 10.0 ** rng.uniform(-6, 2, n),  # depths >= h_eps
    "div_nonneg": lambda rng, n: 10.0 ** rng.uniform(-6, 2, n),
    "div_static_pos": lambda rng, n: 10.0 ** rng.uniform(-3, 3, n),  # Thomas pivots
}


TINY_NUM = 2.0 ** -960  # bsq_device.cuh: the helpers' exact range starts here


@pytest.mark.parametrize("name", sorted(OPS))
def test_quotient_helper_bitwise(name):
    """Exact for every numerator of magnitude >= 2^-960 (and zeros); under it
    the Markstein residual can underflow and an ulp is lost -- the kernels
    detect such numerators and divide exactly there (test_gpu_tiny.py).  The
    miss rate below the bound is measured, so the bound is not vacuous."""
    rng = np.random.default_rng(OPS[name] + 100)
    n = 1 << 20
    d = DIVISORS[name](rng, n)
    for cls, x in numerators(rng, n).items():
        got = run(OPS[name], x, d)
        want = x / d
        bad = ~same(got, want)
        big = np.abs(x) >= TINY_NUM
        assert not (bad & big).any(), (
            f"{name}, {cls} numerators: {int((bad & big).sum())} of {n} differ, e.g. "
            f"{x[bad & big][:3]} / {d[bad & big][:3]} -> {got[bad & big][:3]} vs "
            f"{want[bad & big][:3]}")
        if cls == "subnormal":
            print(f"{name}: {int(bad.sum())} of {n} subnormal numerators miss IEEE by an ulp")
            assert bad.any()  # the class the kernels' detection exists for


@pytest.mark.parametrize("lo,hi", [(-2000, -960), (-1074, -1020), (-330, -289)])
def test_div_tiny_exact_bitwise(lo, hi):
    """div_tiny_exact (op 7): the kernels' call-free division for numerators
    under 2^-960 is IEEE's x / d bit for bit -- subnormal results, the ties
    its second rounding can create, both signs -- over divisors 2^-400..2^400."""
    rng = np.random.default_rng(-lo)
    n = 1 << 21
    x = rng.uniform(1.0, 2.0, n) * 2.0 ** rng.integers(lo, hi, n).astype(np.float64)
    x = np.where(x < 2.0 ** -1074, 5e-324 * rng.integers(1, 4, n), x) * rng.choice([-1.0, 1.0], n)
    x = np.where(np.abs(x) < 2.0 ** -960, x, 2.0 ** -961)
    d = rng.uniform(1.0, 2.0, n) * 2.0 ** rng.integers(-20, 21, n) * rng.choice([-1.0, 1.0], n)
    d[: n // 8] = rng.choice([3.0, 6.0, 0.5, 1.5, 2.0 ** -30, 2.0 ** 30], n // 8)
    got = run(7, x, d)
    want = x / d
    bad = ~same(got, want)
    assert not bad.any(), (x[bad][:3], d[bad][:3], got[bad][:3], want[bad][:3])


@pytest.mark.parametrize("name", ["div_static", "div_pos", "div_rcp", "div_rcp_pos",
                                  "div_nonneg", "div_static_pos"])
def test_quotient_helper_special_values(name):
    """Signed zeros give IEEE's signed zero; non-finite numerators give a
    non-finite quotient (inf / d is NaN in the select-free residual forms, as
    in the library's; the stage's non-finite scan only asks "finite?")."""
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 1.7976931348623157e308])
    d = np.array([0.5, 3.0, 6.0, 1e-6, 7.25, 2.0, 1e3])
    x = np.repeat(sp, d.size)
    dd = np.tile(d, sp.size)
    got = run(OPS[name], x, dd)
    want = x / dd
    fin = np.isfinite(want)
    assert same(got[fin], want[fin]).all()
    assert not np.isfinite(got[~fin]).any()
