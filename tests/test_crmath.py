"""CPU checks of the device math headers, compiled for the host exactly as the device compiles them
(explicit roundings, no contraction):
  csrc/libm_ref.cuh  glibc's exp / log restated (K7's decisions): bit-identical to the host libm
  csrc/crmath.cuh    double-double, correctly rounded exp / log / pow: equal to 50-digit decimal
                     arithmetic, and the correctly rounded side wherever glibc is not."""
import ctypes
import os
import subprocess
from decimal import Decimal, getcontext

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "crmath_host.cpp")
LIB = os.path.join(ROOT, "tests", "native", "build", "libcrmath_host.so")


@pytest.fixture(scope="module")
def crm():
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", LIB, SRC], check=True)
    return ctypes.CDLL(LIB)


def _call(lib, fn, *arrs):
    out = np.empty_like(arrs[0])
    args = [a.ctypes.data_as(ctypes.c_void_p) for a in arrs]
    getattr(lib, fn)(*args, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(arrs[0].size))
    return out


def _exact(vals, f):
    getcontext().prec = 60
    out = []
    for v in vals:
        d = Decimal(float(v))
        out.append(float(d.exp() if f == "exp" else d.ln()))  # Decimal -> float rounds correctly
    return np.array(out)


@pytest.mark.parametrize("f,gen", [
    ("exp", lambda r: r.uniform(-30, 30, 400_000)),
    ("exp", lambda r: r.uniform(-1e-3, 1e-3, 100_000)),
    ("exp", lambda r: r.uniform(-700, 700, 100_000)),
    ("log", lambda r: np.exp(r.uniform(-700, 700, 400_000))),
    # the V initialisation's argument p / (1 - p) (calibrate.cpp:108-110), dense around 1
    ("log", lambda r: (lambda p: p / (1 - p))((np.clip(r.uniform(0, 1, 400_000), 1e-4, 1 - 1e-4) + 0.1) / 1.2)),
    ("log", lambda r: 1 + r.uniform(-1e-9, 1e-9, 100_000)),
])
def test_correctly_rounded_where_glibc_disagrees(crm, f, gen):
    rng = np.random.default_rng(hash(f) % 1000)
    x = gen(rng)
    ours = _call(crm, "crm_" + f, x)
    glibc = _call(crm, "glibc_" + f, x)
    sample = rng.choice(x.size, 200, replace=False)
    assert np.array_equal(ours[sample], _exact(x[sample], f))
    diff = np.nonzero(ours != glibc)[0]
    # glibc is within 0.52 ulp: it differs from the correctly rounded value on ~0.1% of inputs,
    # and at every such input ours is the correctly rounded one
    assert diff.size <= 2e-3 * x.size
    d = diff[:100]
    assert np.array_equal(ours[d], _exact(x[d], f))


def test_pow_and_special_values(crm):
    rng = np.random.default_rng(3)
    x = rng.uniform(1e-12, 1.0, 50_000)
    e = rng.uniform(1.0, 9.0, 50_000)  # the regulariser's pow(|2h - 1|, beta - 1), beta in [2, 10]
    ours = _call(crm, "crm_pow", x, e)
    glibc = _call(crm, "glibc_pow", x, e)
    assert np.mean(ours == glibc) > 0.998
    assert np.max(np.abs(ours - glibc) / glibc) < 2.3e-16
    sp = np.array([0.0, -0.0, 1.0, np.inf, -1.0, np.nan, 5e-324, 1.7976931348623157e308])
    assert np.array_equal(_call(crm, "crm_log", sp), _call(crm, "glibc_log", sp), equal_nan=True)
    se = np.array([0.0, -0.0, 709.78, 710.0, -708.0, -745.2, -800.0, np.inf, -np.inf, np.nan])
    assert np.array_equal(_call(crm, "crm_exp", se), _call(crm, "glibc_exp", se), equal_nan=True)


@pytest.mark.parametrize("f,gen", [
    ("exp", lambda r: r.uniform(-40, 40, 2_000_000)),
    ("exp", lambda r: r.uniform(-800, 800, 1_000_000)),  # incl. the over/underflow special case
    ("exp", lambda r: r.uniform(-760, -700, 500_000)),   # subnormal results
    ("log", lambda r: np.exp(r.uniform(-745, 709, 2_000_000))),
    ("log", lambda r: 1 + r.uniform(-0.1, 0.1, 1_000_000)),  # glibc's separate near-1 path
    ("log", lambda r: (lambda p: p / (1 - p))((np.clip(r.uniform(0, 1, 1_000_000), 1e-4, 1 - 1e-4) + 0.1) / 1.2)),
    ("log", lambda r: r.uniform(0, 2.3e-308, 200_000)),  # subnormal inputs
])
def test_libm_restatement_matches_host_glibc(crm, f, gen):
    x = gen(np.random.default_rng(11))
    ours = _call(crm, "ref_" + f, x)
    glibc = _call(crm, "glibc_" + f, x)
    same = (ours == glibc) | (np.isnan(ours) & np.isnan(glibc))
    assert same.all(), (x[~same][:5], ours[~same][:5], glibc[~same][:5])


def test_libm_restatement_special_values(crm):
    sp = np.array([0.0, -0.0, 1.0, np.inf, -np.inf, -1.0, np.nan, 5e-324, 2.2250738585072014e-308,
                   1.7976931348623157e308, 709.782712893384, 709.79, -745.1332191019411, -745.14, 1e-300])
    for f in ("exp", "log"):
        a, b = _call(crm, "ref_" + f, sp), _call(crm, "glibc_" + f, sp)
        assert np.array_equal(a, b, equal_nan=True), f


@pytest.mark.parametrize("gen", [
    # the regulariser's pow(max(|2h - 1|, 1e-12), beta - 1), beta annealed 20 -> 2 (calibrate.cpp:358)
    lambda r: (np.maximum(np.abs(r.uniform(-1, 1, 2_000_000)), 1e-12), r.uniform(1.0, 19.0, 2_000_000)),
    lambda r: (np.exp(r.uniform(-700, 700, 1_000_000)), r.uniform(-3, 3, 1_000_000)),
    lambda r: (r.uniform(0.5, 2.0, 1_000_000), r.uniform(-1000, 1000, 1_000_000)),  # over / underflow
    lambda r: (np.exp(r.uniform(-2, 2, 500_000)), r.uniform(300, 700, 500_000)),    # the exp specialcase
    lambda r: (-r.integers(1, 50, 500_000).astype(np.float64) * r.uniform(0.9, 1.1, 500_000),
               r.integers(-60, 60, 500_000).astype(np.float64)),                   # x < 0, integer y
    lambda r: (r.uniform(0, 2.3e-308, 300_000), r.uniform(-0.5, 0.5, 300_000)),     # subnormal x
])
def test_libm_pow_matches_host_glibc(crm, gen):
    x, e = gen(np.random.default_rng(17))
    ours = _call(crm, "ref_pow", x, e)
    glibc = _call(crm, "glibc_pow", x, e)
    same = (ours == glibc) | (np.isnan(ours) & np.isnan(glibc))
    assert same.all(), (x[~same][:5], e[~same][:5], ours[~same][:5], glibc[~same][:5])


def test_libm_pow_special_values(crm):
    v = np.array([0.0, -0.0, 1.0, -1.0, 2.0, -2.0, 0.5, np.inf, -np.inf, np.nan, 5e-324, 3.0, -3.0,
                  1e-300, 1e300, 1 + 2 ** -52, 1e-20, 2.0 ** -70, 2.0 ** 70], dtype=np.float64)
    x, e = np.meshgrid(v, v)
    x, e = x.ravel().copy(), e.ravel().copy()
    a, b = _call(crm, "ref_pow", x, e), _call(crm, "glibc_pow", x, e)
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    assert same.all(), (x[~same], e[~same], a[~same], b[~same])
