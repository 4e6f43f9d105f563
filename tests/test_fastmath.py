"""Accuracy of csrc/fastmath.cuh (the FP64 sincospi / log / exp / sqrt / divide
the fast particle kernels use) through a host build of the same header,
against mpmath at 40 digits.  The device build differs only in the rcp/rsqrt
seeds (MUFU vs float), which the Newton steps wash out; the GPU tests compare
the device Box-Muller pairs with the oracle's libm ones (test_gpu_parity.py).
"""
import ctypes as C
import subprocess
from pathlib import Path

import mpmath
import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def fm(tmp_path_factory):
    out = tmp_path_factory.mktemp("fm") / "libfm.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", "-o", str(out),
                    str(ROOT / "tests/cpp/fastmath_host.cpp")], check=True)
    lib = C.CDLL(str(out))
    P = C.POINTER(C.c_double)
    for name, n in [("fm_sincospi", 4), ("fm_sincospi_shift", 4), ("fm_log", 3), ("fm_log_tab", 3), ("fm_exp", 3), ("fm_exp_bump", 3), ("fm_sqrt", 3),
                    ("fm_div", 4)]:
        getattr(lib, name).restype = None
    return lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def ulp_err(got, exact):
    got = np.asarray(got, dtype=np.float64)
    ex = np.array([float(e) for e in exact])
    ulp = np.spacing(np.abs(ex))
    d = np.array([float(abs(mpmath.mpf(g) - e)) for g, e in zip(got, exact)])
    return np.max(d / ulp)


mpmath.mp.dps = 40
RNG = np.random.default_rng(7)


def test_sincospi(fm):
    a = np.concatenate([RNG.uniform(-4, 4, 3000), RNG.uniform(0, 2, 1000), np.arange(-8, 9) * 0.25])
    s = np.empty_like(a)
    c = np.empty_like(a)
    fm.fm_sincospi(_p(a), C.c_int64(a.size), _p(s), _p(c))
    es = [mpmath.sinpi(mpmath.mpf(x)) for x in a]
    ec = [mpmath.cospi(mpmath.mpf(x)) for x in a]
    # absolute error in units of 2^-53 (values near zero have tiny ulps)
    ds = max(float(abs(mpmath.mpf(g) - e)) for g, e in zip(s, es)) / 2**-53
    dc = max(float(abs(mpmath.mpf(g) - e)) for g, e in zip(c, ec)) / 2**-53
    assert ds <= 2.0 and dc <= 2.0
    big = np.abs(np.array([float(e) for e in es])) > 0.25
    assert ulp_err(s[big], [e for e, b in zip(es, big) if b]) <= 2.0
    # exact quarter turns
    q = np.arange(-8, 9) * 0.5
    s = np.empty_like(q)
    c = np.empty_like(q)
    fm.fm_sincospi(_p(q), C.c_int64(q.size), _p(s), _p(c))
    assert np.all(np.abs(s) == np.abs(np.round(np.sin(np.pi * q))))
    assert np.all(np.abs(c) == np.abs(np.round(np.cos(np.pi * q))))


def test_log_on_uniforms(fm):
    # the kernels feed it ((r >> 11) + 0.5) 2^-53: (0, 1), down to 2^-54
    x = np.concatenate([RNG.uniform(0, 1, 3000), 2.0 ** -RNG.uniform(1, 54, 1000),
                        [2.0 ** -54, 0.5, 1 - 2.0 ** -53, np.sqrt(0.5), 0.7071067811865476]])
    y = np.empty_like(x)
    fm.fm_log(_p(x), C.c_int64(x.size), _p(y))
    assert ulp_err(y, [mpmath.log(mpmath.mpf(v)) for v in x]) <= 2.0


def test_table_log_on_uniforms(fm):
    """fm::log_tab, the particle kernels' Box-Muller log: <= 1.5 ulp (1.37
    measured over 2e5 uniforms; two roundings in hi + (lo + p)), including
    x -> 1 from below (relative accuracy kept by the c = 1 bins) and tiny x."""
    x = np.concatenate([RNG.uniform(0, 1, 4000), 2.0 ** -RNG.uniform(1, 54, 1000),
                        1 - 2.0 ** -RNG.uniform(8, 53, 500), 1 - RNG.uniform(0, 1e-3, 500),
                        [2.0 ** -54, 0.5, 1 - 2.0 ** -53, np.sqrt(0.5), 0.7071067811865476, 1.4140625 / 2,
                         (1 + 53 / 128) / 2 - 2.0 ** -53, 0.99609375, 0.9921875]])
    y = np.empty_like(x)
    fm.fm_log_tab(_p(x), C.c_int64(x.size), _p(y))
    assert ulp_err(y, [mpmath.log(mpmath.mpf(v)) for v in x]) <= 1.5
    for g in (1.0, 2.0, 3.5, 1e10, 1e-300):  # general normal x
        v = np.array([g])
        w = np.empty_like(v)
        fm.fm_log_tab(_p(v), C.c_int64(1), _p(w))
        assert ulp_err(w, [mpmath.log(mpmath.mpf(g))]) <= 1.0


def test_exp(fm):
    x = np.concatenate([RNG.uniform(-700, 0, 2000), RNG.uniform(-5, 5, 2000), [0.0, -1e-300]])
    y = np.empty_like(x)
    fm.fm_exp(_p(x), C.c_int64(x.size), _p(y))
    assert ulp_err(y, [mpmath.exp(mpmath.mpf(v)) for v in x]) <= 2.0
    z = np.array([-800.0, -745.5])
    w = np.empty_like(z)
    fm.fm_exp(_p(z), C.c_int64(2), _p(w))
    assert w[0] == 0.0 and w[1] == 0.0
    z = np.array([710.0, 1e14, -1e300, -708.0, 709.0])
    w = np.empty_like(z)
    fm.fm_exp(_p(z), C.c_int64(z.size), _p(w))
    assert np.isinf(w[0]) and np.isinf(w[1]) and w[2] == 0.0
    assert ulp_err(w[3:], [mpmath.exp(mpmath.mpf(v)) for v in z[3:]]) <= 2.0


def test_sincospi_shift_quadrant_identical(fm):
    """sincospi<true> (quadrant from the 1.5 2^52 shifter, the walkers) equals
    sincospi<false> (rint) bit for bit, ties and quarter turns included."""
    a = np.concatenate([RNG.uniform(-4, 4, 4000), RNG.uniform(0, 2, 2000), np.arange(-16, 17) * 0.125,
                        np.arange(-8, 9) * 0.25 + 2.0 ** -40, [1e6 + 0.25, -3e9 + 0.75, 0.0, -0.0]])
    s0, c0, s1, c1 = (np.empty_like(a) for _ in range(4))
    fm.fm_sincospi(_p(a), C.c_int64(a.size), _p(s0), _p(c0))
    fm.fm_sincospi_shift(_p(a), C.c_int64(a.size), _p(s1), _p(c1))
    assert np.array_equal(s0.view(np.uint64), s1.view(np.uint64))
    assert np.array_equal(c0.view(np.uint64), c1.view(np.uint64))


def test_exp_bump(fm):
    """fm::exp_bump, the walkers' table exponential, on its whole domain [-708, 0]
    (the launcher proves the bump exponents lie in [-700, 0])."""
    x = np.concatenate([RNG.uniform(-708, 0, 3000), RNG.uniform(-1, 0, 1000), -RNG.uniform(0, 1e-3, 500),
                        [0.0, -0.0, -1e-300, -708.0, -700.0, -np.log(2) / 512, -np.log(2) / 256]])
    y = np.empty_like(x)
    fm.fm_exp_bump(_p(x), C.c_int64(x.size), _p(y))
    assert ulp_err(y, [mpmath.exp(mpmath.mpf(v)) for v in x]) <= 1.5
    assert y[-7] == 1.0 and y[-6] == 1.0 and y[-5] == 1.0


def test_sqrt_and_div_correctly_rounded(fm):
    v = np.concatenate([-2 * np.log(RNG.uniform(0, 1, 4000)), [2.0 ** -53, 75.0, 1.0, 4.0]])
    y = np.empty_like(v)
    fm.fm_sqrt(_p(v), C.c_int64(v.size), _p(y))
    assert np.array_equal(y, np.sqrt(v))
    f = RNG.uniform(np.sqrt(0.5) - 1, np.sqrt(2) - 1, 4000)
    d = 2.0 + f
    q = np.empty_like(f)
    fm.fm_div(_p(f), _p(d), C.c_int64(f.size), _p(q))
    assert np.array_equal(q, f / d)
