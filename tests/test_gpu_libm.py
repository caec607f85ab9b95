"""The device restatement of glibc 2.39's exp / log / log1p / acosh / acos / pow / sincos
(csrc/glibc_libm.cuh) against the HOST glibc the reference links (oracle.orc_libm_eval):
bitwise equality, no tolerance.

Inputs are seeded draws from the argument ranges the reference's sampler produces
(rng.hpp:221 pow(U, 1/k); partition.hpp:66 acosh(c), c in [1, cosh(alpha R)];
sweep.hpp:125 exp(r), r in [1e-12, R]; sweep.hpp:66 acos(arg), arg in (-1, 1);
sweep.hpp:138-139 sincos(theta), theta in [0, 2 pi)) plus wide ranges and raw bit
patterns.  RHG_LIBM_SAMPLES (default 2^22) sets the draws per domain;
tools/libm/check_device.py runs the same check at 10^8 per function
(profiles/r02/libm_device_check.log).
"""
import os

import numpy as np
import pytest

import paper_1710_07565_b200 as rhg

pytestmark = pytest.mark.gpu

N = int(float(os.environ.get("RHG_LIBM_SAMPLES", 1 << 22)))
TWO_PI = 6.283185307179586


def _u01(g, n):
    return (g.integers(0, 2**63, n, dtype=np.uint64) >> np.uint64(10)).astype(np.float64) * 2.0 ** -53


def _logu(g, lo, hi, n):
    return np.exp2(np.log2(lo) + _u01(g, n) * (np.log2(hi) - np.log2(lo)))


def _bits(g, n):
    return g.integers(0, 2**64, n, dtype=np.uint64).view(np.float64)


def _signed(g, v):
    return np.where(g.integers(0, 2, v.size) == 1, -v, v)


# name -> (function, generator(g, n) -> (x, y))
DOMAINS = {
    "exp_r": ("exp", lambda g, n: (1e-12 + _u01(g, n) * 45, None)),
    "exp_logu": ("exp", lambda g, n: (_logu(g, 1e-13, 50, n), None)),
    "exp_wide": ("exp", lambda g, n: ((_u01(g, n) - 0.5) * 1500, None)),
    "exp_bits": ("exp", lambda g, n: (_bits(g, n), None)),
    "log_wide": ("log", lambda g, n: (_logu(g, 1e-300, 1e300, n), None)),
    "log_near1": ("log", lambda g, n: (0.9 + 0.2 * _u01(g, n), None)),
    "log_bits": ("log", lambda g, n: (_bits(g, n), None)),
    "log1p_03": ("log1p", lambda g, n: (3 * _u01(g, n), None)),
    "log1p_logu": ("log1p", lambda g, n: (_logu(g, 1e-20, 1e20, n), None)),
    "log1p_neg": ("log1p", lambda g, n: (-_u01(g, n), None)),
    "acosh_12": ("acosh", lambda g, n: (1 + _u01(g, n), None)),
    "acosh_tiny": ("acosh", lambda g, n: (1 + _logu(g, 1e-16, 1, n), None)),
    "acosh_big": ("acosh", lambda g, n: (_logu(g, 2, 1e19, n), None)),
    "acosh_wide": ("acosh", lambda g, n: (_logu(g, 1, 1e300, n), None)),
    "acos_unit": ("acos", lambda g, n: (2 * _u01(g, n) - 1, None)),
    "acos_near1": ("acos", lambda g, n: (_signed(g, 1 - _logu(g, 1e-17, 0.05, n)), None)),
    "acos_small": ("acos", lambda g, n: (_signed(g, _logu(g, 1e-20, 0.2, n)), None)),
    "acos_bits": ("acos", lambda g, n: (_bits(g, n), None)),
    "pow_sampler": ("pow", lambda g, n: (_u01(g, n), 1.0 / np.floor(_logu(g, 1, 2.0 ** 32, n)))),
    "pow_smallk": ("pow", lambda g, n: (_u01(g, n), 1.0 / (1 + g.integers(0, 4096, n)).astype(np.float64))),
    "pow_near1": ("pow", lambda g, n: (1 - _logu(g, 2.0 ** -53, 1e-3, n),
                                       1.0 / np.floor(_logu(g, 1, 2.0 ** 30, n)))),
    "pow_wide": ("pow", lambda g, n: (_logu(g, 1e-300, 1e300, n), (_u01(g, n) - 0.5) * 40)),
    "pow_bits": ("pow", lambda g, n: (_bits(g, n), _bits(g, n))),
    "sin_theta": ("sin", lambda g, n: (_u01(g, n) * TWO_PI, None)),
    "cos_theta": ("cos", lambda g, n: (_u01(g, n) * TWO_PI, None)),
    "sin_small": ("sin", lambda g, n: (_signed(g, _logu(g, 1e-20, 1, n)), None)),
    "cos_small": ("cos", lambda g, n: (_signed(g, _logu(g, 1e-20, 1, n)), None)),
    "sin_wide": ("sin", lambda g, n: ((_u01(g, n) - 0.5) * 2e8, None)),
    "cos_wide": ("cos", lambda g, n: ((_u01(g, n) - 0.5) * 2e8, None)),
}


def mismatches(fn, x, y, oracle):
    want = oracle.libm_eval(rhg.LIBM_FUNCTIONS.index(fn), x, y)
    got = rhg.libm_eval(fn, x, y)
    same = (want.view(np.uint64) == got.view(np.uint64)) | (np.isnan(want) & np.isnan(got))
    return np.flatnonzero(~same), want, got


@pytest.mark.parametrize("domain", sorted(DOMAINS))
def test_device_libm_bit_exact(oracle, domain):
    fn, gen = DOMAINS[domain]
    g = np.random.default_rng(sorted(DOMAINS).index(domain) + 1)
    x, y = gen(g, N)
    bad, want, got = mismatches(fn, x, y, oracle)
    assert bad.size == 0, [(x[i].hex(), None if y is None else y[i].hex(), want[i].hex(), got[i].hex())
                           for i in bad[:5]]


def test_libm_edge_values(oracle):
    specials = np.array([0.0, -0.0, 1.0, -1.0, 2.0, 0.5, np.inf, -np.inf, np.nan, 1e-320, -1e-320,
                         np.nextafter(1.0, 0), np.nextafter(1.0, 2), 2.0 ** -1022, 709.78, -745.1, 2.0 ** 28,
                         2.0 ** 28 + 2, 0.96875, -0.96875, 0.125, 0.855468, 2.426265, 1.05e8])
    x = np.repeat(specials, specials.size)
    y = np.tile(specials, specials.size)
    for fn in rhg.LIBM_FUNCTIONS:
        if fn in ("sin", "cos"):
            xs = x[np.abs(x) <= 1.05e8]  # |x| >= 105414350 (__branred) is outside the path
            ys = None
        else:
            xs, ys = x, (y if fn == "pow" else None)
        bad, want, got = mismatches(fn, xs, ys, oracle)
        assert bad.size == 0, (fn, [(xs[i], want[i], got[i]) for i in bad[:5]])
