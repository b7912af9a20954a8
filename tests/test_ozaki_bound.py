"""The error bound of the int8 digit engine (ozaki_engine.cuh) checked on an exact
emulation of its arithmetic -- CPU only, no GPU, no product code.

The engine maps x_i to N_i = rn(x_i 2^(54-E_i)) (2^(E_i-1) <= ||x_i||_inf < 2^E_i), writes N_i in 7
balanced base-256 digits, keeps the digit-pair sums acc_l of levels l = a + b <= 6 (exact integers),
forms V = sum_{l<4} 2^(8(3-l)) acc_l and W = sum_{l=4..6} 2^(8(6-l)) acc_l exactly and rounds ONCE:
s~ = fl(V + 2^-24 W) 2^(E_i+E_j-36).  The claim (plssvm.h):
    |s~ - s| <= u |s| + 13.04 d u ||x_i||_inf ||x_j||_inf        (u = 2^-53)
Here every quantity is an exact rational (fractions), so the test checks the DERIVATION: that the
constant covers the input rounding of features below 2^(E-2) and the dropped levels 7..12, including
digit patterns built to make the dropped levels as large as possible; and that the bound is not loose
by orders of magnitude on those patterns (it is a worst-case bound, attained within a factor ~2).
The GPU kernel is checked against the oracle separately (tests/test_gpu_fp64_engines.py)."""
import math
from fractions import Fraction

import numpy as np
import pytest

U = Fraction(1, 2**53)


def split(x):
    mx = max(abs(v) for v in x)
    E = math.frexp(mx)[1] if mx > 0 else 0
    sc = Fraction(2) ** (54 - E)
    N = []
    for v in x:
        t = Fraction(v) * sc
        f = math.floor(t)
        r = t - f
        n = f + (1 if (r > Fraction(1, 2) or (r == Fraction(1, 2) and f % 2 == 1)) else 0)  # round half even
        N.append(n)
    D = np.zeros((7, len(x)), dtype=np.int64)
    for k, n in enumerate(N):
        for a in range(6, -1, -1):  # least significant first, balanced digits in [-128, 127]
            dd = ((n & 0xFF) ^ 0x80) - 0x80
            n = (n - dd) >> 8
            D[a, k] = dd
        assert n == 0
    return D, E


def engine_dot(xi, xj):
    Di, Ei = split(xi)
    Dj, Ej = split(xj)
    acc = [sum(int(Di[a] @ Dj[l - a]) for a in range(7) if 0 <= l - a <= 6) for l in range(7)]
    V = (acc[0] << 24) + (acc[1] << 16) + (acc[2] << 8) + acc[3]
    W = (acc[4] << 16) + (acc[5] << 8) + acc[6]
    assert abs(V) < 2**53 and abs(W) < 2**53  # both convert to fp64 exactly
    core = float(Fraction(V) + Fraction(W, 2**24))  # the one rounding (fma)
    return Fraction(core) * Fraction(2) ** (Ei + Ej - 36)


def check_pair(xi, xj):
    s = sum(Fraction(a) * Fraction(b) for a, b in zip(xi, xj))
    st = engine_dot(xi, xj)
    d = len(xi)
    bound = U * abs(s) + Fraction(1304, 100) * d * U * Fraction(max(abs(v) for v in xi)) * \
        Fraction(max(abs(v) for v in xj))
    assert abs(st - s) <= bound, float(abs(st - s) / bound)
    return float(abs(st - s) / bound) if bound else 0.0


@pytest.mark.parametrize("kind", ["normal", "spike", "orthogonal", "wide_range", "integers"])
def test_bound_holds_on_data(kind):
    rng = np.random.default_rng(hash(kind) % 2**32)
    d = 64
    for _ in range(20):
        if kind == "normal":
            xi, xj = rng.standard_normal(d), rng.standard_normal(d)
        elif kind == "spike":
            xi, xj = rng.standard_normal(d) * 1e-3, rng.standard_normal(d) * 1e-3
            xi[3], xj[3] = 1.0, -0.75
        elif kind == "orthogonal":
            xi, xj = rng.standard_normal(d) * 1e-6, rng.standard_normal(d) * 1e-6
            xi[0], xj[1] = 1.0, 1.0
        elif kind == "wide_range":
            xi = rng.standard_normal(d) * np.ldexp(1.0, rng.integers(-60, 5, d))
            xj = rng.standard_normal(d) * np.ldexp(1.0, rng.integers(-60, 5, d))
        else:
            xi, xj = rng.integers(-1000, 1001, d).astype(float), rng.integers(-1000, 1001, d).astype(float)
        check_pair(list(xi), list(xj))


def test_integer_data_is_exact():
    rng = np.random.default_rng(5)
    xi, xj = rng.integers(-2**20, 2**20, 32).astype(float), rng.integers(-2**20, 2**20, 32).astype(float)
    assert engine_dot(list(xi), list(xj)) == sum(Fraction(a) * Fraction(b) for a, b in zip(xi, xj))


def test_bound_is_nearly_attained_by_adversarial_digits():
    """N with every low digit at -128 for x_i and a pattern that makes every dropped-level product
    positive for x_j: the dropped levels then reach most of their worst case, so the constant 13.04
    cannot be much smaller than stated (the test asserts the emulated error is >= 1/4 of the bound's
    contraction part)."""
    d = 32
    worst = 0.0
    for top in (64, 63, 40):
        # N = top 256^6 - 128 (256^5 + ... + 1): digits (top, -128, ..., -128), |N| < 2^53 -> x exact
        Nn = top * 256**6 - 128 * sum(256**k for k in range(6))
        Ni = [Nn] * d
        Nj = [Nn] * d
        E = 0
        xi = [float(Fraction(n, 2**54) * 2**E) for n in Ni]
        xj = [float(Fraction(n, 2**54) * 2**E) for n in Nj]
        assert all(Fraction(v) * 2**54 == n for v, n in zip(xi, Ni))
        s = sum(Fraction(a) * Fraction(b) for a, b in zip(xi, xj))
        st = engine_dot(xi, xj)
        part = Fraction(1304, 100) * d * U * Fraction(max(xi)) * Fraction(max(xj))
        assert abs(st - s) <= U * abs(s) + part
        worst = max(worst, float((abs(st - s) - U * abs(s)) / part))
    assert worst >= 0.25, worst
