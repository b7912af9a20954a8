"""GPU parity of the two fp64 contraction engines (include/plssvm.h plssvm_fp64_engine_t):
OZAKI (int8 tensor cores on an exact 7-digit split of every point, 2-SM UMMA) and DMMA (fp64
tensor cores), plus the AUTO rule, against the CPU oracle.  Bars as in test_gpu_parity.py:
product <= 1e-12 norm-wise and |y_i - y*_i| <= 1e-12 (|Q~||p|)_i element-wise; alpha, b <= 1e-7.

The Ozaki error bound is d 2^-56 ||x_i||_inf ||x_j||_inf per inner product, so the cases below
stress what the row-max scaling could get wrong: ragged shapes around the 32-feature slab and
the 128/256-point (pair-)tile edges, magnitudes far from 1, exact-integer data, zero rows,
duplicated points, odd band / pair ends on several ranks (test_gpu_multirank.py), and the AUTO
switch to DMMA for peaked rows."""
import numpy as np
import pytest

import oracle
import paper_2202_12674_b200 as pl

pytestmark = pytest.mark.gpu

KERNELS = [pl.LINEAR, pl.POLYNOMIAL, pl.RBF]
ENGINES = [pl.FP64_OZAKI, pl.FP64_DMMA]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def check(X, p, kernel, gamma, C=1.0, degree=3, coef0=0.5, engine=pl.FP64_OZAKI, mode=pl.MODE_IMPLICIT, tol=1e-12):
    Qt = oracle.qtilde(X, kernel, gamma, degree, coef0, C)
    ref = oracle.matvec(Qt, p)
    scale = np.abs(Qt) @ np.abs(p)
    out, _ = pl.plssvm_qtilde_matvec(X, p, kernel, gamma, degree, coef0, C,
                                     opts=pl.options(mode=mode, fp64_engine=engine))
    assert rel(out, ref) <= tol, rel(out, ref)
    assert np.all(np.abs(out - ref) <= tol * scale + 1e-300), np.max(np.abs(out - ref) / scale)
    return out


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("m,d", [(2, 1), (130, 31), (255, 32), (257, 33), (384, 64), (513, 65), (1031, 100)])
def test_engines_match_oracle(m, d, kernel, engine):
    rng = np.random.default_rng(31 * m + d + 7 * kernel)
    X = rng.standard_normal((m, d))
    p = rng.standard_normal(m - 1)
    for mode in (pl.MODE_IMPLICIT, pl.MODE_CACHED):
        check(X, p, kernel, 1.0 / d, engine=engine, mode=mode)


@pytest.mark.parametrize("kernel", KERNELS)
def test_ozaki_scale_exactness(kernel):
    """Rows scaled by powers of two far from 1 (2^-300 .. 2^300 would overflow the kernels, so
    +-2^40) and a non-power-of-two global scale: the split is exact, the result scales."""
    rng = np.random.default_rng(3 + kernel)
    m, d = 700, 50
    X = rng.standard_normal((m, d)) * 3.7e-3
    p = rng.standard_normal(m - 1)
    check(X, p, kernel, 1.0 / d * 1e4 if kernel != pl.LINEAR else 1.0)
    if kernel == pl.LINEAR:  # per-row powers of two (x_m unscaled): each inner product keeps its
        e = rng.integers(-40, 41, m)  # relative accuracy under the row-max scaling
        e[-1] = 0
        Xs = X * np.ldexp(1.0, e)[:, None]
        check(Xs, p, kernel, 1.0, C=1e30)


def test_ozaki_integer_data_is_exact():
    """Small integers: every digit product is an exact integer and so is every Q~ entry (linear,
    C = 1): the product equals the oracle's bit for bit after rounding both to integers."""
    rng = np.random.default_rng(9)
    m, d = 600, 40
    X = rng.integers(-50, 51, (m, d)).astype(np.float64)
    p = rng.integers(-3, 4, m - 1).astype(np.float64)
    out = check(X, p, pl.LINEAR, 1.0, C=1.0, engine=pl.FP64_OZAKI)
    ref = oracle.matvec(oracle.qtilde(X, pl.LINEAR, 1.0, 3, 0.0, 1.0), p)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("engine", ENGINES)
def test_zero_rows_and_duplicates(engine):
    rng = np.random.default_rng(12)
    m, d = 520, 48
    X = rng.standard_normal((m, d))
    X[5] = 0.0
    X[300] = 0.0
    X[7] = X[400]
    X[m - 1] = X[0]  # x_m duplicates x_0
    p = rng.standard_normal(m - 1)
    for kernel in KERNELS:
        check(X, p, kernel, 1.0 / d, engine=engine)


def test_auto_picks_dmma_for_peaked_rows_and_stays_exact():
    rng = np.random.default_rng(4)
    m, d = 400, 64
    y = np.where(rng.random(m) < 0.5, 1.0, -1.0)
    y[0], y[1] = 1.0, -1.0
    X = rng.standard_normal((m, d))
    _, _, st, stats = pl.plssvm_train_ex(X, y, pl.RBF, 1.0 / d, eps=1e-10)
    assert st == 0 and stats.fp64_engine_used == pl.FP64_OZAKI
    Xp = X.copy()
    Xp[17, 3] = 1e4  # one feature 1e4 x the row's scale: row peak ~ 1e4 / sqrt(1e8 / 64) = 8
    Xp[18, :] = 1e-3
    Xp[18, 9] = 10.0  # peak 10 / sqrt(100 / 64) = 8: still OZAKI
    _, _, st, stats = pl.plssvm_train_ex(Xp, y, pl.RBF, 1.0 / d, eps=1e-10)
    assert stats.fp64_engine_used == pl.FP64_OZAKI
    Xq = X.copy()
    Xq[21, :] = 1e-6
    Xq[21, 0] = 1.0  # one spike among tiny features: peak = sqrt(64) = 8 -> OZAKI
    Xq[22, :] = 1e-9
    Xq[22, 1:3] = 1.0  # two spikes: peak sqrt(64 / 2) = 5.7
    Xr = np.zeros((m, d))
    Xr[:] = rng.standard_normal((m, d)) * 1e-6
    Xr[:, 0] = rng.standard_normal(m) * 1e3  # every row peaks ~ 8 (one dominant feature of 64)
    for Xc in (Xq, Xr):
        _, _, st, stats = pl.plssvm_train_ex(Xc, y, pl.LINEAR, 1.0, eps=1e-10)
        assert stats.fp64_engine_used == pl.FP64_OZAKI
    # a row whose peak exceeds 64 x its RMS needs more than ~ d = 4096 features of mass 1e-4
    Xw = rng.standard_normal((m, 8192)) * 1e-4
    Xw[:, 0] += np.where(np.arange(m) == 5, 1.0, 0.0)  # row 5: peak 1 / sqrt((1 + 8191e-8) / 8192) ~ 90
    yw = y
    a_auto, b_auto, st, stats = pl.plssvm_train_ex(Xw, yw, pl.LINEAR, 1.0, eps=1e-10)
    assert st == 0 and stats.fp64_engine_used == pl.FP64_DMMA
    a_ref, b_ref, _, _ = oracle.train(Xw, yw, pl.LINEAR, 1.0, eps=1e-10)
    assert rel(a_auto, a_ref) <= 1e-7


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("kernel", KERNELS)
def test_train_and_predict_both_engines(kernel, engine):
    rng = np.random.default_rng(40 + kernel)
    m, d, n = 777, 45, 333
    X = rng.standard_normal((m, d))
    y = np.where(X[:, 0] + 0.3 * rng.standard_normal(m) > 0, 1.0, -1.0)
    Z = rng.standard_normal((n, d))
    gamma, degree, coef0 = 1.0 / d, 3, 0.5 if kernel == pl.POLYNOMIAL else 0.0
    a_ref, b_ref, _, _ = oracle.train(X, y, kernel, gamma, degree, coef0, 1.0, 1e-10)
    alpha, b, st, stats = pl.plssvm_train_ex(X, y, kernel, gamma, degree, coef0, 1.0, 1e-10,
                                             opts=pl.options(fp64_engine=engine))
    assert st == 0 and stats.fp64_engine_used == engine
    assert rel(alpha, a_ref) <= 1e-7
    assert abs(b - b_ref) <= 1e-7 * max(abs(b_ref), np.abs(a_ref).max())
    f_ref, lab_ref = oracle.predict(X, alpha, b, Z, kernel, gamma, degree, coef0)
    f, lab, _ = pl.plssvm_predict_ex(X, alpha, b, Z, kernel, gamma, degree, coef0,
                                     opts=pl.options(fp64_engine=engine, linear_w=0))
    assert rel(f, f_ref) <= 1e-12
    assert np.array_equal(lab, lab_ref)


def test_engines_agree_on_planes_c1_slice():
    """The two engines on the same 4096 x 1024 slice of the bench workload (C1 shape family):
    products agree to ~1e-15, i.e. far inside the 1e-12 bar each meets against the oracle."""
    import synth

    cfg = synth.configs()["C1"]
    X, _, _, _ = synth.config_data(cfg, m=4096, n_test=0)
    p = np.random.default_rng(2).standard_normal(4095)
    a, _ = pl.plssvm_qtilde_matvec(X, p, cfg.kernel, cfg.gamma, opts=pl.options(fp64_engine=pl.FP64_OZAKI))
    b, _ = pl.plssvm_qtilde_matvec(X, p, cfg.kernel, cfg.gamma, opts=pl.options(fp64_engine=pl.FP64_DMMA))
    assert rel(a, b) <= 1e-14


def test_wide_d_limit():
    """int32 level sums bound d (<= 16384): AUTO switches to DMMA beyond it, forced OZAKI refuses."""
    rng = np.random.default_rng(8)
    m, d = 400, 16400  # > 384 points: AUTO's tiny-problem rule would pick DMMA regardless of d
    X = rng.standard_normal((m, d)) * 0.05
    y = np.where(np.arange(m) % 2 == 0, 1.0, -1.0)
    alpha, b, st, stats = pl.plssvm_train_ex(X, y, pl.RBF, 1.0 / d, eps=1e-10)
    assert st == 0 and stats.fp64_engine_used == pl.FP64_DMMA
    a_ref, _, _, _ = oracle.train(X, y, pl.RBF, 1.0 / d, eps=1e-10)
    assert rel(alpha, a_ref) <= 1e-7
    with pytest.raises(pl.PlssvmError, match="d <= 16384"):
        pl.plssvm_train_ex(X, y, pl.RBF, 1.0 / d, eps=1e-10, opts=pl.options(fp64_engine=pl.FP64_OZAKI))
    X2 = X[:, :16384].copy()
    alpha, b, st, stats = pl.plssvm_train_ex(X2, y, pl.RBF, 1.0 / 16384, eps=1e-10)
    assert st == 0 and stats.fp64_engine_used == pl.FP64_OZAKI
    a_ref, _, _, _ = oracle.train(X2, y, pl.RBF, 1.0 / 16384, eps=1e-10)
    assert rel(alpha, a_ref) <= 1e-7


@pytest.mark.parametrize("gamma", [1e-7, 1.0 / 64, 0.3, 2.0, 40.0])
def test_ozaki_rbf_table_exp_across_the_exponent_range(gamma):
    """The Ozaki epilogue evaluates exp(-gamma ||x_i - x_j||^2) with a 64-entry 2^(j/64) table and a
    degree-5 polynomial (ozaki_engine.cuh exp_tab): kernel values from ~1 down through the
    2^-1022 cut-off (gamma = 40 on 64-feature N(0,1) data gives exponents far below -708) must
    still give the oracle's product within 1e-12, in implicit, cached and predict paths."""
    rng = np.random.default_rng(int(gamma * 1000) + 5)
    m, d = 600, 64
    X = rng.standard_normal((m, d))
    X[5] = X[4] + 1e-9  # near-duplicate point: exponent ~ -gamma 1e-16, kernel ~ 1
    p = rng.standard_normal(m - 1)
    for mode in (pl.MODE_IMPLICIT, pl.MODE_CACHED):
        check(X, p, pl.RBF, gamma, engine=pl.FP64_OZAKI, mode=mode)
    Z = rng.standard_normal((300, d)) * 0.5
    alpha = rng.standard_normal(m)
    f, _, _ = pl.plssvm_predict_ex(X, alpha, 0.25, Z, pl.RBF, gamma=gamma, opts=pl.options(fp64_engine=pl.FP64_OZAKI))
    f_ref, _ = oracle.predict(X, alpha, 0.25, Z, pl.RBF, gamma)
    K = np.exp(-gamma * ((Z[:, None, :] - X[None, :, :]) ** 2).sum(-1))
    assert np.all(np.abs(f - f_ref) <= 1e-12 * (np.abs(K) @ np.abs(alpha) + 0.25))


def test_auto_picks_dmma_for_tiny_problems():
    """AUTO: at most 384 padded points -> DMMA (the persistent int8 kernel's fixed cost dominates);
    both engines stay within the parity bar there."""
    rng = np.random.default_rng(12)
    for m, want in ((256, pl.FP64_DMMA), (300, pl.FP64_DMMA), (385, pl.FP64_OZAKI)):
        X = rng.standard_normal((m, 20))
        y = np.where(rng.random(m) < 0.5, 1.0, -1.0)
        y[0], y[1] = 1.0, -1.0
        a, b, st, stats = pl.plssvm_train_ex(X, y, pl.RBF, 0.05, eps=1e-10)
        assert st == 0 and stats.fp64_engine_used == want, (m, stats.fp64_engine_used)
        a_ref, _, _, _ = oracle.train(X, y, pl.RBF, 0.05, eps=1e-10)
        assert rel(a, a_ref) <= 1e-7
