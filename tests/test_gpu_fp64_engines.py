"""GPU parity of the two fp64 contraction engines (include/plssvm.h plssvm_fp64_engine_t):
OZAKI (int8 tensor cores on an exact 7-digit split of every point, 2-SM UMMA) and DMMA (fp64
tensor cores), plus the AUTO rule, against the CPU oracle.  Bars as in test_gpu_parity.py:
product <= 1e-12 norm-wise and |y_i - y*_i| <= 1e-12 (|Q~||p|)_i element-wise; alpha, b <= 1e-7.

The Ozaki error bound is u|s| + 13.04 d u ||x_i||_inf ||x_j||_inf per inner product s (u = 2^-53,
DESIGN.md §5), so the cases below stress what the row-max scaling could get wrong: ragged shapes around the 32-feature slab and
the 128/256-point (pair-)tile edges, magnitudes far from 1, exact-integer data, zero rows,
duplicated points, odd band / pair ends on several ranks (test_gpu_multirank.py), peaked rows across
the band peak / RMS = 12 .. 63 forced onto the int8 engine, the bound entry by entry, and the AUTO
rule (OZAKI iff 13.04 rho^2 <= d)."""
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


def peaked(rng, m, d, rho, sigma_scale=1.0, spike_col=None):
    """m rows of spike + noise with max_k |x_k| / rms_k(x_k) = rho exactly: the spike s = sigma_scale sits
    in column spike_col(i) (default: random, so different rows' spikes are mostly orthogonal)."""
    X = np.empty((m, d))
    for i in range(m):
        s = sigma_scale * (1.0 + rng.random())
        sig = s * np.sqrt(max(d / rho**2 - 1.0, 0.0) / (d - 1))
        x = rng.standard_normal(d)
        x *= sig / max(np.sqrt(np.mean(x**2)), 1e-300)
        k = rng.integers(0, d) if spike_col is None else spike_col(i)
        x = np.clip(x, -0.99 * s, 0.99 * s)
        x[k] = s if rng.random() < 0.5 else -s
        ss = np.sum(x**2) - s * s  # rescale the noise so that rho is exact
        want = s * s * (d / rho**2) - s * s
        if ss > 0 and want > 0:
            mask = np.arange(d) != k
            x[mask] *= np.sqrt(want / ss)
        X[i] = x
    return X


def row_peak(X):
    return np.max(np.abs(X).max(1) / np.sqrt((X**2).mean(1)))


@pytest.mark.parametrize("rho", [12, 24, 32, 48, 63])
@pytest.mark.parametrize("kernel", KERNELS)
def test_ozaki_forced_across_the_peak_band(rho, kernel):
    """rows with peak / RMS = rho (spike + small noise, spikes of different rows mostly
    orthogonal), FORCED onto the int8 engine: the product meets the parity bars against the oracle
    (1e-12 norm- and element-wise vs |Q~||p|), in implicit and cached mode; and the model trained on
    them meets the 1e-7 bar.  d = 4096 so that rho up to 63 is possible (rho <= sqrt(d))."""
    rng = np.random.default_rng(1000 * rho + kernel)
    m, d = 400, 4096
    X = peaked(rng, m, d, rho)
    assert abs(row_peak(X) - rho) <= 1e-6 * rho
    p = rng.standard_normal(m - 1)
    gamma = 1.0 / d if kernel != pl.LINEAR else 1.0
    for mode in (pl.MODE_IMPLICIT, pl.MODE_CACHED):
        check(X, p, kernel, gamma, engine=pl.FP64_OZAKI, mode=mode)
    y = np.where(rng.random(m) < 0.5, 1.0, -1.0)
    y[0], y[1] = 1.0, -1.0
    a_ref, b_ref, _, st_ref = oracle.train(X, y, kernel, gamma, 3, 0.5, 1.0, 1e-10)
    a, b, st, s = pl.plssvm_train_ex(X, y, kernel, gamma, 3, 0.5, 1.0, 1e-10,
                                     opts=pl.options(fp64_engine=pl.FP64_OZAKI, mode=pl.MODE_IMPLICIT))
    assert st == st_ref == 0 and s.fp64_engine_used == pl.FP64_OZAKI
    assert rel(a, a_ref) <= 1e-7 and abs(b - b_ref) <= 1e-7 * max(abs(b_ref), np.abs(a_ref).max())


@pytest.mark.parametrize("rho", [8, 32, 63])
def test_ozaki_entries_within_the_derived_bound(rho):
    """Per-entry check of the documented bound (ozaki_engine.cuh): with p = e_j the product
    is column j of Q~, so Q~_ij = k_ij - q_i - q_j + Q_mm comes out entry by entry; for the linear kernel
    |Q~gpu_ij - Q~_ij| <= 13.04 d u ||x_i||inf ||x_j||inf (the contraction) + the fp64 rounding of Eq. 16's
    four terms and of the oracle's own dot products (4 u (|k_ij| + |q_i| + |q_j| + Q_mm) + d u sum|x x|)."""
    rng = np.random.default_rng(77 + rho)
    m, d = 300, 4096
    X = peaked(rng, m, d, rho)
    u = 2.0**-53
    Qt = oracle.qtilde(X, pl.LINEAR, 1.0, 3, 0.0, 1e300)  # C = 1e300: the 1/C terms vanish
    q, Qmm = oracle.q_cache(X, pl.LINEAR, C=1e300)
    inf = np.abs(X).max(1)
    absdot = np.abs(X) @ np.abs(X).T
    for j in (0, 7, 150, m - 2):
        e = np.zeros(m - 1)
        e[j] = 1.0
        col, _ = pl.plssvm_qtilde_matvec(X, e, pl.LINEAR, 1.0, 3, 0.0, 1e300,
                                         opts=pl.options(mode=pl.MODE_IMPLICIT, fp64_engine=pl.FP64_OZAKI))
        k = Qt[:, j] + q + q[j] - Qmm
        bound = (13.04 * d * u * inf[:-1] * inf[j] + 4 * u * (np.abs(k) + np.abs(q) + abs(q[j]) + Qmm)
                 + d * u * absdot[:-1, j])
        err = np.abs(col - Qt[:, j])
        assert np.all(err <= bound), (j, np.max(err / bound))


def test_auto_rule_follows_the_bound_and_stays_exact():
    """AUTO takes OZAKI iff 13.04 rho^2 <= d (driver.cu oz_choose): on each side of the threshold the engine
    choice is as the rule says and the trained model meets the 1e-7 bar."""
    rng = np.random.default_rng(4)
    m, d = 400, 1024  # threshold rho* = sqrt(1024 / 13.04) = 8.86
    y = np.where(rng.random(m) < 0.5, 1.0, -1.0)
    y[0], y[1] = 1.0, -1.0
    for rho, want in ((6.0, pl.FP64_OZAKI), (8.5, pl.FP64_OZAKI), (9.5, pl.FP64_DMMA), (30.0, pl.FP64_DMMA)):
        X = rng.standard_normal((m, d))
        X[17] = peaked(rng, 1, d, rho)[0]  # the N(0,1) rows peak at ~4.5: this row decides
        rho_max = row_peak(X)
        a, b, st, s = pl.plssvm_train_ex(X, y, pl.RBF, 1.0 / d, eps=1e-10)
        assert st == 0 and s.fp64_engine_used == want, (rho, rho_max, s.fp64_engine_used)
        assert (13.04 * rho_max**2 <= d) == (want == pl.FP64_OZAKI)
        a_ref, b_ref, _, _ = oracle.train(X, y, pl.RBF, 1.0 / d, eps=1e-10)
        assert rel(a, a_ref) <= 1e-7 and abs(b - b_ref) <= 1e-7 * max(abs(b_ref), np.abs(a_ref).max())


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
    d = 512  # N(0,1) rows peak at rho ~ 4.3: 13.04 rho^2 < d, so only the size rule decides
    for m, want in ((256, pl.FP64_DMMA), (300, pl.FP64_DMMA), (385, pl.FP64_OZAKI)):
        X = rng.standard_normal((m, d))
        y = np.where(rng.random(m) < 0.5, 1.0, -1.0)
        y[0], y[1] = 1.0, -1.0
        a, b, st, stats = pl.plssvm_train_ex(X, y, pl.RBF, 1.0 / d, eps=1e-10)
        assert st == 0 and stats.fp64_engine_used == want, (m, stats.fp64_engine_used)
        a_ref, _, _, _ = oracle.train(X, y, pl.RBF, 1.0 / d, eps=1e-10)
        assert rel(a, a_ref) <= 1e-7


def test_exponent_range_limit():
    """The epilogue builds the digit scales' exponents directly (ozaki_engine.cuh scaled_exact: 2^k V in
    one fp64 operation), which needs row maxima within 2^-480 .. 2^480 (driver.cu kOzMaxExp): rows at
    2^-470 and 2^470 still run on OZAKI within the parity bars; a row at 2^-500 makes AUTO take DMMA
    and forced OZAKI refuse."""
    rng = np.random.default_rng(21)
    m, d = 600, 64
    X = rng.standard_normal((m, d))
    X[7] *= 2.0 ** -470
    X[9] *= 2.0 ** 470
    p = rng.standard_normal(m - 1)
    Qt = oracle.qtilde(X, pl.LINEAR, 1.0, 3, 0.0, 1.0)
    ref = oracle.matvec(Qt, p)
    scale = np.abs(Qt) @ np.abs(p)
    s0 = np.abs(ref).max()  # ~2^940: normalise before the norms (their squares would overflow)
    for mode in (pl.MODE_IMPLICIT, pl.MODE_CACHED):
        out, _ = pl.plssvm_qtilde_matvec(X, p, pl.LINEAR, 1.0, 3, 0.0, 1.0,
                                         opts=pl.options(mode=mode, fp64_engine=pl.FP64_OZAKI))
        assert rel(out / s0, ref / s0) <= 1e-12
        assert np.all(np.abs(out - ref) <= 1e-12 * scale)
    X2 = rng.standard_normal((m, d))
    X2[7] *= 2.0 ** -470
    check(X2, p, pl.RBF, 1.0 / d, engine=pl.FP64_OZAKI)
    # AUTO's own rule: at d = 1024 N(0,1) rows pass the peak test (13.04 rho^2 <= d), so only the
    # exponent range decides
    X3 = rng.standard_normal((m, 1024))
    y = np.where(np.arange(m) % 2 == 0, 1.0, -1.0)
    _, _, st, stats = pl.plssvm_train_ex(X3, y, pl.RBF, 1.0 / 1024, eps=1e-10)
    assert st == 0 and stats.fp64_engine_used == pl.FP64_OZAKI
    X3[7] *= 2.0 ** -500
    alpha, b, st, stats = pl.plssvm_train_ex(X3, y, pl.RBF, 1.0 / 1024, eps=1e-10)
    assert st == 0 and stats.fp64_engine_used == pl.FP64_DMMA
    a_ref, _, _, _ = oracle.train(X3, y, pl.RBF, 1.0 / 1024, eps=1e-10)
    assert rel(alpha, a_ref) <= 1e-7
    with pytest.raises(pl.PlssvmError, match="row maxima within"):
        pl.plssvm_train_ex(X3, y, pl.RBF, 1.0 / 1024, eps=1e-10, opts=pl.options(fp64_engine=pl.FP64_OZAKI))


@pytest.mark.parametrize("d", [8096, 8128])
def test_conversion_width_boundary(d):
    """|V| < 2^51 (the one-operation conversion of pass 0's levels) holds up to d8 = 8096; wider points
    convert V exactly in pass 0 instead (ozaki_engine.cuh bigd).  Both sides of the switch vs the oracle."""
    rng = np.random.default_rng(d)
    m = 420
    X = rng.standard_normal((m, d))
    p = rng.standard_normal(m - 1)
    check(X, p, pl.RBF, 1.0 / d, engine=pl.FP64_OZAKI)
    check(X, p, pl.LINEAR, 1.0, engine=pl.FP64_OZAKI)
