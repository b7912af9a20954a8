"""fp32 on the int8 tensor cores (options.fp32_engine = OZAKI): every point split into 3 balanced
base-256 digits (rounded to 22 bits below its row maximum), the 6 digit pairs of levels <= 2
summed exactly in int32 by the same 2-SM tcgen05 kernel as the fp64 engine (one TMEM pass), the
epilogue in fp32.  Bars as every fp32 path (north_star): product <= 1e-5 norm-wise and
element-wise against (|Q~||p|)_i, vs the oracle on the fp32-rounded inputs (R-12);
predict <= 1e-5; training reaches the tcgen05 engine's model to fp32 CG accuracy."""
import numpy as np
import pytest

import oracle
import paper_2202_12674_b200 as pl
import synth

pytestmark = pytest.mark.gpu
KERNELS = [pl.LINEAR, pl.POLYNOMIAL, pl.RBF]


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("m,d", [(2, 1), (129, 3), (257, 33), (1000, 33), (2177, 70), (4097, 300)])
def test_fp32_ozaki_product_matches_oracle(m, d, kernel):
    rng = np.random.default_rng(7000 * m + d + kernel)
    X = rng.standard_normal((m, d)).astype(np.float32)
    p = rng.standard_normal(m - 1).astype(np.float32)
    gamma = float(np.float32(1.0 / d))
    coef0 = 0.5 if kernel == pl.POLYNOMIAL else 0.0
    Qt = oracle.qtilde(X.astype(np.float64), kernel, gamma, 3, coef0, 1.0)
    ref = Qt @ p.astype(np.float64)
    scale = np.abs(Qt) @ np.abs(p.astype(np.float64))
    for mode in (pl.MODE_IMPLICIT, pl.MODE_CACHED):
        out, _ = pl.plssvm_qtilde_matvec(X, p, kernel, gamma, 3, coef0, 1.0,
                                         opts=pl.options(mode=mode, fp32_engine=pl.FP32_OZAKI))
        out = out.astype(np.float64)
        assert rel(out, ref) <= 1e-5, (mode, rel(out, ref))
        assert np.all(np.abs(out - ref) <= 1e-5 * scale + 1e-30), np.max(np.abs(out - ref) / scale)


@pytest.mark.parametrize("kernel", KERNELS)
def test_fp32_ozaki_predict_and_train(kernel):
    X, y, Z, yz = synth.planes(1500, 40, 400, seed=90 + kernel)
    X, y, Z = X.astype(np.float32), y.astype(np.float32), Z.astype(np.float32)
    gamma = float(np.float32(1.0 / 40))
    coef0 = 0.5 if kernel == pl.POLYNOMIAL else 0.0
    a, b, st, s = pl.plssvm_train_ex(X, y, kernel, gamma, 3, coef0, 1.0, 1e-6,
                                     opts=pl.options(fp32_engine=pl.FP32_OZAKI, mode=pl.MODE_IMPLICIT))
    a2, b2, st2, s2 = pl.plssvm_train_ex(X, y, kernel, gamma, 3, coef0, 1.0, 1e-6,
                                         opts=pl.options(fp32_engine=pl.FP32_TCGEN05, mode=pl.MODE_IMPLICIT))
    assert st == st2 == 0 and abs(s.iterations - s2.iterations) <= 3
    assert rel(a, a2) <= 1e-3  # fp32 CG accuracy (R-12)
    f, lab, _ = pl.plssvm_predict_ex(X, a, float(b), Z, kernel, gamma, 3, coef0,
                                     opts=pl.options(fp32_engine=pl.FP32_OZAKI))
    f_ref, _ = oracle.predict(X.astype(np.float64), a.astype(np.float64), float(b), Z.astype(np.float64), kernel,
                              gamma, 3, coef0)
    # element-wise against sum_i |alpha_i| |k(x_i, z)| + |b| (the matvec bar's form): the split's
    # error is relative to the row maxima, not to |f| (trained alphas cancel in f)
    Xd, Zd = X.astype(np.float64), Z.astype(np.float64)
    if kernel == pl.LINEAR:
        K = Zd @ Xd.T
    elif kernel == pl.POLYNOMIAL:
        K = (gamma * (Zd @ Xd.T) + coef0) ** 3
    else:
        K = np.exp(-gamma * ((Zd[:, None, :] - Xd[None, :, :]) ** 2).sum(-1))
    scale = np.abs(K) @ np.abs(a.astype(np.float64)) + abs(float(b))
    assert np.all(np.abs(f - f_ref) <= 1e-5 * scale), np.max(np.abs(f - f_ref) / scale)


def test_fp32_ozaki_scale_and_peaked_rows():
    """Magnitudes far from 1 and rows with one large feature: the split is per row, the bound is
    d 2^-22 ||x_i||_inf ||x_j||_inf, so a peaked row loses relative accuracy in its small features
    -- still inside the fp32 bar on these data (the fp32 AUTO choice stays the tcgen05 engine)."""
    rng = np.random.default_rng(5)
    m, d = 700, 50
    X = (rng.standard_normal((m, d)) * 3.7e-3).astype(np.float32)
    X[::7, 3] *= 20.0
    p = rng.standard_normal(m - 1).astype(np.float32)
    Qt = oracle.qtilde(X.astype(np.float64), pl.LINEAR, 1.0, 3, 0.0, 1.0)
    ref = Qt @ p.astype(np.float64)
    out, _ = pl.plssvm_qtilde_matvec(X, p, pl.LINEAR, 1.0, 3, 0.0, 1.0,
                                     opts=pl.options(mode=pl.MODE_IMPLICIT, fp32_engine=pl.FP32_OZAKI))
    assert rel(out, ref) <= 1e-5, rel(out, ref)


@pytest.mark.parametrize("kernel", KERNELS)
def test_fp32_ozaki_zero_and_duplicate_rows(kernel):
    """Zero rows (E = 0, all digits 0) and duplicated points (exact-zero RBF distance): the product
    stays within the fp32 bars against the oracle on the same fp32 inputs.  (Rows scaled by 1e15
    are NOT a fair fp32 case: Eq. 16's q corrections then cancel catastrophically in any fp32
    arithmetic -- tools/diag_fp32_rows.py: int8 2.7e-3, 3xTF32 7.3e-4, even FFMA 3.4e-5 of |Q~||p|.)"""
    rng = np.random.default_rng(77 + kernel)
    m, d = 600, 40
    X = rng.standard_normal((m, d)).astype(np.float32)
    X[10] = 0.0
    X[11] = X[12]
    X[30:40] = 0.0
    p = rng.standard_normal(m - 1).astype(np.float32)
    gamma = float(np.float32(1.0 / d))
    coef0 = 0.5 if kernel == pl.POLYNOMIAL else 0.0
    Qt = oracle.qtilde(X.astype(np.float64), kernel, gamma, 3, coef0, 1.0)
    ref = Qt @ p.astype(np.float64)
    scale = np.abs(Qt) @ np.abs(p.astype(np.float64))
    for mode in (pl.MODE_IMPLICIT, pl.MODE_CACHED):
        out, _ = pl.plssvm_qtilde_matvec(X, p, kernel, gamma, 3, coef0, 1.0,
                                         opts=pl.options(mode=mode, fp32_engine=pl.FP32_OZAKI))
        out = out.astype(np.float64)
        assert np.all(np.abs(out - ref) <= 1e-5 * scale + 1e-30), (mode, np.max(np.abs(out - ref) / scale))
