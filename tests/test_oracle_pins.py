"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Nothing here compares the oracle with itself: every expected value is (a) printed in the
paper/spec worked examples (tests/golden, each fixture cites its passage), (b) an exact
rational solution of the full LS-SVM system Eq. 11 computed here by Fraction
Gaussian elimination, (c) a library routine applied to a DIFFERENT formulation (dense LU of
the full KKT matrix instead of the reduced CG route; B^T Q B instead of Eq. 16; ridge
regression closed form for the linear kernel; scipy cdist/cho_solve), or (d) an invariant.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg
from scipy.spatial.distance import cdist

import oracle
import synth
from conftest import load_golden

KERNELS = [oracle.LINEAR, oracle.POLYNOMIAL, oracle.RBF]


# ---------------------------------------------------------------- independent references
def gram_lib(X, Z, kernel, gamma, degree, coef0):
    """Kernel matrix through library primitives (BLAS matmul / scipy cdist)."""
    if kernel == oracle.LINEAR:
        return X @ Z.T
    if kernel == oracle.POLYNOMIAL:
        return np.power(gamma * (X @ Z.T) + coef0, degree)
    return np.exp(-gamma * cdist(X, Z, "sqeuclidean"))


def kkt_solve(X, y, kernel, gamma, degree, coef0, C):
    """Dense LU solve of the FULL system Eq. 11: [[Q, 1],[1^T, 0]] [alpha; b] = [y; 0]."""
    m = X.shape[0]
    Q = gram_lib(X, X, kernel, gamma, degree, coef0) + np.eye(m) / C
    A = np.zeros((m + 1, m + 1))
    A[:m, :m] = Q
    A[:m, m] = 1.0
    A[m, :m] = 1.0
    sol = np.linalg.solve(A, np.concatenate([y, [0.0]]))
    return sol[:m], sol[m]


def frac_solve(A, rhs):
    """Exact Gaussian elimination over the rationals (textbook, partial pivot on nonzero)."""
    n = len(A)
    M = [list(map(Fraction, row)) + [Fraction(r)] for row, r in zip(A, rhs)]
    for c in range(n):
        piv = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[piv] = M[piv], M[c]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c] / M[c][c]
                M[r] = [a - f * b for a, b in zip(M[r], M[c])]
    return [M[i][n] / M[i][i] for i in range(n)]


def frac_kernel(a, b, kernel, gamma, degree, coef0):
    s = sum(Fraction(x) * Fraction(z) for x, z in zip(a, b))
    if kernel == 0:
        return s
    if kernel == 1:
        return (Fraction(gamma) * s + Fraction(coef0)) ** degree
    raise ValueError("exact RBF not rational")


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- kernel functions
def test_kernel_closed_forms():
    # S:186-189 worked values
    assert oracle.kernel([1, 2], [3, 4], oracle.LINEAR) == 11.0
    assert oracle.kernel([0.3, -1.7, 2.0], [0.3, -1.7, 2.0], oracle.RBF, gamma=3.0) == 1.0
    assert oracle.kernel([0, 0], [1, 0], oracle.RBF, gamma=0.5) == math.exp(-0.5)
    assert abs(oracle.kernel([0, 0], [1, 0], oracle.RBF, gamma=0.5) - 0.60653065971263342) < 1e-16
    # (1*11 + 1)^3 = 1728 exactly; integer degree by repeated multiplication
    assert oracle.kernel([1, 2], [3, 4], oracle.POLYNOMIAL, gamma=1.0, degree=3, coef0=1.0) == 1728.0
    # 3-4-5 triangle: ||x-z||^2 = 25, gamma = 1/25 -> e^-1
    assert abs(oracle.kernel([0, 0], [3, 4], oracle.RBF, gamma=1 / 25) - math.exp(-1)) < 1e-16


def test_poly_degree1_equals_linear():
    rng = np.random.default_rng(1)
    for _ in range(20):
        a, b = rng.standard_normal(7), rng.standard_normal(7)
        assert oracle.kernel(a, b, oracle.POLYNOMIAL, 1.0, 1, 0.0) == oracle.kernel(a, b, oracle.LINEAR)


def test_kernel_matches_library_gram():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((9, 5))
    for k, (g, deg, r) in [(oracle.LINEAR, (1, 1, 0)), (oracle.POLYNOMIAL, (0.3, 3, 0.5)),
                           (oracle.RBF, (0.2, 1, 0))]:
        G = gram_lib(X, X, k, g, deg, r)
        for i in range(9):
            for j in range(9):
                v = oracle.kernel(X[i], X[j], k, g, deg, r)
                assert abs(v - G[i, j]) <= 1e-13 * max(1.0, abs(G[i, j]))
                assert v == oracle.kernel(X[j], X[i], k, g, deg, r)  # exact symmetry


# ---------------------------------------------------------------- worked examples (golden)
GOLDEN = ["spec_3point_linear.txt", "square_4point_linear.txt", "square_4point_poly.txt",
          "generic_4point_linear.txt"]


def _golden_problem(g):
    X = np.array([[float(v) for v in row] for row in g["X"]])
    y = np.array([float(v) for v in g["labels"]])
    return X, y, int(g["kernel"]), float(g["gamma"]), int(g["degree"]), float(g["coef0"]), float(g["C"])


@pytest.mark.parametrize("name", GOLDEN)
def test_golden_fixture_solves_eq11_exactly(name):
    """The fixture's (alpha, b) is the exact solution of Eq. 11 (rational arithmetic)."""
    g = load_golden(name)
    X = g["X"]
    m = len(X)
    k, gam, deg, r, C = int(g["kernel"]), g["gamma"], int(g["degree"]), g["coef0"], g["C"]
    A = [[frac_kernel(X[i], X[j], k, gam, deg, r) + (Fraction(1) / C if i == j else 0) for j in range(m)]
         + [Fraction(1)] for i in range(m)] + [[Fraction(1)] * m + [Fraction(0)]]
    sol = frac_solve(A, list(g["labels"]) + [0])
    assert sol[:m] == list(g["alpha"])
    assert sol[m] == g["b"]


@pytest.mark.parametrize("name", GOLDEN)
def test_oracle_on_golden(name):
    g = load_golden(name)
    X, y, k, gam, deg, r, C = _golden_problem(g)
    q, Qmm = oracle.q_cache(X, k, gam, deg, r, C)
    if "q" in g:
        assert list(q) == [float(v) for v in g["q"]]
        assert Qmm == float(g["Qmm"])
    if "Qtilde" in g:
        Qt = oracle.qtilde(X, k, gam, deg, r, C)
        assert Qt.tolist() == [[float(v) for v in row] for row in g["Qtilde"]]
        p = np.array([float(v) for v in g["matvec_p"]])
        assert oracle.matvec(Qt, p).tolist() == [float(v) for v in g["matvec_y"]]
    alpha, b, it, st = oracle.train(X, y, k, gam, deg, r, C, eps=1e-14)
    assert st == oracle.OK
    assert np.allclose(alpha, [float(v) for v in g["alpha"]], rtol=0, atol=1e-13)
    assert abs(b - float(g["b"])) <= 1e-13
    if "decision" in g:
        Z = np.array([[float(v) for v in row] for row in g["Z"]])
        f, lab = oracle.predict(X, np.array([float(v) for v in g["alpha"]]), float(g["b"]), Z, k, gam, deg, r)
        assert np.allclose(f, [float(v) for v in g["decision"]], rtol=0, atol=1e-14)
        assert lab.tolist() == [1 if float(v) >= 0 else -1 for v in g["decision"]]


def test_tie_break_exact_zero_is_plus_one():
    # sgn(0) -> +1.  f(1/4, 1/2) = 0 exactly with the exact alpha, b.
    g = load_golden("square_4point_linear.txt")
    X = np.array([[float(v) for v in row] for row in g["X"]])
    f, lab = oracle.predict(X, np.array([0.5, 0.5, -0.5, -0.5]), 0.5, np.array([[0.25, 0.5]]), oracle.LINEAR)
    assert f[0] == 0.0 and lab[0] == 1
    f, lab = oracle.predict(X, np.array([0.5, 0.5, -0.5, -0.5]), 0.5 - 2**-40, np.array([[0.25, 0.5]]),
                            oracle.LINEAR)
    assert f[0] < 0 and lab[0] == -1


# ---------------------------------------------------------------- dense KKT (Eq. 11) pins
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("C", [0.1, 1.0, 10.0])
def test_train_matches_dense_kkt_lu(kernel, C):
    rng = np.random.default_rng(100 + kernel * 10 + int(C * 10))
    for trial in range(5):
        m, d = int(rng.integers(2, 64)), int(rng.integers(1, 9))
        X, y = synth.random_small(rng, m, d)
        gam, deg, r = 1.0 / d, int(rng.integers(1, 4)), float(rng.uniform(0, 1))
        a_ref, b_ref = kkt_solve(X, y, kernel, gam, deg, r, C)
        alpha, b, it, st = oracle.train(X, y, kernel, gam, deg, r, C, eps=1e-13)
        assert st in (oracle.OK, oracle.W_NOT_CONVERGED)
        assert rel(alpha, a_ref) <= 1e-8, (m, d, trial)
        assert abs(b - b_ref) <= 1e-8 * max(abs(b_ref), np.abs(a_ref).max())
        assert abs(alpha.sum()) <= 1e-12 * (1 + np.abs(alpha).max())  # 1^T alpha = 0 (Eq. 11 last row)


def test_m2_closed_form():
    # m = 2: alpha~ = (y1 - y2) / (k11 - 2 k12 + k22 + 2/C)
    X = np.array([[0.5, -1.0], [2.0, 0.25]])
    y = np.array([1.0, -1.0])
    for C in (0.5, 3.0):
        K = X @ X.T
        a1 = (y[0] - y[1]) / (K[0, 0] - 2 * K[0, 1] + K[1, 1] + 2 / C)
        alpha, b, it, st = oracle.train(X, y, oracle.LINEAR, C=C, eps=1e-14)
        assert abs(alpha[0] - a1) <= 1e-15 * abs(a1) * 4 and alpha[1] == -alpha[0]
        assert it == 1


# ---------------------------------------------------------------- Q~ structure pins
@pytest.mark.parametrize("kernel", KERNELS)
def test_qtilde_equals_BtQB(kernel):
    """Eq. 13 as a congruence: Q~ = B^T Q B with B = [I; -1^T] (independent of Eq. 16)."""
    rng = np.random.default_rng(7 + kernel)
    for C in (0.1, 1.0, 10.0):
        m, d = 40, 6
        X, _ = synth.random_small(rng, m, d)
        Q = gram_lib(X, X, kernel, 0.3, 3, 0.7) + np.eye(m) / C
        B = np.vstack([np.eye(m - 1), -np.ones((1, m - 1))])
        ref = B.T @ Q @ B
        Qt = oracle.qtilde(X, kernel, 0.3, 3, 0.7, C)
        assert rel(Qt, ref) <= 1e-13
        assert rel(Qt, Qt.T) <= 1e-15  # symmetric up to the rounding order of Eq. 16's terms
        # SPD with lambda_min >= 1/C (Q >= I/C and B^T B = I + 11^T >= I)
        scipy.linalg.cholesky(Qt)
        assert np.linalg.eigvalsh(Qt).min() >= (1.0 / C) * (1 - 1e-9)


def test_qtilde_rows_match_full():
    rng = np.random.default_rng(11)
    X, _ = synth.random_small(rng, 30, 4)
    Qt = oracle.qtilde(X, oracle.RBF, 0.25)
    rows = [0, 5, 28]
    assert np.array_equal(oracle.qtilde_rows(X, rows, oracle.RBF, 0.25), Qt[rows])


def test_matvec_matches_blas():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((300, 300))
    p = rng.standard_normal(300)
    assert rel(oracle.matvec(A, p), A @ p) <= 1e-14


# ---------------------------------------------------------------- CG pins
def test_cg_worked_2x2():
    # Q~ = [[6,3],[3,3]], rhs = (2,2) -> (0, 2/3)
    x, it, st = oracle.cg(np.array([[6.0, 3.0], [3.0, 3.0]]), np.array([2.0, 2.0]), eps=1e-12)
    assert st == oracle.OK and np.allclose(x, [0.0, 2.0 / 3.0], atol=1e-14) and it <= 2


def test_cg_identity_one_iteration_and_zero_rhs():
    b = np.arange(1.0, 6.0)
    x, it, st = oracle.cg(np.eye(5), b, eps=1e-12)
    assert it == 1 and np.array_equal(x, b) and st == oracle.OK
    x, it, st = oracle.cg(np.eye(5) * 3, np.zeros(5), eps=1e-12)  # rhs = 0 -> 0 iterations
    assert it == 0 and np.array_equal(x, np.zeros(5)) and st == oracle.OK


def test_cg_matches_cholesky_and_recurrence_contract():
    rng = np.random.default_rng(5)
    X, y = synth.random_small(rng, 200, 10)
    Qt = oracle.qtilde(X, oracle.RBF, 0.1, C=1.0)
    rhs = y[:-1] - y[-1]
    x, it, st, tr = oracle.cg(Qt, rhs, eps=1e-11, trace=True)
    ref = scipy.linalg.cho_solve(scipy.linalg.cho_factor(Qt), rhs)
    kappa = np.linalg.cond(Qt)
    assert st == oracle.OK
    assert rel(x, ref) <= kappa * 1e-11 * 10
    assert tr[-1] <= 1e-11 * np.linalg.norm(rhs) and tr[-2] > 1e-11 * np.linalg.norm(rhs)
    # true residual close to the recurrence residual at this conditioning
    assert np.linalg.norm(rhs - Qt @ x) <= 1e-9 * np.linalg.norm(rhs)


def test_cg_linear_low_rank_iteration_bound():
    # Linear kernel: Q~ = I/C + rank(<= d+1)  -> exact-arithmetic CG needs <= d+2 iterations
    rng = np.random.default_rng(9)
    X, y = synth.random_small(rng, 300, 3)
    alpha, b, it, st = oracle.train(X, y, oracle.LINEAR, C=1.0, eps=1e-10)
    assert st == oracle.OK and it <= 3 + 2 + 2  # d+2 plus fp slack


def test_cg_iterations_monotone_in_eps():
    rng = np.random.default_rng(12)
    X, y = synth.random_small(rng, 150, 8)
    its = [oracle.train(X, y, oracle.RBF, 0.125, eps=e)[2] for e in (1e-2, 1e-4, 1e-6, 1e-8, 1e-10)]
    assert its == sorted(its)


# ---------------------------------------------------------------- linear kernel: ridge closed form
def test_linear_ridge_closed_form():
    """Linear LS-SVM = ridge regression with unpenalised intercept:
    w = (Xc^T Xc + I/C)^-1 Xc^T yc, b = ybar - xbar.w, alpha = C (y - X w - b)."""
    X, y, _, _ = synth.planes(400, 12, seed=77)
    C = 1.0
    xbar, ybar = X.mean(0), y.mean()
    Xc, yc = X - xbar, y - ybar
    w = np.linalg.solve(Xc.T @ Xc + np.eye(12) / C, Xc.T @ yc)
    b_ref = ybar - xbar @ w
    a_ref = C * (y - X @ w - b_ref)
    alpha, b, it, st = oracle.train(X, y, oracle.LINEAR, C=C, eps=1e-12)
    assert st == oracle.OK
    assert rel(alpha, a_ref) <= 1e-8 and abs(b - b_ref) <= 1e-8


# ---------------------------------------------------------------- invariants
def test_label_flip_and_permutation_and_rotation():
    rng = np.random.default_rng(21)
    X, y = synth.random_small(rng, 50, 5)
    a0, b0, _, _ = oracle.train(X, y, oracle.RBF, 0.2, eps=1e-13)
    a1, b1, _, _ = oracle.train(X, -y, oracle.RBF, 0.2, eps=1e-13)
    assert rel(a1, -a0) <= 1e-12 and abs(b1 + b0) <= 1e-12
    # permutation (changes which point is x_m): (alpha, b) permute, unique solution of Eq. 11
    perm = rng.permutation(50)
    a2, b2, _, _ = oracle.train(X[perm], y[perm], oracle.RBF, 0.2, eps=1e-13)
    assert rel(a2, a0[perm]) <= 1e-9 and abs(b2 - b0) <= 1e-9
    # orthogonal rotation leaves all three kernels' Gram matrices unchanged
    R, _ = np.linalg.qr(rng.standard_normal((5, 5)))
    for k in KERNELS:
        ak, bk, _, _ = oracle.train(X, y, k, 0.2, 2, 0.5, eps=1e-13)
        ar, br, _, _ = oracle.train(X @ R, y, k, 0.2, 2, 0.5, eps=1e-13)
        assert rel(ar, ak) <= 1e-9 and abs(br - bk) <= 1e-9
    # RBF translation invariance
    a3, b3, _, _ = oracle.train(X + 3.5, y, oracle.RBF, 0.2, eps=1e-13)
    assert rel(a3, a0) <= 1e-9 and abs(b3 - b0) <= 1e-9


def test_training_rows_reproduce_labels():
    """Q alpha + b 1 = y (the first block row of Eq. 11)."""
    rng = np.random.default_rng(31)
    X, y = synth.random_small(rng, 60, 4)
    alpha, b, _, _ = oracle.train(X, y, oracle.POLYNOMIAL, 0.5, 2, 1.0, C=2.0, eps=1e-13)
    Q = gram_lib(X, X, oracle.POLYNOMIAL, 0.5, 2, 1.0) + np.eye(60) / 2.0
    assert np.abs(Q @ alpha + b - y).max() <= 1e-9


def test_predict_matches_library_decision_values():
    rng = np.random.default_rng(41)
    X, y = synth.random_small(rng, 70, 6)
    Z = rng.standard_normal((33, 6))
    alpha = rng.standard_normal(70)
    for k in KERNELS:
        f, lab = oracle.predict(X, alpha, 0.3, Z, k, 0.15, 3, 0.4)
        ref = gram_lib(Z, X, k, 0.15, 3, 0.4) @ alpha + 0.3
        assert rel(f, ref) <= 1e-13
        assert np.array_equal(lab, np.where(f >= 0, 1, -1))


def test_generator_recipe_hash():
    """synth.planes at C0 reproduces the SURVEY §8(d) measured hash (sklearn 1.9 / numpy 2.3)."""
    cfg = synth.configs()["C0"]
    X, y, Z, yz = synth.planes(cfg.m, cfg.d, cfg.n_test, seed=synth.SEED_BASE)
    assert synth.sha16(np.vstack([X, Z])) == "5885be14d48a0e4f"
    assert set(np.unique(y)) == {-1.0, 1.0}


def test_c0_reference_values():
    """C0 reference values quoted in SURVEY §8(d): iterations ~20, b ~ -0.2180755, KKT parity."""
    cfg = synth.configs()["C0"]
    X, y, Z, yz = synth.config_data(cfg)
    alpha, b, it, st = oracle.train(X, y, cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C, cfg.eps)
    a_ref, b_ref = kkt_solve(X, y, cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C)
    assert st == oracle.OK and 17 <= it <= 25
    assert rel(alpha, a_ref) <= 1e-9 and abs(b - b_ref) <= 1e-9
    assert abs(b - (-0.218075516159)) <= 1e-9


# ---------------------------------------------------------------- CG options: x0 = ONES, residual replacement
# (these branches of oracle_cg / oracle_train were only compared with the GPU.)  The
# KKT solution of Eq. 11 is unique, so every start vector and replacement period must reach it; the
# traces pin WHAT the branches compute (r0 = rhs - Q~ x0, the replaced residual is the true one).
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("x0", [0, 1])
@pytest.mark.parametrize("R", [0, 1, 3, 5])
def test_train_options_match_dense_kkt_lu(kernel, x0, R):
    rng = np.random.default_rng(300 + 10 * kernel + 2 * R + x0)
    for trial in range(3):
        m, d = int(rng.integers(8, 80)), int(rng.integers(2, 9))
        X, y = synth.random_small(rng, m, d)
        gam, deg, r = 1.0 / d, int(rng.integers(1, 4)), float(rng.uniform(0, 1))
        a_ref, b_ref = kkt_solve(X, y, kernel, gam, deg, r, 1.0)
        # imax = 10 m: in floating point CG may need more than m - 1 iterations to reach 1e-12
        alpha, b, it, st = oracle.train(X, y, kernel, gam, deg, r, 1.0, eps=1e-12, x0=x0, replace_every=R,
                                        imax=10 * m)
        assert st == oracle.OK
        assert rel(alpha, a_ref) <= 1e-9, (m, d, trial)
        assert abs(b - b_ref) <= 1e-8 * max(abs(b_ref), np.abs(a_ref).max())


def test_cg_start_vector_residual():
    """r0 = rhs - A x0 (Shewchuk B2 line 2): A = diag(2, 3, 4), rhs = (2, 6, 12), x0 = 1 gives
    r0 = (0, 3, 8), |r0| = sqrt(73); x0 = the exact solution (1, 2, 3) gives r0 = 0 and no iteration."""
    A = np.diag([2.0, 3.0, 4.0])
    rhs = np.array([2.0, 6.0, 12.0])
    x, it, st, tr = oracle.cg(A, rhs, eps=1e-14, x0=np.ones(3), trace=True)
    assert tr[0] == math.sqrt(73.0)
    assert np.allclose(x, [1.0, 2.0, 3.0], rtol=0, atol=1e-14) and st == oracle.OK
    x, it, st = oracle.cg(A, rhs, eps=1e-14, x0=np.array([1.0, 2.0, 3.0]))
    assert it == 0 and np.array_equal(x, [1.0, 2.0, 3.0])


def test_train_x0_ones_first_residual():
    """oracle.train(x0=1): delta_0 = |rhs - Q~ 1|^2 with rhs = y_bar - y_m 1 (Eq. 14) -- checked through
    the trace of the same system, Q~ built independently as B^T Q B (Eq. 13)."""
    rng = np.random.default_rng(41)
    X, y = synth.random_small(rng, 30, 4)
    m = X.shape[0]
    Q = gram_lib(X, X, oracle.RBF, 0.25, 1, 0.0) + np.eye(m)
    B = np.vstack([np.eye(m - 1), -np.ones((1, m - 1))])
    Qt = B.T @ Q @ B
    rhs = y[:-1] - y[-1]
    _, _, _, tr = oracle.cg(oracle.qtilde(X, oracle.RBF, 0.25), rhs, eps=1e-12, x0=np.ones(m - 1), trace=True)
    assert abs(tr[0] - np.linalg.norm(rhs - Qt @ np.ones(m - 1))) <= 1e-12 * tr[0]
    a_ref, b_ref = kkt_solve(X, y, oracle.RBF, 0.25, 1, 0.0, 1.0)
    alpha, b, it, st = oracle.train(X, y, oracle.RBF, 0.25, eps=1e-12, x0=1)
    assert st == oracle.OK and rel(alpha, a_ref) <= 1e-9


def _ill_conditioned(n=120, cond=1e10, seed=17):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (U * np.geomspace(1.0, cond, n)) @ U.T
    return 0.5 * (A + A.T), rng.standard_normal(n)


@pytest.mark.parametrize("R", [3, 5, 7])
def test_residual_replacement_period_and_value(R):
    """Residual replacement (Shewchuk B2, option R): the trace equals the pure recurrence's bit for bit
    up to iteration R (no replacement before i = R), departs from it at the first replacement, and at
    every replacement iteration (i - 1) % R == 0, i > 1, the recorded |r_i| is the TRUE residual
    |rhs - A x_i| (x_i from a run capped at imax = i) to rounding."""
    A, rhs = _ill_conditioned()
    imax = 40
    _, _, _, tr0 = oracle.cg(A, rhs, eps=1e-30, imax=imax, replace_every=0, trace=True)
    x, it, st, tr = oracle.cg(A, rhs, eps=1e-30, imax=imax, replace_every=R, trace=True)
    assert it == imax
    assert np.array_equal(tr[:R + 1], tr0[:R + 1]) and tr[R + 1] != tr0[R + 1]
    for i in range(R + 1, it + 1, R):
        xi, iti, _ = oracle.cg(A, rhs, eps=1e-30, imax=i, replace_every=R)
        assert iti == i
        assert abs(tr[i] - np.linalg.norm(rhs - A @ xi)) <= 1e-12 * np.linalg.norm(rhs)


def test_stagnation_guard():
    """Stagnation guard (R-20): with replacement on and an unreachable
    eps, the oracle stops with W_NOT_CONVERGED W = 2 max(R, 50) iterations after the last 4x drop of
    delta, long before imax, and its x still solves the system to ~kappa u; without replacement (R = 0) the guard is
    off and the loop runs to imax."""
    A, rhs = _ill_conditioned(cond=1e4)
    ref = scipy.linalg.cho_solve(scipy.linalg.cho_factor(A), rhs)
    R, imax = 5, 3000
    x, it, st, tr = oracle.cg(A, rhs, eps=1e-17, imax=imax, replace_every=R, trace=True)
    assert st == oracle.W_NOT_CONVERGED and it < imax
    # the exit is the rule's first firing: the best delta (last 4x drop) is exactly 2R iterations old
    d = tr ** 2
    best, ib = d[0], 0
    fired = None
    for i in range(1, it + 1):
        if d[i] < 0.25 * best:
            best, ib = d[i], i
        elif i - ib >= 2 * max(R, 50):
            fired = i
            break
    assert fired == it
    assert rel(x, ref) <= 1e4 * 1e-15 * 10  # at the attainable accuracy ~ kappa u
    x2, it2, st2 = oracle.cg(A, rhs, eps=1e-17, imax=150, replace_every=0)
    assert it2 == 150 and st2 == oracle.W_NOT_CONVERGED
