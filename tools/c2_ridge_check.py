"""C2 (2^16 x 2^12 linear fp64) trained on the GPU vs the exact solution of Eq. 11 in closed form:
for the linear kernel LS-SVM is ridge regression with an unpenalised intercept,
w = (Xc^T Xc + I/C)^-1 Xc^T yc, b = ybar - xbar.w, alpha = C (y - X w - b).  Prints the relative
alpha / b errors of each mode and CG variant (the north_star bar: 1e-7)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

cfg = synth.configs()["C2"]
X, y, _, _ = synth.config_data(cfg, n_test=0)
C = cfg.C
xb, yb = X.mean(0), y.mean()
Xc, yc = X - xb, y - yb
w = np.linalg.solve(Xc.T @ Xc + np.eye(X.shape[1]) / C, Xc.T @ yc)
b_ex = yb - xb @ w
a_ex = C * (y - X @ w - b_ex)
print(f"exact: sum(alpha) = {a_ex.sum():.3e}, |alpha|_inf = {np.abs(a_ex).max():.4f}, b = {b_ex:.10f}", flush=True)
for name, opts in [("cached", pl.options(mode=pl.MODE_CACHED)), ("implicit", pl.options(mode=pl.MODE_IMPLICIT)),
                   ("lowrank", pl.options(mode=pl.MODE_LOWRANK)),
                   ("cached, single-reduction CG", pl.options(mode=pl.MODE_CACHED, cg_variant=pl.CG_SINGLE_REDUCTION))]:
    a, b, st, s = pl.plssvm_train_ex(X, y, cfg.kernel, cfg.gamma, C=cfg.C, eps=cfg.eps, opts=opts)
    ea = np.linalg.norm(a - a_ex) / np.linalg.norm(a_ex)
    eb = abs(b - b_ex) / max(abs(b_ex), np.abs(a_ex).max())
    print(f"{name:30s} status {st} iterations {s.iterations:3d} recurrence residual {s.rel_residual:.2e}  "
          f"|da|/|a| = {ea:.2e}  db = {eb:.2e}", flush=True)
