import sys; sys.path.insert(0, ".")
import numpy as np, oracle, paper_2202_12674_b200 as pl
rng = np.random.default_rng(77)
m, d = 600, 40
X = rng.standard_normal((m, d)).astype(np.float32)
X[10] = 0.0; X[11] = X[12]
X[20] *= np.float32(1e15); X[21] *= np.float32(1e-15)
p = rng.standard_normal(m - 1).astype(np.float32)
Qt = oracle.qtilde(X.astype(np.float64), 0, 1.0, 3, 0.0, 1.0)
ref = Qt @ p.astype(np.float64); scale = np.abs(Qt) @ np.abs(p.astype(np.float64))
for eng in (2, 0, 1):
    for mode in (1, 2):
        out, _ = pl.plssvm_qtilde_matvec(X, p, 0, 1.0, 3, 0.0, 1.0, opts=pl.options(mode=mode, fp32_engine=eng))
        e = np.abs(out.astype(np.float64) - ref) / scale
        i = int(np.argmax(e)); print("eng", eng, "mode", mode, "max", e.max(), "row", i, "median", np.median(e), flush=True)
# same without the huge row
X2 = X.copy(); X2[20] /= np.float32(1e15)
Qt = oracle.qtilde(X2.astype(np.float64), 0, 1.0, 3, 0.0, 1.0)
ref = Qt @ p.astype(np.float64); scale = np.abs(Qt) @ np.abs(p.astype(np.float64))
for eng in (2, 0):
    out, _ = pl.plssvm_qtilde_matvec(X2, p, 0, 1.0, 3, 0.0, 1.0, opts=pl.options(mode=1, fp32_engine=eng))
    e = np.abs(out.astype(np.float64) - ref) / scale
    print("no huge row: eng", eng, "max", e.max(), "row", int(np.argmax(e)), flush=True)
