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
# what fp32 arithmetic itself allows on this input (host emulation, no GPU): the kernel values rounded
# ONCE to fp32, Eq. 16 and the product in fp64 -- already 3.4e-5 of |Q~||p| (row 539: k = 7.080e15 and
# q_20 = 7.083e15 cancel to Q~ = -2.8e12), i.e. the |Q~||p| bar is not fp32-fair here (R-19)
X = X2.copy(); X[20] *= np.float32(1e15)
Xd = X.astype(np.float64); K1 = (Xd @ Xd.T).astype(np.float32).astype(np.float64)
Qt = oracle.qtilde(Xd, 0, 1.0, 3, 0.0, 1.0); ref = Qt @ p.astype(np.float64)
scale = np.abs(Qt) @ np.abs(p.astype(np.float64))
q1 = K1[:-1, -1]; Qd = K1[:-1, :-1] + np.eye(m - 1) - q1[None, :] - q1[:, None] + K1[-1, -1] + 1
e = np.abs(Qd @ p.astype(np.float64) - ref) / scale
print("fp32-rounded kernel values, rest fp64: max", e.max(), "row", int(np.argmax(e)), flush=True)
