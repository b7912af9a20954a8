"""Where does the end-to-end (host buffers) step spend its time?  C1 train + predict through the
public API on pinned numpy buffers: wall time per call and the library's device-event phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

cfg = synth.configs()[sys.argv[1] if len(sys.argv) > 1 else "C1"]
X, y, Z, _ = synth.config_data(cfg)
hX = torch.from_numpy(X).pin_memory().numpy()
hy = torch.from_numpy(y).pin_memory().numpy()
hZ = torch.from_numpy(Z).pin_memory().numpy()
kw = dict(gamma=cfg.gamma, degree=cfg.degree, coef0=cfg.coef0)
o = pl.options(mode=pl.MODE_IMPLICIT)
for it in range(4):
    t0 = time.perf_counter()
    a, b, st, s = pl.plssvm_train_ex(hX, hy, cfg.kernel, C=cfg.C, eps=cfg.eps, opts=o, **kw)
    t1 = time.perf_counter()
    f, lab, (tk, nl) = pl.plssvm_predict_ex(hX, a, b, hZ, cfg.kernel, opts=o, **kw)
    t2 = time.perf_counter()
    print(f"train wall {1e3*(t1-t0):7.2f} ms (lib t_total {1e3*s.t_total:7.2f}: h2d {1e3*s.t_h2d:6.2f} transform "
          f"{1e3*s.t_transform:6.2f} q {1e3*s.t_q:5.2f} alloc {1e3*s.t_alloc:5.2f} cg {1e3*s.t_cg:7.2f} "
          f"bias/d2h {1e3*s.t_bias_d2h:5.2f})  predict wall {1e3*(t2-t1):6.2f} ms (kernel {1e3*tk:6.2f})")
