"""Predict timing at a config (kernel time from the C ABI and wall time), device-resident inputs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

cfg = synth.configs()[sys.argv[1] if len(sys.argv) > 1 else "C1"]
X, y, Z, yz = synth.config_data(cfg)
tX, ty, tZ = (torch.from_numpy(a).cuda() for a in (X, y, Z))
kw = dict(gamma=cfg.gamma, degree=cfg.degree, coef0=cfg.coef0)
alpha, b, st, s = pl.plssvm_train_ex(tX, ty, cfg.kernel, C=cfg.C, eps=cfg.eps, **kw)
for rep in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f, lab, (tk, nl) = pl.plssvm_predict_ex(tX, alpha, float(b.item()), tZ, cfg.kernel, **kw)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    fl = 2.0 * cfg.m * Z.shape[0] * cfg.d
    print(f"{cfg.name} predict n={Z.shape[0]}: kernel {tk*1e3:.3f} ms ({fl/tk/1e12:.1f} TFLOP/s fp64-equiv), "
          f"wall {1e3*(t1-t0):.3f} ms, launches {nl}")
