"""Host overhead of one bench step (C1): wall time of train / predict vs the device-event phases."""
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
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    alpha, b, st, s = pl.plssvm_train_ex(tX, ty, cfg.kernel, C=cfg.C, eps=cfg.eps, **kw)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    bb = float(b.item())
    t2 = time.perf_counter()
    f, lab, (tk, nl) = pl.plssvm_predict_ex(tX, alpha, bb, tZ, cfg.kernel, **kw)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    dev = s.t_h2d + s.t_transform + s.t_q + s.t_alloc + s.t_precompute + s.t_cg + s.t_bias_d2h
    print(f"train wall {1e3*(t1-t0):.3f} ms (lib t_total {1e3*s.t_total:.3f}, device phases {1e3*dev:.3f}: "
          f"h2d {1e3*s.t_h2d:.3f} tr {1e3*s.t_transform:.3f} q {1e3*s.t_q:.3f} alloc {1e3*s.t_alloc:.3f} "
          f"cg {1e3*s.t_cg:.3f} bias {1e3*s.t_bias_d2h:.3f}) | item {1e3*(t2-t1):.3f} | predict wall {1e3*(t3-t2):.3f} "
          f"(kernel {1e3*tk:.3f})")
