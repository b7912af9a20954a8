"""A/B timing of two library builds in bench.py's loop (sustained clocks): K bench steps (train on
HBM-resident C1 + predict), mean product time from the library's per-launch events, step time
from CUDA events.  Run alternately per build:  PLSSVM_LIB_PATH=<so> python tools/ab_step.py [C1] [K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

cfg = synth.configs()[sys.argv[1] if len(sys.argv) > 1 else "C1"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
X, y, Z, _ = synth.config_data(cfg)
tX, ty, tZ = (torch.from_numpy(a).cuda() for a in (X, y, Z))
kw = dict(gamma=cfg.gamma, degree=cfg.degree, coef0=cfg.coef0)


def step():
    o = pl.options(mode=pl.MODE_IMPLICIT, cg_loop=pl.CG_BATCHED)
    alpha, b, st, s = pl.plssvm_train_ex(tX, ty, cfg.kernel, C=cfg.C, eps=cfg.eps, opts=o, **kw)
    f, lab, (tk, nl) = pl.plssvm_predict_ex(tX, alpha, float(b.item()), tZ, cfg.kernel, opts=o, **kw)
    return s, tk


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = [step() for _ in range(K)]
e1.record()
torch.cuda.synchronize()
its = sum(s.iterations for s, _ in res)
mv = sum(s.t_matvec for s, _ in res) / its
pr = sum(t for _, t in res) / K
ms = e0.elapsed_time(e1) / K
print(f"{os.path.basename(pl.binding.lib_path())}: product {mv*1e3:.4f} ms  predict {pr*1e3:.4f} ms"
      f"  step {ms:.3f} ms  CG it/s {its / (K * ms / 1e3):.1f}", flush=True)
