"""Cycle accounting of k_tile_ozaki (the experiment build: PLSSVM_EXPERIMENT_LIB=1, the .so built with
-DPLSSVM_OZ_EXPERIMENTS): where the MMA thread, the TMA thread and the epilogue spend their cycles in
one Q~p product.  Usage: PLSSVM_EXPERIMENT_LIB=1 python tools/oz_profile.py [C1|C2|C3|C4] [repeats]"""
import ctypes as ct
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
assert os.environ.get("PLSSVM_EXPERIMENT_LIB") == "1", "run with PLSSVM_EXPERIMENT_LIB=1"
import numpy as np  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
from paper_2202_12674_b200 import _build  # noqa: E402
import synth  # noqa: E402

_build.build(variant="exp")
L = pl.load()
L.plssvm_exp_oz_profile.argtypes = [ct.c_void_p, ct.c_int]
cfg = synth.configs()[sys.argv[1] if len(sys.argv) > 1 else "C1"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
X, y, _, _ = synth.config_data(cfg, n_test=0)
p = np.random.default_rng(1).standard_normal(cfg.m - 1).astype(X.dtype)
o = pl.options(mode=pl.MODE_IMPLICIT)
pl.plssvm_qtilde_matvec(X, p, cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C, repeats=1, opts=o)  # warm-up
buf = np.zeros((160, 8), dtype=np.uint64)
L.plssvm_exp_oz_profile(None, 1)
_, (tmean, tmin, _) = pl.plssvm_qtilde_matvec(X, p, cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C, repeats=reps,
                                              opts=o)
L.plssvm_exp_oz_profile(buf.ctypes.data, 0)
lead = buf[0:148:2].astype(np.float64)  # leader CTAs (the MMA issuer lives there)
both = buf[0:148].astype(np.float64)
loop = lead[:, 2].mean()
names = ["MMA waits for the epilogue drain (tempty)", "MMA waits for TMA stages (full)", "MMA loop total",
         "TMA waits for free stages (empty)", "epilogue waits for accumulators (tfull)", "epilogue pass-0 drain",
         "epilogue pass-1 drain", "epilogue fp64 work after release"]
print(f"{cfg.name}: {reps} products, mean {tmean * 1e3:.3f} ms, min {tmin * 1e3:.3f} ms; per leader CTA "
      f"MMA-loop cycles {loop:.4g} ({loop / reps:.4g} per product)")
for k, n in enumerate(names):
    v = lead[:, k].mean() if k < 3 else both[:, k].mean()
    print(f"  [{k}] {n:45s} {v / reps:12.4g} cycles/product  {100 * v / loop:6.2f} % of the MMA loop")
