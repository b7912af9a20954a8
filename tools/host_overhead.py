"""Host-side overhead of one bench step (C1): the Python wrapper vs the raw C-ABI call vs the library's
own wall time (stats.t_total, taken before the call's destructors), and the gap a b.item() adds.
    python tools/host_overhead.py [C1] [reps]"""
import ctypes as ct
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
from paper_2202_12674_b200 import binding as B  # noqa: E402
import synth  # noqa: E402

cfg = synth.configs()[sys.argv[1] if len(sys.argv) > 1 else "C1"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
X, y, Z, _ = synth.config_data(cfg)
tX, ty, tZ = (torch.from_numpy(a).cuda() for a in (X, y, Z))
kw = dict(gamma=cfg.gamma, degree=cfg.degree, coef0=cfg.coef0)
L = pl.load()
m, d = tX.shape
for _ in range(3):
    a, b, _, _ = pl.plssvm_train_ex(tX, ty, cfg.kernel, C=cfg.C, eps=cfg.eps,
                                    opts=pl.options(mode=pl.MODE_IMPLICIT, cg_loop=pl.CG_BATCHED), **kw)
torch.cuda.synchronize()
for r in range(reps):
    o = pl.options(mode=pl.MODE_IMPLICIT, cg_loop=pl.CG_BATCHED)
    t0 = time.perf_counter()
    a, b, st, s = pl.plssvm_train_ex(tX, ty, cfg.kernel, C=cfg.C, eps=cfg.eps, opts=o, **kw)
    t1 = time.perf_counter()
    bb = float(b.item())
    t2 = time.perf_counter()
    # the raw C call with pre-built arguments (same options, device pointers, outputs)
    o2 = pl.options(mode=pl.MODE_IMPLICIT, cg_loop=pl.CG_BATCHED)
    B._device_opts(o2, [tX])
    stats = B.plssvm_stats_t()
    args = (tX.data_ptr(), ty.data_ptr(), m, d, B._dtype_code(tX), cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C,
            cfg.eps, ct.byref(o2), a.data_ptr(), b.data_ptr(), ct.byref(stats))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    L.plssvm_train_ex(*args)
    t4 = time.perf_counter()
    f, lab, _ = pl.plssvm_predict_ex(tX, a, bb, tZ, cfg.kernel, opts=pl.options(mode=pl.MODE_IMPLICIT), **kw)
    t5 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"rep {r}: wrapper train {1e3*(t1-t0):.3f} ms (lib t_total {1e3*s.t_total:.3f}: wrapper + destructors "
          f"{1e3*(t1-t0-s.t_total):.3f}) | b.item {1e3*(t2-t1):.3f} | raw C call {1e3*(t4-t3):.3f} (lib t_total "
          f"{1e3*stats.t_total:.3f}: after t_total {1e3*(t4-t3-stats.t_total):.3f}) | predict wrapper {1e3*(t5-t4):.3f}",
          flush=True)
