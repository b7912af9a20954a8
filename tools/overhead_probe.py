"""Host / device overhead of one bench step (C1, bench.py's options: implicit, batched CG loop,
torch's current stream): per step, CUDA-event times of the train call and the predict call on the
stream, the library's own phase times, the products' event sum, and the host wall times.
    python tools/overhead_probe.py [C1] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

cfg = synth.configs()[sys.argv[1] if len(sys.argv) > 1 else "C1"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
X, y, Z, yz = synth.config_data(cfg)
tX, ty, tZ = (torch.from_numpy(a).cuda() for a in (X, y, Z))
kw = dict(gamma=cfg.gamma, degree=cfg.degree, coef0=cfg.coef0)


def opts():
    return pl.options(mode=pl.MODE_IMPLICIT, cg_loop=pl.CG_BATCHED)


ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for rep in range(steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record()
    alpha, b, st, s = pl.plssvm_train_ex(tX, ty, cfg.kernel, C=cfg.C, eps=cfg.eps, opts=opts(), **kw)
    ev[1].record()
    t1 = time.perf_counter()
    bb = float(b.item())
    f, lab, (tk, nl) = pl.plssvm_predict_ex(tX, alpha, bb, tZ, cfg.kernel, opts=opts(), **kw)
    ev[2].record()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    dtr, dpr = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    mv = 1e3 * s.t_matvec
    print(f"step {rep}: device train {dtr:.3f} ms (lib t_total {1e3*s.t_total:.3f}: h2d {1e3*s.t_h2d:.3f} "
          f"tr {1e3*s.t_transform:.3f} q {1e3*s.t_q:.3f} alloc {1e3*s.t_alloc:.3f} cg {1e3*s.t_cg:.3f} "
          f"bias {1e3*s.t_bias_d2h:.3f}; {s.iterations} it, products {mv:.3f} = {mv/max(1,s.iterations):.3f}/it, "
          f"cg - products {1e3*s.t_cg - mv:.3f}) | device predict {dpr:.3f} (kernel {1e3*tk:.3f}) | "
          f"host train {1e3*(t1-t0):.3f} step {1e3*(t3-t0):.3f} | non-product {dtr + dpr - mv - 1e3*tk:.3f} ms")
