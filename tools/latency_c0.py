"""C0 (256 x 16 linear) training latency, repeated in one process (GPU clocks ramp up)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

cfg = synth.configs()["C0"]
X, y, Z, yz = synth.config_data(cfg)
tX, ty = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a, b, st, s = pl.plssvm_train_ex(tX, ty, cfg.kernel, cfg.gamma, C=cfg.C, eps=cfg.eps,
                                     opts=pl.options(mode=pl.MODE_IMPLICIT, cg_loop=int(os.environ.get("CG_LOOP", "0"))))
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    if rep % 5 == 4:
        print(f"rep {rep}: train {t*1e3:.3f} ms, cg {s.t_cg*1e3:.3f} ms, {s.iterations} it -> "
              f"{s.iterations / s.t_cg:.0f} CG it/s, matvec {s.t_matvec / s.iterations * 1e6:.1f} us, "
              f"launches {s.gpu_launches}")
