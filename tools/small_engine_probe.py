"""Small problems: CG it/s of the fp64 engines (Ozaki persistent 2-SM kernel vs DMMA tiles) and of
the fp32 engines, per size -- the fixed cost of the persistent int8 kernel vs its throughput."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

for m, d in [(256, 16), (512, 64), (1024, 128), (2048, 256), (4096, 256), (8192, 512)]:
    X, y, _, _ = synth.planes(m, d, 16, seed=1)
    row = []
    for dt, engs in ((np.float64, [("ozaki", dict(fp64_engine=1)), ("dmma", dict(fp64_engine=2))]),
                     (np.float32, [("int8", dict(fp32_engine=2)), ("tf32x3", dict(fp32_engine=0))])):
        tX, ty = torch.from_numpy(X.astype(dt)).cuda(), torch.from_numpy(y.astype(dt)).cuda()
        for name, kw in engs:
            best = None
            for rep in range(8):
                a, b, st, s = pl.plssvm_train_ex(tX, ty, pl.RBF, 1.0 / d, C=1.0, eps=1e-10 if dt == np.float64 else 1e-6,
                                                 opts=pl.options(mode=pl.MODE_IMPLICIT, cg_loop=pl.CG_BATCHED, **kw))
                if rep >= 2 and (best is None or s.t_cg < best.t_cg):
                    best = s
            row.append(f"{name} {best.iterations / best.t_cg:8.0f} it/s (mv {best.t_matvec / best.iterations * 1e6:6.1f} us)")
    print(f"{m:5d} x {d:4d}: " + " | ".join(row), flush=True)
