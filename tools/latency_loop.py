"""CG-loop issue latency: BATCHED host loop vs one CUDA graph (WHILE node), per config shape.
Prints CG it/s (iterations / t_cg) for each, device-resident inputs, after warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

cases = [("C0 256x16 linear implicit", 256, 16, pl.LINEAR, pl.MODE_IMPLICIT),
         ("2^12x2^8 rbf implicit", 4096, 256, pl.RBF, pl.MODE_IMPLICIT),
         ("C1 2^14x2^10 rbf cached", 16384, 1024, pl.RBF, pl.MODE_CACHED),
         ("2^14x2^10 linear lowrank", 16384, 1024, pl.LINEAR, pl.MODE_LOWRANK)]
for name, m, d, kern, mode in cases:
    X, y, _, _ = synth.planes(m, d, 16, seed=1)
    tX, ty = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    res = {}
    for loop in (pl.CG_BATCHED, pl.CG_GRAPH):
        best = None
        for rep in range(12):
            a, b, st, s = pl.plssvm_train_ex(tX, ty, kern, 1.0 / d, C=1.0, eps=1e-10,
                                             opts=pl.options(mode=mode, cg_loop=loop))
            if rep >= 2 and (best is None or s.t_cg < best.t_cg):
                best = s
        res[loop] = best
    sb, sg = res[pl.CG_BATCHED], res[pl.CG_GRAPH]
    print(f"{name}: it {sb.iterations}/{sg.iterations}  batched {sb.iterations / sb.t_cg:9.0f} CG it/s "
          f"(t_cg {sb.t_cg*1e3:.3f} ms, train {sb.t_total*1e3:.3f} ms)   graph {sg.iterations / sg.t_cg:9.0f} CG it/s "
          f"(t_cg {sg.t_cg*1e3:.3f} ms, train {sg.t_total*1e3:.3f} ms)", flush=True)
