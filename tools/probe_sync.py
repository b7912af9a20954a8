import sys; sys.path.insert(0, ".")
import numpy as np, paper_2202_12674_b200 as pl, synth
X, y, _, _ = synth.planes(256, 16, 16, seed=7)
for mode, eng in ((2, 0), (1, 2), (1, 1)):
    try:
        a, b, st, s = pl.plssvm_train_ex(X, y, 0, 1/16, 3, 0.0, 1.0, 1e-10, opts=pl.options(mode=mode, cg_loop=2, fp64_engine=eng))
        print("mode", mode, "engine", eng, "graph ok", s.iterations, flush=True)
    except Exception as e:
        print("mode", mode, "engine", eng, "graph fail", e, flush=True)
        break
