"""NEXT-3: the paper's epsilon sweep (Fig. 3) on its shape, 2^15 x 2^12 linear fp64:
CG iterations, training time and training accuracy per eps, for x0 = zeros (default) and x0 = ones
(the start that reproduces the paper's flat-then-jump curve).

    python tools/eps_sweep.py [--m 32768 --d 4096] [--out profiles/r01_eps_sweep.jsonl]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2**15)
ap.add_argument("--d", type=int, default=2**12)
ap.add_argument("--mode", default="cached")
ap.add_argument("--out", default="")
a = ap.parse_args()
X, y, _, _ = synth.planes(a.m, a.d, 0, seed=synth.SEED_BASE + 100)
tX, ty = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
mode = {"cached": pl.MODE_CACHED, "implicit": pl.MODE_IMPLICIT, "lowrank": pl.MODE_LOWRANK}[a.mode]
out = open(a.out, "w") if a.out else None
for x0 in (0, 1):
    for e in range(1, 16):
        eps = 10.0 ** -e
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        alpha, b, st, s = pl.plssvm_train_ex(tX, ty, pl.LINEAR, C=1.0, eps=eps, opts=pl.options(mode=mode, x0=x0))
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        f, lab, _ = pl.plssvm_predict_ex(tX, alpha, float(b.item()), tX, pl.LINEAR)
        acc = float((lab.cpu().numpy() == y.astype(np.int32)).mean())
        row = {"x0": "ones" if x0 else "zeros", "eps": eps, "status": st, "iterations": s.iterations,
               "train_s": t, "cg_s": s.t_cg, "train_accuracy": acc, "rel_residual": s.rel_residual}
        print(json.dumps(row), flush=True)
        if out:
            out.write(json.dumps(row) + "\n")
