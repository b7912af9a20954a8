"""Run the Q~p product alone on a BASELINE config (for ncu captures and quick timing).

    python tools/run_matvec.py --config C1 --mode implicit --repeats 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C1")
ap.add_argument("--mode", default="implicit")
ap.add_argument("--repeats", type=int, default=3)
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--d", type=int, default=0)
ap.add_argument("--kernel", type=int, default=-1)
ap.add_argument("--fp32-engine", type=int, default=0)
ap.add_argument("--fp64-engine", type=int, default=0, help="0 AUTO, 1 OZAKI, 2 DMMA")
ap.add_argument("--synth", action="store_true", help="use the config's seeded make_classification data (as bench.py) instead of N(0,1)")
ap.add_argument("--compare", action="store_true", help="also run the DMMA fp64 engine (OZAKI if --fp64-engine 2) and compare")
a = ap.parse_args()
cfg = synth.configs()[a.config]
m, d = a.m or cfg.m, a.d or cfg.d
dt = np.float32 if cfg.dtype == "f32" else np.float64
rng = np.random.default_rng(0)
X = rng.standard_normal((m, d)).astype(dt)
if a.synth:
    X = synth.config_data(cfg)[0].astype(dt)
p = rng.standard_normal(m - 1).astype(dt)
mode = {"implicit": pl.MODE_IMPLICIT, "cached": pl.MODE_CACHED, "lowrank": pl.MODE_LOWRANK}[a.mode]
kern = cfg.kernel if a.kernel < 0 else a.kernel
out, t = pl.plssvm_qtilde_matvec(X, p, kern, 1.0 / d, cfg.degree, cfg.coef0, cfg.C, repeats=a.repeats,
                                 opts=pl.options(mode=mode, fp32_engine=a.fp32_engine, fp64_engine=a.fp64_engine))
m1 = m - 1
fl = 2.0 * d * m1 * (m1 + 1) / 2
s = np.dtype(dt).itemsize
print(f"{a.config} m={m} d={d} kernel={kern} mode={a.mode}: mean {t[0]*1e3:.3f} ms min {t[1]*1e3:.3f} ms precompute {t[2]*1e3:.3f} ms"
      f" -> {fl/t[1]/1e12:.2f} TFLOP/s (implicit-equivalent), cached stream {m1*m1*s/t[1]/1e9:.1f} GB/s")
if a.compare and dt == np.float64:
    ref, t2 = pl.plssvm_qtilde_matvec(X, p, kern, 1.0 / d, cfg.degree, cfg.coef0, cfg.C, repeats=a.repeats,
                                      opts=pl.options(mode=mode, fp64_engine=pl.FP64_OZAKI if a.fp64_engine == pl.FP64_DMMA else pl.FP64_DMMA))
    err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    print(f"  other fp64 engine: min {t2[1]*1e3:.3f} ms ({fl/t2[1]/1e12:.2f} TFLOP/s); rel diff {err:.3e}, max abs {np.abs(out-ref).max():.3e}")
