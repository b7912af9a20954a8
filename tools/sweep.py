"""Per-config measurement table (BASELINE metric: 'every config reports CG iterations/s and
FLOP/s or GB/s fraction of peak'): one full training per config on one GPU, on the config's
synthetic data, with the mode the config names.  Writes one JSON object per line.

    python tools/sweep.py [--configs C0,C1,C2,C3,C4] [--out profiles/rNN_sweep.jsonl]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

FP64_PEAK = 148 * 64 * 2 * 1.965e9 / 1e12
def tf32x3_peak():
    try:
        bf16 = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except (OSError, KeyError, ValueError):
        bf16 = 1590.0
    return bf16 * (1.1 / 2.25) / 3.0


FP32_PEAK = tf32x3_peak()
try:  # int8 dense = 2 x the measured sustained bf16 dense rate (bench.py int8_peak_tops)
    INT8_PEAK = 2.0 * json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"]
except (OSError, KeyError, ValueError):
    INT8_PEAK = 2784.4


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        return 6650.0


# (mode, fp64 engine) per config; engine "auto" = the default (Ozaki on these data), "dmma" = fp64
# tensor cores for comparison
MODES = {"C0": [("implicit", "auto")], "C1": [("implicit", "auto"), ("implicit", "dmma"), ("cached", "auto")],
         "C2": [("cached", "auto"), ("implicit", "auto"), ("lowrank", "auto")],
         "C3": [("cached", "auto"), ("implicit", "auto")],
         "C4": [("cached", "auto"), ("implicit", "auto")]}
ENGINES = {"auto": pl.FP64_AUTO, "dmma": pl.FP64_DMMA}


def run(cfg, mode, engine="auto", repeat=2):
    X, y, Z, yz = synth.config_data(cfg)
    dev = torch.device("cuda", 0)
    tX, ty, tZ = (torch.from_numpy(a).to(dev) for a in (X, y, Z))
    kw = dict(gamma=cfg.gamma, degree=cfg.degree, coef0=cfg.coef0)
    md = {"implicit": pl.MODE_IMPLICIT, "cached": pl.MODE_CACHED, "lowrank": pl.MODE_LOWRANK}[mode]
    runs = []
    for _ in range(repeat):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        alpha, b, st, s = pl.plssvm_train_ex(tX, ty, cfg.kernel, C=cfg.C, eps=cfg.eps, opts=pl.options(mode=md, fp64_engine=ENGINES[engine], cg_loop=pl.CG_BATCHED), **kw)
        torch.cuda.synchronize()
        runs.append((time.perf_counter() - t0, s, alpha, b, st))
    # the paper's protocol: median of the repeats plus the coefficient of
    # variation; the first run of a config (cold memory pool) is dropped when there are >= 3
    timed = runs[1:] if len(runs) >= 3 else runs
    tts = np.array([r[0] for r in timed])
    its = np.array([r[1].iterations / r[1].t_cg for r in timed])
    med = int(np.argsort(tts)[len(tts) // 2])
    tt, s, alpha, b, st = timed[med]
    f, lab, (tk, _) = pl.plssvm_predict_ex(tX, alpha, float(b.item()), tZ, cfg.kernel,
                                           opts=pl.options(fp64_engine=ENGINES[engine]), **kw)
    acc = float((lab.cpu().numpy() == yz.astype(np.int32)).mean()) if len(yz) else None
    m1 = cfg.m - 1
    fl = 2.0 * cfg.d * m1 * (m1 + 1) / 2
    peak_f = FP64_PEAK if cfg.dtype == "f64" else FP32_PEAK
    mv = s.t_matvec / max(1, s.iterations)
    row = {"config": cfg.name, "m": cfg.m, "d": cfg.d, "kernel": cfg.kernel, "dtype": cfg.dtype, "mode": mode,
           "status": st, "iterations": s.iterations, "rel_residual": s.rel_residual, "train_s": tt,  # median run
           "cg_s": s.t_cg, "precompute_s": s.t_precompute, "cg_iterations_per_s": s.iterations / s.t_cg,
           "matvec_ms": 1e3 * mv, "bytes_per_gpu": s.bytes_per_gpu,
           "predict_s": tk, "n_test": cfg.n_test, "test_accuracy": acc,
           "repeats": len(timed), "train_s_cov": float(tts.std() / tts.mean()),
           "cg_iterations_per_s_median": float(np.median(its)), "cg_iterations_per_s_cov": float(its.std() / its.mean()),
           "fp64_engine": {1: "ozaki", 2: "dmma"}.get(s.fp64_engine_used),
           "fp32_engine": {0: "tcgen05", 1: "ffma", 2: "ozaki"}.get(s.fp32_engine_used)
           if cfg.dtype == "f32" else None}
    if mode == "lowrank":  # two streams over X per product (a different cost model, NEXT-2)
        sz = 8 if cfg.dtype == "f64" else 4
        row["matvec_gbs"] = 2.0 * cfg.m * cfg.d * sz / mv / 1e9
        row["frac_of_peak"] = row["matvec_gbs"] / hbm_peak()
        row["peak_gbs"] = hbm_peak()
    elif mode == "implicit" and "ozaki" in (row["fp64_engine"], row["fp32_engine"]):
        d8 = -(-cfg.d // 32) * 32
        pairs = 28 if cfg.dtype == "f64" else 6  # digit pairs per entry (ozaki_engine.cuh: 7 / 3 digits)
        row["matvec_tflops"] = fl / mv / 1e12  # fp64- / fp32-equivalent
        row["matvec_int8_tops"] = pairs * fl * d8 / cfg.d / mv / 1e12
        row["peak_int8_tops_sustained"] = INT8_PEAK
        row["frac_of_peak"] = row["matvec_int8_tops"] / INT8_PEAK
    elif mode == "implicit":
        row["matvec_tflops"] = fl / mv / 1e12
        row["frac_of_peak"] = row["matvec_tflops"] / peak_f
        row["peak_tflops"] = peak_f
    else:  # symmetric-packed cached Q~: the stored upper-triangle tiles are streamed once per product
        sz = 8 if cfg.dtype == "f64" else 4
        T = math.ceil(cfg.m / 128)
        row["stored_bytes"] = T * (T + 1) // 2 * 128 * 128 * sz
        row["matvec_gbs"] = row["stored_bytes"] / mv / 1e9
        row["frac_of_peak"] = row["matvec_gbs"] / hbm_peak()
        row["peak_gbs"] = hbm_peak()
        row["precompute_tflops_equiv"] = fl / s.t_precompute / 1e12 if s.t_precompute > 0 else None
    if cfg.n_test and cfg.kernel != pl.LINEAR:
        row["predict_tflops"] = 2.0 * cfg.n_test * cfg.m * cfg.d / tk / 1e12
    elif cfg.n_test:
        row["predict_path"] = "w = X^T alpha (Eq. 15), O((m + n) d)"
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C0,C1,C2,C3,C4")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfgs = synth.configs()
    out = open(a.out, "w") if a.out else None
    for name in a.configs.split(","):
        for mode, engine in MODES[name]:
            if cfgs[name].dtype == "f32" and engine != "auto":
                continue
            slow = (name, mode) in (("C4", "implicit"), ("C2", "implicit"))
            row = run(cfgs[name], mode, engine, repeat=2 if slow else 11)
            line = json.dumps(row)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
                out.flush()


if __name__ == "__main__":
    main()
