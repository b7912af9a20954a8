#!/usr/bin/env python
"""Benchmark of the PLSSVM B200 hot path (one JSON line on rank 0).

    python bench.py [--gpus N --steps K --warmup W] [--config C1] [--mode implicit|cached|auto]
    python bench.py --impl reference ...        # the CPU oracle as the reference arm

Workload (BASELINE.json configs[1], the metric's single-GPU config): C1 = 2^14 points x 2^10
features, RBF (gamma = 1/d), fp64, implicit Q~p, C = 1, eps = 1e-10, synthetic
make_classification "planes" data (synth/).  A step = one pass of the whole hot path
(SURVEY §8(a) rows a0-a8): plssvm_train_ex on inputs resident in HBM (transform, q, CG to
eps, bias/alpha) followed by plssvm_predict_ex on the 2^13 test points.  `value` = CG
iterations per second of the whole job (max over ranks); ms_per_step = train + predict.
N > 1 (torchrun): Q~ row-sharded over the ranks (NCCL all-gather of p, all-reduce of the CG
scalars), test points sharded for predict; the problem size is fixed -> "scaling": "strong".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "CG iterations/s & kernel-matvec FLOP/s (% peak), train time; 1/2/4/8 B200"
UNIT = "CG it/s"
KNAMES = {0: "linear", 1: "polynomial", 2: "rbf"}
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.2: SMs x DFMA/clk/SM x 2 x max SM clock
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4: FFMA (options.fp32_engine = 1)


def tf32x3_peak_tflops():
    """Useful-flop peak of the 3xTF32 tcgen05 path: the measured bf16 dense peak x the guide's
    nominal tf32/bf16 ratio (1.1 / 2.25 PFLOP/s), / 3 MMAs per useful product."""
    return measured_peaks().get("bf16_tflops", 1590.0) * (1.1 / 2.25) / 3.0


OZAKI_DIGIT_PAIRS = 28  # 7 balanced base-256 digits per point, digit pairs (a, b) with a + b <= 6 (ozaki_engine.cuh)


def int8_peak_tops(sustained=True):
    """Dense int8 tensor peak: the measured bf16 dense peak x the guide's nominal int8/bf16 ratio
    (4.5 / 2.25 POPS).  The Q~p kernel runs back to back inside the CG loop at the power cap, so the
    roofline uses the SUSTAINED bf16 figure (MEASURED_PEAKS.json bf16_tflops_sustained)."""
    pk = measured_peaks()
    bf = pk.get("bf16_tflops_sustained", 1392.0) if sustained else pk.get("bf16_tflops", 1645.0)
    return 2.0 * bf


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


def ncu_entry(key):
    """The ncu capture record of the dominant kernel (profiles/roofline_traffic.json), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as fh:
            return json.load(fh).get(key) or {}
    except (OSError, ValueError):
        return {}


def traffic_for(key):
    """ncu-measured DRAM bytes per launch of the dominant kernel (profiles/roofline_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as fh:
            e = json.load(fh).get(key)
        return None if e is None else e["dram_read_bytes"] + e["dram_write_bytes"]
    except (OSError, ValueError, KeyError):
        return None


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms; summary() keeps the samples taken
    inside the timed region (window(t0, t1), host wall clock; nvidia-smi stamps every sample).  The
    sampler starts before the warm-up steps, so its ~0.5 s start-up does not eat a short timed region."""

    def __init__(self, device, enabled=True):
        self.device = device
        self.enabled = enabled
        self.proc = None
        self.path = None
        self.t0 = self.t1 = None

    def window(self, t0, t1):
        self.t0, self.t1 = t0, t1

    def __enter__(self):
        if not self.enabled:
            return self
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,timestamp")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        if not self.enabled:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["sampled on rank 0"], "samples": 0}
        try:
            with open(self.path) as fh:
                for ln in fh:
                    parts = [x.strip() for x in ln.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
            if self.t0 is not None and rows and len(rows[0]) >= 10:  # samples inside the timed region
                import datetime

                def stamp(r):
                    try:
                        return datetime.datetime.strptime(r[9], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    except ValueError:
                        return None
                inside = [r for r in rows if (stamp(r) or 0.0) >= self.t0 - 0.1 and (stamp(r) or 0.0) <= self.t1 + 0.1]
                rows = inside or rows
        except OSError:
            pass
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": reasons, "samples": len(rows)}
        gpus = sorted({r[0] for r in rows})
        if len(gpus) > 1:  # every GPU of the job: median SM clock and reasons per device
            out["per_gpu"] = {g: {"sm_mhz": statistics.median([float(r[1]) for r in rows if r[0] == g and
                                                               r[1].replace(".", "").isdigit()] or [0.0]),
                                  "reasons": sorted({names[k] for r in rows if r[0] == g for k in range(4)
                                                     if r[5 + k].lower() == "active"})} for g in gpus}
        return out


def matvec_flops(m, d):
    """Algorithmic flops of one Q~p product: 2d per distinct entry of the symmetric Q~."""
    m1 = m - 1
    return 2.0 * d * m1 * (m1 + 1) / 2.0


def host_info():
    """CPU model and core counts of the box (state the CPU beside every oracle number)."""
    info = {"cpu_model": None, "nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                info["cpu_model"] = v
            elif k == "Socket(s)":
                info["sockets"] = int(v)
            elif k == "Core(s) per socket":
                info["cores_per_socket"] = int(v)
            elif k == "Thread(s) per core":
                info["threads_per_core"] = int(v)
    except (OSError, ValueError, subprocess.SubprocessError):
        pass
    return info


def c0_single_thread():
    """C0 also single-threaded -- the oracle's full C0 training in a child process with
    OMP_NUM_THREADS=1 (the OpenMP runtime fixes its thread count at load)."""
    code = ("import sys, time; sys.path.insert(0, %r); import oracle, synth; cfg = synth.configs()['C0']; "
            "X, y, _, _ = synth.config_data(cfg, n_test=0); t = time.perf_counter(); "
            "a, b, it, st = oracle.train(X, y, cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C, cfg.eps); "
            "print(it, time.perf_counter() - t, oracle.num_threads())") % ROOT
    try:
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120,
                             env=dict(os.environ, OMP_NUM_THREADS="1")).stdout.split()
        it, ts, th = int(out[0]), float(out[1]), int(out[2])
        return {"value": it / ts, "unit": UNIT, "cores": th, "sample": f"C0 (256 x 16 linear): {it} CG iterations "
                                                                      f"in {ts * 1e3:.2f} ms, one thread"}
    except (OSError, ValueError, IndexError, subprocess.SubprocessError):
        return None


def cpu_baseline(cfg, X, y, target_s=15.0, m_cap=None):
    """The oracle (as it stands) on the host cores: oracle.train on the first m_s points (same d,
    same kernel), m_s sized for ~target_s of CPU work; both of its phases (Q~ formation and the
    dense CG GEMVs) are O(m^2), so iterations/s is scaled by (m_s/m)^2 to the full workload."""
    import oracle

    oracle.build()
    cores = oracle.num_threads()
    m = cfg.m
    t0 = time.perf_counter()
    ms0 = min(m, 1024)
    oracle.train(X[:ms0], y[:ms0], cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C, cfg.eps)
    t1 = time.perf_counter() - t0
    ms = int(min(m, ms0 * math.sqrt(target_s / max(t1, 1e-3))) // 128 * 128)
    ms = max(ms0, ms if m_cap is None else min(ms, m_cap))
    Xs, ys = X[:ms], y[:ms]
    if ys.min() == ys.max():
        ys = ys.copy()
        ys[-1] = -ys[0]
    t0 = time.perf_counter()
    alpha, b, it, st, tm = oracle.train(Xs, ys, cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C, cfg.eps,
                                        timings=True)
    ts = time.perf_counter() - t0
    scale = (m / ms) ** 2
    return {"value": it / (ts * scale), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"oracle.train on the first {ms} of {m} points (d={cfg.d}, {KNAMES[cfg.kernel]}, eps "
                      f"{cfg.eps:g}): {it} CG iterations in {ts:.2f} s (Q~ formation {tm[0]:.2f} s, CG {tm[1]:.2f} s);"
                      f" time scaled by (m/m_s)^2 = {scale:.2f} to the full workload"
                      + (" (extrapolated)" if scale > 1.0 else " (full workload, not extrapolated)"),
            "extrapolated": scale > 1.0,
            "build": "gcc -O3 -march=native -ffp-contract=off, OpenMP over rows (oracle/__init__.py)",
            "host": host_info(),
            "sample_seconds": ts, "sample_iterations": it, "sample_m": ms}


def run_reference(args, cfg):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    import oracle

    oracle.build()
    X, y, Z, yz = synth.config_data(cfg, n_test=0)
    # size one step for ~ (a few minutes) / (steps + warmup)
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    cal = cpu_baseline(cfg, X, y, target_s=per_step)
    ms = cal["sample_m"]
    Xs, ys = X[:ms], y[:ms]
    for _ in range(args.warmup):
        oracle.train(Xs, ys, cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C, cfg.eps)
    its, t0 = 0, time.perf_counter()
    for _ in range(args.steps):
        _, _, it, _ = oracle.train(Xs, ys, cfg.kernel, cfg.gamma, cfg.degree, cfg.coef0, cfg.C, cfg.eps)
        its += it
    ts = time.perf_counter() - t0
    scale = (cfg.m / ms) ** 2
    value = its / (ts * scale)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * ts * scale / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_dict(cfg, args, "oracle"),
                           workload=f"{cfg.name} oracle training (CG to eps={cfg.eps:g}) on the first {ms} of {cfg.m} "
                                    f"points, time scaled by (m/m_s)^2; no predict (CG it/s counts training only)"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cal["cores"], "kind": "oracle",
                             "sample": f"each step: oracle.train on the first {ms} of {cfg.m} points; time scaled "
                                       f"by (m/m_s)^2 = {scale:.2f}" + (" (extrapolated)" if scale > 1.0 else ""),
                             "extrapolated": scale > 1.0, "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                    "extrapolated": scale > 1.0}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(cfg, args, mode):
    return {"workload": f"{cfg.name}: 2^{int(math.log2(cfg.m))} x 2^{int(math.log2(cfg.d))} {KNAMES[cfg.kernel]} "
                        f"{cfg.dtype} {mode} Q~p, CG to eps={cfg.eps:g}, + predict on {cfg.n_test} test points",
            "m": cfg.m, "d": cfg.d, "kernel": KNAMES[cfg.kernel], "gamma": cfg.gamma, "degree": cfg.degree,
            "coef0": cfg.coef0, "C": cfg.C, "eps": cfg.eps, "mode": mode, "n_test": cfg.n_test,
            "parallelism": f"row-sharded Q~ x{args.gpus}" if args.gpus > 1 else "1 GPU",
            "l2": l2_note(cfg)}


def l2_note(cfg):
    """The per-step working set against the 126 MB L2 (inputs larger than L2: no flush between steps)."""
    s = 4 if cfg.dtype == "f32" else 8
    digits = 3 if cfg.dtype == "f32" else 7  # int8 digit planes of the tensor-core engines
    d8 = -(-cfg.d // 32) * 32
    x, z = cfg.m * cfg.d * s, cfg.n_test * cfg.d * s
    dx, dz = digits * cfg.m * d8, digits * cfg.n_test * d8
    mib = lambda b: f"{b / 2**20:.0f} MiB"  # noqa: E731
    return (f"inputs larger than L2: X {mib(x)} + its digits {mib(dx)} (train, again in predict) + Z {mib(z)} + "
            f"its digits {mib(dz)} per step > 126 MB L2; no flush")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C1")
    ap.add_argument("--mode", default="implicit", choices=["implicit", "cached", "auto"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    # testing the multi-rank bench logic on a one-GPU box: every rank on cuda:0, exchanges through
    # the host-staged gloo transport (NCCL refuses two ranks on one device).  Not for measurement.
    ap.add_argument("--transport", default="nccl", choices=["nccl", "gloo"])
    args = ap.parse_args()
    cfg = synth.configs()[args.config]
    bad = sorted(k for k in os.environ if k.startswith("PLSSVM_"))
    if bad:  # experiment switches / library overrides must not leak into a measurement
        print(json.dumps({"error": f"refusing to benchmark with {bad} set"}), flush=True)
        return 2
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` launches its own N ranks (one process per GPU, NCCL), the same way the
        # driver's scaling run does; this process only waits for them
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 2000}",
               os.path.abspath(__file__), *sys.argv[1:]]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_2202_12674_b200 as pl

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0) if args.transport == "nccl" else 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.transport == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    if world > 1:
        comm = pl.comm_from_torch_distributed(local) if args.transport == "nccl" else \
            pl.comm_host_staged(local, circulant=True)
        if rank == 0:  # the communicator the library uses, for the driver's rank check
            print(f"[bench] communicator: {args.transport} nranks={world} devices={world if args.transport == 'nccl' else 1}"
                  f" ({pl.plssvm_version()})", file=sys.stderr, flush=True)
    else:
        comm = None
    rdev = dev if args.transport == "nccl" else torch.device("cpu")  # device of the timing all-reduces

    mode = {"implicit": pl.MODE_IMPLICIT, "cached": pl.MODE_CACHED, "auto": pl.MODE_AUTO}[args.mode]
    dt = np.float32 if cfg.dtype == "f32" else np.float64
    X, y, Z, yz = synth.config_data(cfg)
    n = Z.shape[0]
    z0, z1 = rank * n // world, (rank + 1) * n // world  # test-point shard of this rank
    tX = torch.from_numpy(X).to(dev)
    ty = torch.from_numpy(y).to(dev)
    tZ = torch.from_numpy(np.ascontiguousarray(Z[z0:z1])).to(dev)
    kw = dict(gamma=cfg.gamma, degree=cfg.degree, coef0=cfg.coef0)

    def opts():
        # the batched CG loop (AUTO's choice at the bench workload): per-launch CUDA events on the
        # product's stream give roofline.achieved (no events inside a CUDA-graph loop body)
        return pl.options(mode=mode, comm=comm, device=local, cg_loop=pl.CG_BATCHED)

    def step():
        alpha, b, st, stats = pl.plssvm_train_ex(tX, ty, cfg.kernel, C=cfg.C, eps=cfg.eps, opts=opts(), **kw)
        f, lab, (tk, nl) = pl.plssvm_predict_ex(tX, alpha, float(b.item()), tZ, cfg.kernel, opts=opts(), **kw)
        return stats, nl, alpha, b, lab

    # clocks of every GPU of the job (rank 0 samples them all; one process per GPU, devices 0..N-1),
    # started before the warm-up; only the samples inside the timed region are summarised
    sampler = ClockSampler(",".join(str(i) for i in range(world)) if args.transport == "nccl" else local,
                           enabled=rank == 0)
    per = []
    with sampler:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.time()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            per.append(step())
        ev1.record()
        torch.cuda.synchronize()
        sampler.window(w0, time.time())
    if world > 1:
        dist.barrier()
    t = ev0.elapsed_time(ev1) / 1e3
    if world > 1:
        tt = torch.tensor([t], device=rdev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    clocks = sampler.summary()
    iters = sum(s.iterations for s, *_ in per)
    matvecs = sum(s.iterations for s, *_ in per)
    t_mv = sum(s.t_matvec for s, *_ in per)
    launches = sum(s.gpu_launches + int(nl) for s, nl, *_ in per)
    stats0 = per[-1][0]
    mode_used = {1: "implicit", 2: "cached"}[stats0.mode_used]

    # ---- roofline of the dominant kernel (the Q~p product), timed with CUDA events on its stream
    avg_mv = t_mv / max(1, matvecs)
    if cfg.dtype == "f64":
        engine = {1: "ozaki", 2: "dmma"}.get(stats0.fp64_engine_used, "dmma")
    else:
        engine = {0: "tcgen05-3xtf32", 1: "ffma", 2: "ozaki"}.get(stats0.fp32_engine_used, "tcgen05-3xtf32")
    if mode_used == "implicit" and engine == "ozaki":
        # int8 digit products per launch: 28 pairs x 2 d8 ops per distinct Q~ entry (d8 = d rounded up to
        # the 32-feature slab), this rank's ~1/P share; fp64-equivalent rate reported beside it
        fl = matvec_flops(cfg.m, cfg.d) / world
        d8 = -(-cfg.d // 32) * 32
        pairs = OZAKI_DIGIT_PAIRS if cfg.dtype == "f64" else 6  # fp32 engine: 3 digits, levels <= 2
        ops = pairs * fl * d8 / cfg.d
        peak = int8_peak_tops(sustained=True)
        achieved = ops / avg_mv / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS (int8)", "frac": achieved / peak,
                "traffic": traffic_for(f"{cfg.name}/implicit/k_tile_ozaki") if world == 1 else None,
                "traffic_unit": "bytes per launch (ncu dram read+write)", "kernel": "k_tile_ozaki (OZ_MATVEC)",
                "per_launch": f"{pairs} digit pairs x 2*d8 int8 ops per distinct Q~ entry, E = m'(m'+1)/2 "
                              f"({ops:.4g} int8 ops per launch per rank)",
                "peak_source": "int8 dense = 2 x MEASURED_PEAKS.json bf16_tflops_sustained (guide ratio 4.5/2.25; "
                               "the kernel runs back to back at the 1 kW power cap)",
                "frac_of_burst_peak": achieved / int8_peak_tops(sustained=False),
                # utilisation as ncu counts it (one cold, serialised capture; profiles/): the tensor pipe's
                # active cycles, which the fractions above (against a measured GEMM rate) can overstate
                "ncu_tensor_pipe_pct": ncu_entry(f"{cfg.name}/implicit/k_tile_ozaki").get("ncu_tensor_pipe_pct")
                if world == 1 else None,
                "avg_launch_s": avg_mv}
        if cfg.dtype == "f64":
            roof["fp64_equivalent"] = {"achieved_tflops": fl / avg_mv / 1e12, "dmma_peak_tflops": FP64_PEAK_TFLOPS,
                                       "ratio": fl / avg_mv / 1e12 / FP64_PEAK_TFLOPS}
        else:
            roof["fp32_equivalent"] = {"achieved_tflops": fl / avg_mv / 1e12,
                                       "tf32x3_peak_tflops": tf32x3_peak_tflops(),
                                       "ratio": fl / avg_mv / 1e12 / tf32x3_peak_tflops()}
    elif mode_used == "implicit":
        fl = matvec_flops(cfg.m, cfg.d) / world  # this rank's share (symmetric work split)
        peak = FP64_PEAK_TFLOPS if cfg.dtype == "f64" else tf32x3_peak_tflops()
        achieved = fl / avg_mv / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic_for(f"{cfg.name}/implicit/k_matvec_implicit") if world == 1 else None,
                "traffic_unit": "bytes per launch (ncu dram read+write)", "kernel": "k_matvec_implicit",
                "per_launch": f"2*d*E flops, E = m'(m'+1)/2 distinct Q~ entries ({fl:.4g} flops per launch per rank)",
                "peak_source": "fp64: 148 SMs x 64 FMA/clk x 2 x 1.965 GHz = 37.2 (DMMA measured 37.1, "
                               "profiles/r01_fp64_peak.txt); fp32: measured bf16 x 1.1/2.25 / 3 (3xTF32 tcgen05)",
                "avg_launch_s": avg_mv}
    else:
        s = 8 if cfg.dtype == "f64" else 4
        T = int(math.ceil(cfg.m / (128 * world)) * world)
        by = T * (T + 1) / 2 / world * 128 * 128 * s  # symmetric-packed tiles, ~1/P per rank
        peak = measured_peaks().get("hbm_gbs", 6650.0)
        achieved = by / avg_mv / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic_for(f"{cfg.name}/cached/k_gemv_sym") if world == 1 else None, "kernel": "k_gemv_sym", "per_launch": f"{by:.4g} bytes of stored (symmetric-packed) Q~ tiles per rank",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)", "avg_launch_s": avg_mv}

    line = {"metric": METRIC, "value": iters / t, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic (sklearn make_classification planes, seeded)",
            "config": dict(config_dict(cfg, args, mode_used), fp64_engine=engine if cfg.dtype == "f64" else None,
                           fp32_engine=engine if cfg.dtype == "f32" else None,
                           contraction=(("int8 digit products (exact int32 sums) combined in f64" if cfg.dtype == "f64" else
                                         "int8 digit products of a 3-digit (22-bit) split, exact int32 sums, "
                                         "f32 epilogue") if engine == "ozaki"
                                        else None)),
            "gpu_launches": launches, "clocks": clocks,
            "roofline": roof,
            "train": {"iterations_per_step": iters / args.steps, "t_train_s": stats0.t_total,
                      "t_cg_s": stats0.t_cg, "t_precompute_s": stats0.t_precompute,
                      "t_transform_s": stats0.t_transform, "t_q_s": stats0.t_q, "rel_residual": stats0.rel_residual,
                      "t_comm_s": stats0.t_comm,
                      "bytes_per_gpu": stats0.bytes_per_gpu, "launches_in_cg": stats0.launches_in_cg,
                      "matvec_ms_avg": 1e3 * avg_mv, "matvec_ms_min": 1e3 * stats0.t_matvec_min,
                      # the paper's variability measure: coefficient of variation over the K steps
                      "t_train_cov": float(np.std([st.t_total for st, *_ in per]) /
                                           max(np.mean([st.t_total for st, *_ in per]), 1e-30))}}

    # ---- e2e: same metric through the public API with HOST buffers (pinned), copies inside
    if not args.no_e2e:
        hX = torch.from_numpy(X).pin_memory().numpy()
        hy = torch.from_numpy(y).pin_memory().numpy()
        hZ = torch.from_numpy(np.ascontiguousarray(Z[z0:z1])).pin_memory().numpy()
        for _ in range(1):
            a_h, b_h, _, _ = pl.plssvm_train_ex(hX, hy, cfg.kernel, C=cfg.C, eps=cfg.eps, opts=opts(), **kw)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        its_e, t_h2d = 0, 0.0
        for _ in range(args.steps):
            a_h, b_h, st, stt = pl.plssvm_train_ex(hX, hy, cfg.kernel, C=cfg.C, eps=cfg.eps, opts=opts(), **kw)
            f_h, lab_h, _ = pl.plssvm_predict_ex(hX, a_h, b_h, hZ, cfg.kernel, opts=opts(), **kw)
            its_e += stt.iterations
            t_h2d += stt.t_h2d
        te = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([te], device=rdev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        es = X.itemsize
        h2d = X.nbytes + y.nbytes + X.nbytes + a_h.nbytes + hZ.nbytes
        d2h = a_h.nbytes + es + f_h.nbytes + lab_h.nbytes
        line["e2e"] = {"value": its_e / te, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                       "ms_per_step": 1e3 * te / args.steps,
                       # training's own staging copy (device events; predict's copies are inside its call)
                       "train_h2d_ms_per_step": 1e3 * t_h2d / args.steps,
                       "api": "plssvm_train_ex + plssvm_predict_ex on pinned host numpy buffers"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, X, y)
        line["cpu_baseline"]["c0_single_thread"] = c0_single_thread()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        pl.plssvm_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
