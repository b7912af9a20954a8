"""Kernel timeline of bench steps (C1 by default) through torch.profiler (CUPTI activity records of
every kernel / memcpy / memset in the process, the library's included): per step, the GPU busy time,
the idle gaps between consecutive device activities and the largest gaps with their neighbours --
where the non-product time of a step goes.  Not a bench number (the profiler is attached).
    python tools/timeline.py [C1] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2202_12674_b200 as pl  # noqa: E402
import synth  # noqa: E402

cfg = synth.configs()[sys.argv[1] if len(sys.argv) > 1 else "C1"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
X, y, Z, _ = synth.config_data(cfg)
tX, ty, tZ = (torch.from_numpy(a).cuda() for a in (X, y, Z))
kw = dict(gamma=cfg.gamma, degree=cfg.degree, coef0=cfg.coef0)


def step():
    o = pl.options(mode=pl.MODE_IMPLICIT, cg_loop=pl.CG_BATCHED)
    alpha, b, st, s = pl.plssvm_train_ex(tX, ty, cfg.kernel, C=cfg.C, eps=cfg.eps, opts=o, **kw)
    pl.plssvm_predict_ex(tX, alpha, float(b.item()), tZ, cfg.kernel, opts=o, **kw)


for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(steps):
        with torch.profiler.record_function("bench_step"):
            step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
marks = sorted((e.time_range.start, e.time_range.end) for e in prof.events() if e.name == "bench_step"
               and e.device_type == torch.autograd.DeviceType.CPU)
t0, t1 = ev[0].time_range.start, ev[-1].time_range.end
busy = sum(e.time_range.end - e.time_range.start for e in ev)
print(f"{len(ev)} device activities over {steps} steps: span {(t1 - t0) / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, "
      f"idle {(t1 - t0 - busy) / 1e3:.3f} ms ({(t1 - t0 - busy) / 1e3 / steps:.3f} ms per step)")
names = {}
for e in ev:
    k = e.name.split("(")[0][:60]
    n, t = names.get(k, (0, 0.0))
    names[k] = (n + 1, t + (e.time_range.end - e.time_range.start))
for k, (n, t) in sorted(names.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:62s} {n:5d} {t / 1e3 / steps:9.3f} ms/step")
gaps = [(ev[i + 1].time_range.start - ev[i].time_range.end, ev[i].name.split("(")[0][:40], ev[i + 1].name.split("(")[0][:40])
        for i in range(len(ev) - 1)]
print(f"gaps > 5 us: {sum(1 for g in gaps if g[0] > 5)}, total {sum(g[0] for g in gaps if g[0] > 5) / 1e3 / steps:.3f} ms/step")
for g, a, b in sorted(gaps, reverse=True)[:25]:
    print(f"  {g:9.1f} us  after {a:40s} before {b}")
