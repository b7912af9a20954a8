"""Host logic of bench.py (no GPU): the clock sampler keeps only the samples taken inside the timed
region (nvidia-smi stamps each sample; the sampler starts before the warm-up), falls back to all
samples when the stamps cannot be parsed, and reports the throttle reasons the contract names; the
per-step working-set note and the algorithmic flop count of one product."""
import datetime
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402


def _sampler_with_rows(rows):
    cs = bench.ClockSampler(0)
    fd, cs.path = tempfile.mkstemp(suffix=".csv")
    os.close(fd)
    with open(cs.path, "w") as fh:
        for r in rows:
            fh.write(", ".join(str(x) for x in r) + "\n")
    return cs


def _row(mhz, t, power_cap="Active", thermal="Not Active"):
    ts = datetime.datetime.fromtimestamp(t).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
    return [0, mhz, 1965, 900.0, "0x4", "Not Active", "Not Active", thermal, power_cap, ts]


def test_clock_sampler_keeps_the_timed_window():
    t0 = time.time()
    rows = [_row(1000 + k, t0 + 0.2 * k) for k in range(10)]  # samples at t0 .. t0 + 1.8 s
    rows[1] = _row(500, t0 + 0.2, thermal="Active")  # a throttled warm-up sample, outside the window
    cs = _sampler_with_rows(rows)
    cs.window(t0 + 0.55, t0 + 1.25)  # inside (+-0.1 s): samples 3 .. 6
    out = cs.summary()
    assert out["samples"] == 4
    assert out["sm_mhz"] == 1004.5
    assert out["sm_max_mhz"] == 1965.0
    assert out["reasons"] == ["sw_power_cap"]  # the warm-up's thermal reason is not in the window


def test_clock_sampler_without_parsable_stamps_uses_all_samples():
    rows = [[0, 1700 + k, 1965, 900.0, "0x0", "Not Active", "Active", "Not Active", "Not Active", "n/a"]
            for k in range(3)]
    cs = _sampler_with_rows(rows)
    cs.window(time.time() - 1.0, time.time())
    out = cs.summary()
    assert out["samples"] == 3 and out["sm_mhz"] == 1701.0 and out["reasons"] == ["hw_thermal_slowdown"]


def test_l2_note_and_product_flops():
    c1 = synth.configs()["C1"]
    note = bench.l2_note(c1)
    assert "X 128 MiB" in note and "digits 112 MiB" in note and "Z 64 MiB" in note and "no flush" in note
    m1 = c1.m - 1
    assert bench.matvec_flops(c1.m, c1.d) == 2.0 * c1.d * m1 * (m1 + 1) / 2.0  # 2d per distinct entry (§5)
