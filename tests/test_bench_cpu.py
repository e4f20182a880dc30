"""bench.py host-side pieces that need no GPU: the clock sampler's timed-region window (the
contract requires nvidia-smi samples taken DURING the timed region; a region shorter than
nvidia-smi's start-up once produced a line with 0 samples) and its throttle-reason parsing."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def row(sm, reasons=("Not Active",) * 4):
    return [str(sm), "1965", "700.00", *reasons]


def sampler(rows, t0, t1):
    c = bench.ClockSampler(0)
    c.rows = rows
    c.t0, c.t1 = t0, t1
    return c


def test_rows_inside_the_region_only():
    rows = [(0.9, row(1200)), (1.05, row(1965)), (1.10, row(1950)), (1.30, row(1100))]
    s = sampler(rows, 1.0, 1.2).summary()
    assert s["samples"] == 2 and s["sm_mhz"] == 1957.5 and s["sm_max_mhz"] == 1965.0 and s["reasons"] == []


def test_region_shorter_than_the_period_takes_the_nearest_row():
    rows = [(0.5, row(1500)), (1.02, row(1965)), (2.0, row(900))]
    s = sampler(rows, 1.0, 1.001).summary()  # 1 ms region, no row inside (+60 ms grace covers 1.02)
    assert s["samples"] == 1 and s["sm_mhz"] == 1965.0
    s = sampler([(0.5, row(1500)), (3.0, row(900))], 1.0, 1.001).summary()
    assert s["samples"] == 1 and s["sm_mhz"] == 1500.0  # nearest to the region's middle


def test_throttle_reasons_are_reported():
    rows = [(1.05, row(1800, ("Not Active", "Active", "Not Active", "Active")))]
    s = sampler(rows, 1.0, 1.2).summary()
    assert s["reasons"] == ["hw_thermal_slowdown", "sw_power_cap"]


def test_no_rows_no_clock():
    s = sampler([], 1.0, 1.2).summary()
    assert s == {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
