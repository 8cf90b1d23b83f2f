"""bench.py host logic on CPU: step statistics, FLOP / byte accounting of the roofline, and the
oracle cost model used for the labelled CPU extrapolation."""
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_step_stats_first_last():
    ms = [10.0] * 10 + [12.0] * 10
    s = bench.step_stats(ms)
    assert s["first_mean"] == 10.0 and s["last_mean"] == 12.0 and s["first_last_n"] == 10
    assert s["mean"] == 11.0 and s["median"] == 11.0 and s["min"] == 10.0 and s["max"] == 12.0
    assert bench.step_stats([3.0, 5.0])["first_last_n"] == 1


def test_flop_conventions():
    # reading #14: fwd = 4 B Hq N^2 d (x1/2 causal); C3 fwd 8.80e12
    assert abs(bench.fwd_flops(16, 8192, 32, 128, True) - 8.796e12) / 8.796e12 < 1e-3
    # oracle cost 12 G n^2 d (x1/2 causal) per unit; full C3 2.6e13
    assert abs(bench.oracle_full_cost(bench.CONFIGS["C3"]) - 2.64e13) / 2.64e13 < 1e-2


def test_kernel_table_labels_dq_executed_vs_algorithmic():
    ff = 1e12
    pb = types.SimpleNamespace(fwd_flops=ff, B=1, N=1024, Hq=8, d=128, name="X")
    peaks = {"burst": 1600.0, "sustained": 1400.0, "hbm_gbs": 6000.0, "source": "t", "sustained_at_mhz": None}
    kern = {"fwd": 1.0, "bwd_pre": 0.1, "bwd_dkdv": 2.0, "bwd_dq": 1.5}
    table, roof, dom = bench.kernel_table(pb, kern, peaks, 1)
    assert dom == "bwd_dkdv" and roof["peak"] == 1600.0  # burst denominator
    assert abs(roof["achieved"] - 1000.0) < 1e-6 and abs(roof["frac"] - 0.625) < 1e-9
    assert table["bwd_dq"]["tflops_executed"] == 1000.0 and abs(table["bwd_dq"]["tflops_algorithmic"] - 333.3) < 0.1
    assert table["fwd"]["tflops_executed"] == table["fwd"]["tflops_algorithmic"] == 1000.0
