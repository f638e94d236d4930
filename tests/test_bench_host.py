"""Host-side logic of bench.py (no GPU): the roofline of the executed work, the peak selection by
the observed clocks, the round-robin channel deal of E5 and the CPU description."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_roofline_binding_roof_and_peak_choice():
    pk = bench.peaks()
    # one launch moving exactly HBM-peak bytes in 1 ms, with few flops: HBM-bound at frac 1
    by = pk["hbm_gbs"] * 1e9 * 1e-3
    prof = {"bank_stage": {"launches": 1, "ms": 1.0, "bytes": by, "flops": 1e9, "exec_bytes": by,
                           "exec_flops": 1e9, "pipe": "tf32"}}
    r = bench.roofline(prof, "fp32", "E2", {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0})
    assert r["bound"] == "hbm" and abs(r["frac"] - 1.0) < 1e-9
    assert r["executed"]["tensor_peak"] == "burst"
    # many flops: tensor-bound; the sustained peak when the clocks were power-capped
    fl = pk["bf16_tflops_sustained"] * 1e12 * 1e-3
    prof = {"mimo_tc_stage": {"launches": 2, "ms": 2.0, "bytes": 1e6, "flops": fl * 2, "exec_bytes": 1e6,
                              "exec_flops": fl * 2, "pipe": "bf16"}}
    r = bench.roofline(prof, "bf16", "E4", {"sm_mhz": 1000.0, "sm_max_mhz": 1965.0})
    assert r["bound"] == "tensor" and abs(r["frac"] - 1.0) < 1e-9 and r["executed"]["tensor_peak"] == "sustained"
    assert r["avg_launch_ms"] == 1.0
    # the same rate against the burst / sustained / datasheet peaks
    fo = r["frac_other_peaks"]
    assert abs(fo["sustained"] - 1.0) < 1e-9 and fo["burst"] < 1.0 and abs(fo["datasheet"] - fl * 2 / 2e-3 / 1e12 / 2250.0) < 1e-9


def test_e5_round_robin_by_order_balances_stages():
    rng = np.random.default_rng(0)
    N = rng.integers(7, 16, 4096)
    for world in (2, 4, 8):
        parts = [bench.e5_channels(N, world, r) for r in range(world)]
        assert sorted(c for p in parts for c in p) == list(range(4096))      # a partition
        loads = [int((N[p] + 1).sum()) for p in parts]
        assert max(loads) - min(loads) <= 16                                # balanced sum (N_c + 1)


def test_cpu_info_fields():
    ci = bench.cpu_info()
    assert ci["nproc"] >= 1 and ci["blas_threads"] >= 1 and "cpu_model" in ci
