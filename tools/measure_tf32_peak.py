"""Measure the dense TF32 tensor-core peak of this B200 the same way MEASURED_PEAKS.json measures
bf16 (driver recipe): torch.matmul at 8192^3 (2 N^3 flops), best of 10 (burst) and back to back
for 4 s (sustained), CUDA events on the current stream, clocks sampled by nvidia-smi during the
sustained loop. Here the inputs are fp32 with TF32 math enabled (cuBLAS tf32 tensor-core GEMM).

Writes profiles/r02_tf32_peak.json; bench.py reads it as the tf32 roofline denominator (the
3xTF32 kernels issue three tf32 products per source, judged against this peak).

usage (on a B200, e.g. under gpurun): python tools/measure_tf32_peak.py [out.json]
"""
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r02_tf32_peak.json")
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=torch.float32)
    b = torch.randn(n, n, device="cuda", dtype=torch.float32)
    c = torch.empty(n, n, device="cuda", dtype=torch.float32)
    flops = 2.0 * n ** 3
    for _ in range(5):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    fd, clk = tempfile.mkstemp(suffix=".csv")
    os.close(fd)
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                            "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
                            "clocks_event_reasons.sw_thermal_slowdown",
                            "--format=csv,noheader,nounits", "-lms", "200"], stdout=open(clk, "w"),
                           stderr=subprocess.DEVNULL)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    e0.record()
    t_end = time.time() + 4.0
    while time.time() < t_end:
        for _ in range(10):
            torch.matmul(a, b, out=c)
        iters += 10
        torch.cuda.current_stream().synchronize() if iters % 100 == 0 else None
    e1.record()
    torch.cuda.synchronize()
    sustained_s = e0.elapsed_time(e1) / 1e3
    smi.terminate()
    smi.wait()
    sm, reasons = [], set()
    for line in open(clk):
        p = [x.strip() for x in line.split(",")]
        try:
            f = float(p[0])
        except (ValueError, IndexError):
            continue
        if f > 400:
            sm.append(f)
            for nm, v in zip(("sw_power_cap", "hw_slowdown", "sw_thermal_slowdown"), p[3:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
    os.unlink(clk)
    res = {
        "tf32_tflops": flops / best / 1e12,
        "tf32_tflops_sustained": flops * iters / sustained_s / 1e12,
        "gpu_name": torch.cuda.get_device_name(0),
        "torch": torch.__version__,
        "how": "torch.matmul fp32 inputs, allow_tf32, 8192^3 (2 N^3): best of 10 (burst) and back to back "
               "for 4 s (sustained), CUDA events",
        "clocks_sustained": {"sm_mhz_median": statistics.median(sm) if sm else None, "samples": len(sm),
                             "reasons": sorted(reasons)},
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
