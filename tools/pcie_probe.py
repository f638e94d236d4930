"""Diagnostics: host<->device copy rates from pinned memory (alone and both directions at once)."""
import sys
import time

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = int(gb * 2**30) // 4
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for label in ("h2d", "d2h", "both", "h2d 64MB chunks"):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if label in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if label in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
        if label == "h2d 64MB chunks":
            c = 2**24
            with torch.cuda.stream(s1):
                for i in range(0, n, c):
                    d_in[i:i + c].copy_(h_in[i:i + c], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{label}: {gb:.1f} GiB in {dt * 1e3:.1f} ms = {gb * 2**30 / dt / 1e9:.1f} GB/s per direction")
