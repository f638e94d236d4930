"""Diagnostics: host->device->host timing pieces of the E2 e2e path (casc_run_host)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as S  # noqa: E402
import paper_2411_17729_b200 as pk  # noqa: E402
from paper_2411_17729_b200.runner import storage_to_torch  # noqa: E402

wl = S.make_E2()
n = wl.n_ch
f = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
Ab, Bb, C, D = f(wl.Abar), f(wl.Bbar), f(wl.C), f(wl.D)
u_h = storage_to_torch(wl.u_storage(), "fp32").reshape(n, wl.batch, wl.L, 1).pin_memory()
y_h = torch.empty_like(u_h).pin_memory()
Ns = [int(x) for x in wl.N]
ws = torch.empty(pk.run_host_bytes(n, wl.m, 1, 1, wl.L, wl.batch, max(Ns), "fp32"), dtype=torch.uint8, device="cuda")
u_d = torch.empty_like(u_h, device="cuda")
for _ in range(3):
    pk.run_host(Ab, Bb, C, D, u_h, y_h, Ns, "fp32", ws)
torch.cuda.synchronize()
for label in ("run_host", "h2d u", "d2h y", "h2d+d2h concurrent"):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if label == "run_host":
            pk.run_host(Ab, Bb, C, D, u_h, y_h, Ns, "fp32", ws)
        elif label == "h2d u":
            u_d.copy_(u_h, non_blocking=True)
        elif label == "d2h y":
            y_h.copy_(u_d, non_blocking=True)
        else:
            s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
            with torch.cuda.stream(s1):
                u_d.copy_(u_h, non_blocking=True)
            with torch.cuda.stream(s2):
                y_h.copy_(u_d, non_blocking=True)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{label}: {np.median(ts):.3f} ms (wall)", os.environ.get("CASC_RUN_HOST_SERIAL"), flush=True)

if os.environ.get("E2E_TRACE"):
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pk.run_host(Ab, Bb, C, D, u_h, y_h, Ns, "fp32", ws)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    t0 = min(e.time_range.start for e in evs)
    for e in sorted(evs, key=lambda e: e.time_range.start):
        sid = getattr(e, "device_resource_id", None)
        print(f"{(e.time_range.start - t0) / 1e3:8.3f} {(e.time_range.end - t0) / 1e3:8.3f}  s{sid}  {e.name[:60]}")
