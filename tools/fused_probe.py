"""Diagnostics for the fused bank kernel: run a bank workload with CASC_FUSED_DBG=1 (per-role
wait-cycle accounting printed by the library) and time the apply with CUDA events.
usage: CASC_FUSED_DBG=1 python tools/fused_probe.py [E2|E5] [n_ch]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as S  # noqa: E402
from paper_2411_17729_b200 import api  # noqa: E402
from paper_2411_17729_b200.runner import DeviceWorkload  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "E2"
n_ch = int(sys.argv[2]) if len(sys.argv) > 2 else None
wl = S.make_E2(n_ch=n_ch or 256) if cfg == "E2" else S.make_E5(n_ch=n_ch or 512)
dw = DeviceWorkload(wl)
dw.step()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    e0.record(st)
    api.apply_bank(dw.pw, dw.Bbar, dw.C, dw.D, dw.u, y=dw.y, ws=dw.ws)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"{cfg}: apply {e0.elapsed_time(e1):.3f} ms  env={ {k: v for k, v in os.environ.items() if k.startswith('CASC_')} }",
          flush=True)
