"""One device step (powers + apply) of a BASELINE config, optionally at a reduced length, for
ncu captures of individual kernels (diagnostics).  usage: python tools/prof_step.py E4 [L] [batch]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as S  # noqa: E402
from paper_2411_17729_b200.runner import DeviceWorkload  # noqa: E402

cfg = sys.argv[1]
kw = {}
if len(sys.argv) > 2:
    kw["L"] = int(sys.argv[2])
if len(sys.argv) > 3:
    kw["batch"] = int(sys.argv[3])
wl = {"E2": S.make_E2, "E3": S.make_E3, "E4": S.make_E4, "E5": S.make_E5}[cfg](**kw)
dw = DeviceWorkload(wl)
for _ in range(2):
    dw.step()
torch.cuda.synchronize()
print("ok", cfg, kw)
