"""Diagnostic: MIMO tensor-core error vs number of stages (N) and K."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle
from synth import configs as S
from paper_2411_17729_b200.runner import DeviceWorkload

def err(wl):
    dw = DeviceWorkload(wl); dw.step(); torch.cuda.synchronize()
    y = dw.y_f64(); u = wl.u_all(); ref = oracle.apply_workload(wl, u=u)
    return float(np.linalg.norm(y - ref) / np.linalg.norm(ref))

for m, p in ((64, 64), (256, 64), (256, 256)):
    for N in (0, 1, 2, 4, 8):
        wl = S.make_random_mimo(m, p, p, L=2048, batch=1, N=N, rho=0.9)
        print(m, p, N, "%.3e" % err(wl), flush=True)
