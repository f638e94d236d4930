"""Diagnostic: relative L2 error (y and state part) of the GPU path vs the oracle for a few shapes."""
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
    Du = np.stack([u[c] @ wl.D[c].T for c in range(wl.n_ch)])
    r = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    return r(y, ref), r(y - Du, ref - Du)

cases = {
  "E3red": lambda: S.make_E3(L=4096, batch=2),
  "E3red_N5": lambda: S.make_E3(L=4096, batch=2, N=5),
  "m256_rand": lambda: S.make_random_mimo(256, 64, 64, L=4096, batch=2, N=11, rho=0.98),
  "m64_rand": lambda: S.make_random_mimo(64, 64, 64, L=4096, batch=2, N=11, rho=0.98),
  "E2red": lambda: S.make_E2(n_ch=8, L=4096, batch=2),
}
for name, mk in cases.items():
    print(name, "%.3e %.3e" % err(mk()), flush=True)
