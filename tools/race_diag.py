"""diagnostics: repeat the full-size E2 run_host vs device comparison; print mismatch stats"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from synth import configs as S
import test_gpu_e2e_paths as T
wl = S.make_E2()
for k in range(int(os.environ.get("REPS", "3"))):
    wlk, u = T._inputs(wl, k)
    yh = T._run_host(wlk, u)
    yd = T._device_y(wlk, u)
    yd2 = T._device_y(wlk, u)
    d = yh != yd
    dd = yd != yd2
    idx = np.argwhere(d)
    print(f"call {k}: host!=dev {int(d.sum())} (max {np.abs(yh-yd).max():.3e}), dev!=dev {int(dd.sum())}, finite {np.isfinite(yh).all()}",
          "first", idx[:3].tolist(), "chans", sorted(set(idx[:,0].tolist()))[:20], flush=True)
    for a, b_ in ((yh, yd), (yd, yd2)):
        for i in np.argwhere(a != b_)[:40]:
            c, bb, l = int(i[0]), int(i[1]), int(i[2])
            print(f"   ch {c} b {bb} l {l} (tile {l // 128} row {l % 128}) N {int(wlk.N[c])} {a[tuple(i)]:.6e} vs {b_[tuple(i)]:.6e}")
