"""Diagnostics: E2 outputs of the history-resident stage kernel vs the multi-source GEMM path,
per channel and per 128-row tile (worst tiles listed). usage: python tools/hist_diag.py [mode A] [mode B]"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(env_val, out):
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r})
from synth import configs as S
from paper_2411_17729_b200.runner import DeviceWorkload
wl = S.make_E2()
import os
if os.environ.get('DIAG_N'): wl.N[:] = int(os.environ['DIAG_N'])
dw = DeviceWorkload(wl); dw.step(); torch.cuda.synchronize()
np.save({out!r}, dw.y_f64()[..., 0].astype(np.float64)); np.save({out!r}.replace('.npy','_N.npy'), wl.N)
"""
    env = dict(os.environ, CASC_BANK_HIST=env_val)
    subprocess.run([sys.executable, "-c", code], env=env, check=True)


mode = sys.argv[1] if len(sys.argv) > 1 else "1"
run(mode, "/tmp/y_hist.npy")
run(sys.argv[2] if len(sys.argv) > 2 else "0", "/tmp/y_mimo.npy")
a, b = np.load("/tmp/y_hist.npy"), np.load("/tmp/y_mimo.npy")
N = np.load("/tmp/y_hist_N.npy")
nch, batch, L = a.shape
err = np.linalg.norm((a - b).reshape(nch, -1), axis=1) / np.linalg.norm(b.reshape(nch, -1), axis=1)
print("channels with rel diff > 1e-6:", [(int(c), int(N[c]), float(err[c])) for c in np.argsort(-err)[:10] if err[c] > 1e-6])
c = int(np.argmax(err))
d = np.abs(a[c] - b[c]).reshape(batch, L // 128, 128).max(axis=2)
bad = np.argwhere(d > 1e-5 * np.abs(b[c]).max())
print("worst channel", c, "N", int(N[c]), "bad (batch, tile):", bad[:40].tolist(), "count", len(bad))
if len(bad):
    bb, tt = bad[0]
    rows = np.abs(a[c, bb, tt * 128:(tt + 1) * 128] - b[c, bb, tt * 128:(tt + 1) * 128])
    scale = np.abs(b[c, bb, tt * 128:(tt + 1) * 128]).max()
    print("tile", int(bb), int(tt), "rows with diff > 1e-5*scale:", np.nonzero(rows > 1e-5 * scale)[0].tolist())
