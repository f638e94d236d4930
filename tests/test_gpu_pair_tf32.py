"""GPU parity of the 3xTF32 CTA-pair stage GEMM (mimo_tc3.cu: fp32 MIMO stages with n_out % 128
== 0 on 256 x 128 tiles over two CTAs) against the float64 oracle, and against the one-CTA
3xTF32 GEMM it replaces (CASC_GEMM_PAIR_TF32=0, subprocess: settings are read once). Cases: the
E3 shape reduced, ragged lengths (a pair tile's second half partly or wholly past L), one and
several sequences, stages skipped at the front (t_first odd and even)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from synth import configs as S

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2411_17729_b200 as pk
    pk.lib()


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


CASES = [  # (m, p, q, L, batch, N)
    (256, 64, 64, 4096, 2, 11),      # E3 shape, reduced length
    (256, 64, 64, 3000, 3, 12),      # ragged: last pair tile half past L
    (128, 64, 128, 385, 1, 9),       # 1.5 pair tiles
    (128, 64, 64, 129, 2, 8),        # second CTA of the only pair tile nearly empty
    (256, 128, 64, 1000, 1, 10),
]


def _wl(m, p, q, L, batch, N):
    return S.make_random_mimo(m, p, q, L=L, batch=batch, N=N, rho=0.98, mode="fp32", seed=m + L + N)


def _gpu_y(case, env=None):
    if not env:
        from paper_2411_17729_b200.runner import DeviceWorkload
        dw = DeviceWorkload(_wl(*case))
        dw.step()
        torch.cuda.synchronize()
        return dw.y_f64()
    out = os.path.join("/tmp", f"pair_tf32_y_{os.getpid()}.npy")
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r})
from test_gpu_pair_tf32 import _wl
from paper_2411_17729_b200.runner import DeviceWorkload
dw = DeviceWorkload(_wl(*{tuple(case)!r})); dw.step(); torch.cuda.synchronize()
np.save({out!r}, dw.y_f64())
"""
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), check=True, timeout=600, cwd=ROOT)
    y = np.load(out)
    os.remove(out)
    return y


@pytest.mark.parametrize("case", CASES)
def test_pair_tf32_vs_oracle(case):
    wl = _wl(*case)
    y = _gpu_y(case)
    u = wl.u_all()
    y_ref = oracle.apply_workload(wl, u=u, channels=range(wl.n_ch))
    Du = np.stack([u[c] @ wl.D[c].T for c in range(wl.n_ch)])
    assert np.all(np.isfinite(y))
    e, es = rel(y, y_ref), rel(y - Du, y_ref - Du)
    assert e <= 1e-5 and es <= 1e-5, (e, es)


@pytest.mark.parametrize("case", CASES[:2])
def test_pair_tf32_matches_single_cta_gemm(case):
    """Same stage products on one CTA per 128 x 128 tile: equal to the 3xTF32 accuracy (the
    correction terms are summed in a different order)."""
    y_pair = _gpu_y(case)
    y_one = _gpu_y(case, {"CASC_GEMM_PAIR_TF32": "0"})
    assert rel(y_pair, y_one) < 2e-6


@pytest.mark.parametrize("case", [(64, 64, 64, 1000, 3, 9), (192, 64, 64, 700, 2, 8)])
def test_64_wide_outputs(case):
    """64-column outputs (m = 64 stages, q = 64 output stages) stay on the one-CTA 3xTF32 kernel
    (a 256 x 64 pair tile measured slower); parity against the oracle."""
    wl = _wl(*case)
    y = _gpu_y(case)
    u = wl.u_all()
    y_ref = oracle.apply_workload(wl, u=u, channels=range(wl.n_ch))
    assert rel(y, y_ref) <= 1e-5
