"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(runner.DeviceWorkload.step: powers + apply on device-resident inputs), checked on sampled
outputs. The oracle computes each sampled window exactly from the minimal input window
(the cascade is a polynomial of degree 2^(N+1)-1 in the shift; pin T14)."""
import numpy as np
import pytest
import torch

import oracle
from synth import configs as S

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def run_full(wl):
    from paper_2411_17729_b200.runner import DeviceWorkload
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    dw = DeviceWorkload(wl)
    dw.step()
    torch.cuda.synchronize()
    return dw


def sampled_windows(wl, dw, windows, W, tol):
    N = int(wl.N[0])
    P = oracle.powers(wl.Abar[0], N)
    ys, refs, sts, strefs = [], [], [], []
    for b, l0 in windows:
        y = dw.y[b, l0:l0 + W, :].float().cpu().double().numpy()
        ref = oracle.workload_window(wl, 0, b, l0, W, P=P)
        Du = wl.u_window(0, b, l0, l0 + W) @ wl.D[0].T
        ys.append(y); refs.append(ref); sts.append(y - Du); strefs.append(ref - Du)
    e = rel(np.concatenate(ys), np.concatenate(refs))
    es = rel(np.concatenate(sts), np.concatenate(strefs))
    print(f"{wl.name} sampled rel {e:.3e} state {es:.3e}")
    assert e <= tol and es <= tol, (e, es)


def test_E3_full_size_sampled():
    wl = S.make_E3()                                   # m=256, p=q=64, L=65536, batch=16, N=13
    dw = run_full(wl)
    L = wl.L
    windows = [(0, 0), (3, 1000), (7, 16383), (11, 32768 - 7), (15, L - 64), (5, 40000)]
    sampled_windows(wl, dw, windows, 64, 1e-5)


def test_E5_full_size_sampled_channels():
    """configs[4]: 4096 HiPPO channels, L=65536, batch 8 -- states of 550 GB per buffer, so the
    bank runs in channel waves inside the library; channels spanning N_c = min..15 are checked
    over their whole length against the float64 oracle."""
    wl = S.make_E5()
    dw = run_full(wl)
    order = np.argsort(wl.N, kind="stable")
    pick = sorted({int(order[0]), int(order[len(order) // 2]), int(order[-1]), 0, wl.n_ch - 1})
    for c in pick:
        y = dw.y[c].float().cpu().double().numpy()                  # [batch][L]
        u = np.stack([wl.u_window(c, b, 0, wl.L)[:, 0] for b in range(wl.batch)])
        N = int(wl.N[c])
        ref = oracle.cascade(oracle.powers(wl.Abar[c], N), wl.Bbar[c], wl.C[c], wl.D[c], u[:, :, None], N)[:, :, 0]
        Du = u * wl.D[c, 0, 0]
        e, es = rel(y, ref), rel(y - Du, ref - Du)
        print(f"E5 channel {c} N={N}: rel {e:.3e} state {es:.3e}")
        assert e <= 1e-5 and es <= 1e-5, (c, N, e, es)


def test_E4_full_size_sampled():
    wl = S.make_E4()                                   # m=1024, p=q=256, L=2^20, batch=8, bf16
    dw = run_full(wl)
    L = wl.L
    windows = [(0, 0), (2, 4095), (5, L // 2 + 3), (7, L - 48)]
    sampled_windows(wl, dw, windows, 48, 2e-2)


def test_E2_exponential_full_size_sampled_channels():
    """E2's shape (256 channels, L = 16384, batch 4) with the exponential scheme (NEXT-4): channels
    spanning the N_c range checked over their whole length against the float64 oracle."""
    wl = S.make_E2(scheme="exponential")
    dw = run_full(wl)
    order = np.argsort(wl.N, kind="stable")
    for c in sorted({int(order[0]), int(order[len(order) // 2]), int(order[-1])}):
        y = dw.y[c].float().cpu().double().numpy()
        u = np.stack([wl.u_window(c, b, 0, wl.L)[:, 0] for b in range(wl.batch)])
        N = int(wl.N[c])
        ref = oracle.cascade(oracle.powers(wl.Abar[c], N), wl.Bbar[c], wl.C[c], wl.D[c], u[:, :, None], N)[:, :, 0]
        Du = u * wl.D[c, 0, 0]
        e, es = rel(y, ref), rel(y - Du, ref - Du)
        print(f"E2x channel {c} N={N}: rel {e:.3e} state {es:.3e}")
        assert e <= 1e-5 and es <= 1e-5, (c, N, e, es)
