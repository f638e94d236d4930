"""GPU parity of the history-resident bank stage kernel (bank_hist.cu) against the
float64 oracle, in the configurations its tile walk distinguishes: stage pairs and single stages,
shifts of 1..16 tiles, leading tiles skipped (t_first > 0: warm-up tiles), CTA ranges that start
inside a residue-class chain, ragged lengths, outputs stored (non-final passes) and fused into the
(C v, C P_Ne v) parts (final passes), and the same with the fusion off (every pass stores v).
Variants that need a different library setting run in a subprocess (the settings are read once)."""
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


def _bank(n_ch, L, batch, orders, seed=3):
    wl = S.make_E2(n_ch=n_ch, L=L, batch=batch, seed=seed)
    wl.N[:] = np.asarray(orders)
    return wl


def _gpu_y(wl, env=None):
    """y of the bank from the CUDA path; with `env`, in a subprocess with those settings."""
    if not env:
        from paper_2411_17729_b200.runner import DeviceWorkload
        dw = DeviceWorkload(wl)
        dw.step()
        torch.cuda.synchronize()
        return dw.y_f64()
    out = os.path.join("/tmp", f"hist_y_{os.getpid()}.npy")
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r})
from synth import configs as S
from paper_2411_17729_b200.runner import DeviceWorkload
wl = S.make_E2(n_ch={wl.n_ch}, L={wl.L}, batch={wl.batch}, seed=3)
wl.N[:] = np.asarray({[int(x) for x in wl.N]!r})
dw = DeviceWorkload(wl); dw.step(); torch.cuda.synchronize()
np.save({out!r}, dw.y_f64())
"""
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), check=True, timeout=600)
    y = np.load(out)
    os.remove(out)
    return y


def _check(wl, y, tol=1e-5):
    u = wl.u_all()
    y_ref = oracle.apply_workload(wl, u=u, channels=range(wl.n_ch))
    Du = np.stack([u[c] @ wl.D[c].T for c in range(wl.n_ch)])
    assert np.all(np.isfinite(y))
    e, es = rel(y, y_ref), rel(y - Du, y_ref - Du)
    assert e <= tol and es <= tol, (e, es)


# Orders 9..13 give pair passes at k = 7 (shift 1 tile), 9 (4 tiles, t_first = 1) and 11 (16 tiles,
# t_first = 4) and single passes at k = 9 and 11; 48 tiles per sequence keep every shift a divisor.
ORDERS = [9, 10, 11, 12, 13, 13, 12, 11]


def test_hist_pairs_and_singles_vs_oracle():
    wl = _bank(8, 128 * 48, 3, ORDERS)
    _check(wl, _gpu_y(wl))


def test_hist_ragged_length_vs_oracle():
    """L = 48 tiles - 37 rows: the last tile is partial (loads zero-filled, rows >= L not written)."""
    wl = _bank(5, 128 * 48 - 37, 2, [11, 13, 9, 12, 10])
    _check(wl, _gpu_y(wl))


def test_hist_every_pass_stores_v():
    """Output fusion off: every pass (including each channel's last) writes v, the tail forms y."""
    wl = _bank(6, 128 * 48, 2, ORDERS[:6])
    _check(wl, _gpu_y(wl, {"CASC_BANK_AB": "0"}))


def test_hist_matches_multisource_gemm():
    """The history-resident kernel and the multi-source GEMM compute the same passes (different
    summation order inside a tile): outputs agree to the 3xTF32 accuracy."""
    wl = _bank(8, 128 * 48, 2, ORDERS)
    y_hist = _gpu_y(wl)
    y_gemm = _gpu_y(wl, {"CASC_BANK_HIST": "0"})
    assert rel(y_hist, y_gemm) < 2e-6


def test_hist_many_short_ranges():
    """One channel over 148 CTAs: most CTA ranges start inside a chain (up to three warm-up tiles)."""
    wl = _bank(1, 128 * 48, 4, [13])
    _check(wl, _gpu_y(wl))


def test_fold_matches_single_stage_pass():
    """R25 (the last stage of odd channels folded into y, orders 8/10/12 here) against the same
    bank with the single-stage passes run (CASC_BANK_FOLD=0): same sums regrouped."""
    wl = _bank(8, 128 * 48, 2, [8, 9, 10, 11, 12, 13, 10, 8])
    y_fold = _gpu_y(wl)
    _check(wl, y_fold)
    y_single = _gpu_y(wl, {"CASC_BANK_FOLD": "0"})
    assert rel(y_fold, y_single) < 2e-6


# ------------------------------------------------------------------ NEXT-3: triangular skip
def test_triangular_skip_bitwise_equal_dense():
    """HiPPO Abar is lower triangular, so are its powers and the pair weights
    Q_k = P_{k+1} P_k; the stage kernel skips the all-zero upper blocks of every K step
    (SURVEY NEXT-3). The skipped products are exact zeros: y must be bitwise the
    dense kernel's (CASC_BANK_TRI=0), for pairs, single stages (fold off) and the exponential
    scheme's triangular Abar, and within 1e-5 of the oracle."""
    for wl, env in ((_bank(8, 128 * 48, 2, ORDERS), {}),
                    (_bank(6, 128 * 48 - 37, 2, [8, 9, 10, 11, 12, 13]), {"CASC_BANK_FOLD": "0"})):
        y_tri = _gpu_y(wl, env or None)
        y_dense = _gpu_y(wl, {**env, "CASC_BANK_TRI": "0"})
        assert np.array_equal(y_tri, y_dense)
        _check(wl, y_tri)


def test_triangular_flag_off_for_dense_abar():
    """A bank whose Abar has entries above the diagonal must run the dense MMAs: one channel with a
    single non-zero upper entry among HiPPO channels; parity with the oracle catches a skipped block."""
    wl = _bank(4, 128 * 32, 2, [9, 10, 11, 12])
    wl.Abar[2][3, 40] = 1e-3                         # breaks the structure of channel 2 only
    _check(wl, _gpu_y(wl))
