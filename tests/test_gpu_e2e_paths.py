"""GPU parity of the host-buffer entry casc_run_host in the configurations bench.py's e2e leg runs,
plus a per-row bf16 check of an E4-shaped system.

The map y = H_N u must not depend on how the work is cut into input chunks or channel waves
(each sequence's cascade is independent of the others), so every chunked or
waved host-buffer run is compared bitwise with the device-resident path and with the float64
oracle. The device workspace is filled with NaN bytes before each call and every call passes a
different input, so an output computed from a stale or half-copied input cannot pass.

Variants that need a different library setting (CASC_MIMO_CHUNKS) run in a subprocess: the
library reads its settings once per process."""
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
TOL = {"fp32": 1e-5, "bf16": 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2411_17729_b200 as pk
    pk.lib()


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def _host(a):
    return torch.from_numpy(np.ascontiguousarray(a))


def _device_y(wl, u_store):
    """y of the device-resident path (runner.DeviceWorkload) on the given storage input."""
    from paper_2411_17729_b200.runner import DeviceWorkload
    dw = DeviceWorkload(wl, u_host=u_store)
    dw.step()
    torch.cuda.synchronize()
    return dw.y_f64()


def _run_host(wl, u_store, ws_bytes=None, pinned=True):
    """casc_run_host on pinned (or pageable) host buffers with a NaN-filled device workspace."""
    import paper_2411_17729_b200 as pk
    from paper_2411_17729_b200.runner import storage_to_torch
    n = wl.n_ch
    u_h = storage_to_torch(u_store, wl.mode).reshape(n, wl.batch, wl.L, wl.p).clone()
    y_h = torch.full((n, wl.batch, wl.L, wl.q), float("nan"), dtype=u_h.dtype)
    if pinned:
        u_h, y_h = u_h.pin_memory(), y_h.pin_memory()
    need = pk.run_host_bytes(n, wl.m, wl.p, wl.q, wl.L, wl.batch, int(wl.N.max()), wl.mode)
    ws = torch.empty(need if ws_bytes is None else ws_bytes, dtype=torch.uint8, device="cuda")
    ws.fill_(0xFF)                                   # NaN in every float lane
    torch.cuda.synchronize()
    D_h = _host(wl.D) if np.any(wl.D) else None
    pk.run_host(_host(wl.Abar), _host(wl.Bbar), _host(wl.C), D_h, u_h, y_h, list(wl.N), wl.mode, ws)
    return y_h.float().double().numpy()


def _inputs(wl, k):
    """Storage input number k: the workload's u with a different seed per call."""
    wl2 = S.Workload(**{**wl.__dict__, "u_seed": wl.u_seed + 1000 * k})
    return wl2, wl2.u_storage()


def _oracle(wl):
    u = wl.u_all()
    return oracle.apply_workload(wl, u=u, channels=range(wl.n_ch))


# ------------------------------------------------------------------ banks: channel waves
def test_bank_run_host_three_waves_bitwise():
    """A device workspace that holds one third of the bank: the pipelined host path runs >= 3 waves
    (each wave's input copy overlapping the previous wave's compute); two calls with different
    inputs, each bitwise equal to the device-resident path and within 1e-5 of the oracle."""
    import paper_2411_17729_b200 as pk
    wl = S.make_E2(n_ch=9, L=4096, batch=2, seed=5)
    n = wl.n_ch
    full = pk.run_host_bytes(n, wl.m, 1, 1, wl.L, wl.batch, int(wl.N.max()), "fp32")
    per_ch = pk.bank_workspace_bytes(1, wl.m, wl.L, wl.batch, int(wl.N.max()), "fp32")
    apply_full = pk.bank_workspace_bytes(n, wl.m, wl.L, wl.batch, int(wl.N.max()), "fp32")
    ws_bytes = full - apply_full + 3 * per_ch + (per_ch // 2)     # three channels per wave
    for k in range(2):
        wlk, u = _inputs(wl, k)
        y_host = _run_host(wlk, u, ws_bytes)
        y_dev = _device_y(wlk, u)
        assert np.array_equal(y_host, y_dev), f"call {k}: host-buffer waves differ from the device path"
        assert rel(y_host, _oracle(wlk)) <= TOL["fp32"]


def test_bank_run_host_full_size_input_lands_before_use():
    """E2 at full size (268 MB of input, one wave): the head must wait for the input copy. With a
    NaN-filled workspace and a fresh input per call, a head that ran ahead of the copy would read
    NaN or the previous call's input."""
    wl = S.make_E2()
    for k in range(2):
        wlk, u = _inputs(wl, k)
        y_host = _run_host(wlk, u)
        assert np.all(np.isfinite(y_host))
        y_dev = _device_y(wlk, u)
        assert np.array_equal(y_host, y_dev), f"call {k}"


def test_bank_run_host_pageable_buffers_bitwise():
    """Pageable host buffers: the bank path cannot store the last emission straight into y_h (it is
    not device-mapped) and copies it out instead; both runs, over >= 3 ramped waves, are bitwise
    equal to the device-resident path."""
    import paper_2411_17729_b200 as pk
    wl = S.make_E2(n_ch=24, L=4096, batch=2, seed=7)
    n = wl.n_ch
    full = pk.run_host_bytes(n, wl.m, 1, 1, wl.L, wl.batch, int(wl.N.max()), "fp32")
    per_ch = pk.bank_workspace_bytes(1, wl.m, wl.L, wl.batch, int(wl.N.max()), "fp32")
    apply_full = pk.bank_workspace_bytes(n, wl.m, wl.L, wl.batch, int(wl.N.max()), "fp32")
    ws_bytes = full - apply_full + 8 * per_ch + (per_ch // 2)     # eight channels per wave
    wlk, u = _inputs(wl, 3)
    y_dev = _device_y(wlk, u)
    for pinned in (False, True):
        y_host = _run_host(wlk, u, ws_bytes, pinned=pinned)
        assert np.array_equal(y_host, y_dev), f"pinned={pinned}"


# ------------------------------------------------------------------ MIMO: batch chunks
def _chunked_y(case, chunks):
    out = os.path.join("/tmp", f"chunk_y_{os.getpid()}_{chunks}.npy")
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r})
from test_gpu_e2e_paths import _mimo, _inputs, _run_host
wl, u = _inputs(_mimo(*{tuple(case)!r}), 1)
np.save({out!r}, _run_host(wl, u))
"""
    env = dict(os.environ, CASC_MIMO_CHUNKS=str(chunks))
    subprocess.run([sys.executable, "-c", code], env=env, check=True, timeout=900, cwd=ROOT)
    y = np.load(out)
    os.remove(out)
    return y


def _mimo(m, p, q, L, batch, N, mode):
    return S.make_random_mimo(m, p, q, L=L, batch=batch, N=N, rho=0.97, mode=mode, seed=11)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
@pytest.mark.parametrize("chunks", [3, 5])
def test_run_host_mimo_chunks_bitwise(mode, chunks):
    """casc_run_host for one MIMO system in 3 or 5 batch chunks (CASC_MIMO_CHUNKS, the path the
    E3/E4 e2e numbers use: inputs above 64 MiB are cut into one chunk per 64 MiB): bitwise equal to
    the device-resident path on the same input, and within tolerance of the oracle. A ragged split
    (batch 7 into 3 or 5 chunks) makes the chunks unequal."""
    case = (128, 64, 64, 1500, 7, 9, mode)
    y_chunked = _chunked_y(case, chunks)
    wl, u = _inputs(_mimo(*case), 1)
    y_dev = _device_y(wl, u)
    assert np.array_equal(y_chunked, y_dev)
    assert rel(y_chunked, _oracle(wl)) <= TOL[mode]


# ------------------------------------------------------------------ bf16: every row
def test_bf16_every_row_E4_shape():
    """E4's shape (m = 1024, p = q = 256, bf16 storage, fp32 accumulate, rho = 0.995, N = 11) at
    L = 4096, batch 2: every output row (one time step of one sequence, a q-vector) is checked, not
    just the global norm. Bound per row: ||e_row|| <= 2e-2 max(||y_row||, 1e-2 median_row ||y||);
    the floor keeps rows near l = 0 (few inputs seen) from being judged on a tiny norm."""
    wl = S.make_E4(L=4096, batch=2)
    u = wl.u_storage()
    y = _device_y(wl, u)[0]                                     # [batch][L][q]
    ref = _oracle(wl)[0]
    assert np.all(np.isfinite(y))
    err = np.linalg.norm(y - ref, axis=-1)
    nrm = np.linalg.norm(ref, axis=-1)
    floor = 1e-2 * np.median(nrm)
    worst = float(np.max(err / np.maximum(nrm, floor)))
    print(f"E4-shape bf16: global rel {rel(y, ref):.3e}, worst row {worst:.3e}")
    assert worst <= TOL["bf16"], worst
    assert rel(y, ref) <= TOL["bf16"]


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_run_host_mimo_time_windows_bitwise(mode):
    """Single-sequence first and last chunks run as 8 time windows (inputs [r0 - Hu, r1) for outputs
    [r0, r1), Hu = 2^(Ne+1) - 1: exact by the window property, pin T14), so the
    first window's compute starts before the chunk's whole input landed and the last chunk's output
    leaves window by window. Every kept row is computed by the same operations: bitwise the
    device-resident path, and within tolerance of the oracle."""
    case = (128, 64, 64, 8192, 3, 5, mode)             # Ne = 5: Hu = 63, windows of 1024 rows
    y_win = _chunked_y(case, 3)                        # 3 chunks of one sequence each
    wl, u = _inputs(_mimo(*case), 1)
    y_dev = _device_y(wl, u)
    assert np.array_equal(y_win, y_dev)
    assert rel(y_win, _oracle(wl)) <= TOL[mode]



def test_bank_run_host_bf16_bitwise():
    """casc_run_host for a bf16 SISO bank (fp32 tensor-core bank path on converted copies, serial
    host path): bitwise the device-resident path, within the bf16 bound of the oracle."""
    wl = S.make_E2(n_ch=5, L=2048, batch=2, seed=9, mode="bf16")
    for k in range(2):
        wlk, u = _inputs(wl, k)
        y_host = _run_host(wlk, u)
        assert np.array_equal(y_host, _device_y(wlk, u))
        assert rel(y_host, _oracle(wlk)) <= TOL["bf16"]
