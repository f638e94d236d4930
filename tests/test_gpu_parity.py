"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on the same seeded
inputs. Tolerances (BASELINE north_star): relative L2 <= 1e-5 in fp32 mode, <= 2e-2 in bf16
mode, on y and on the state part y - D u (R15); the impulse tail is exactly zero."""
import numpy as np
import pytest
import torch

import oracle
from synth import configs as S

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "bf16": 2e-2}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2411_17729_b200 as pk
    pk.lib()                                 # fails loudly if the library is missing


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def run_gpu(wl, channels=None):
    from paper_2411_17729_b200.runner import DeviceWorkload
    dw = DeviceWorkload(wl, channels=channels)
    dw.step()
    torch.cuda.synchronize()
    return dw.y_f64(), dw


def oracle_y(wl, channels=None):
    chans = range(wl.n_ch) if channels is None else channels
    u = wl.u_all()
    return oracle.apply_workload(wl, u=u, channels=chans), u


def check_parity(wl, channels=None, tol=None):
    tol = TOL[wl.mode] if tol is None else tol
    y_gpu, _ = run_gpu(wl, channels)
    y_ref, u = oracle_y(wl, channels)
    chans = list(range(wl.n_ch)) if channels is None else list(channels)
    assert np.all(np.isfinite(y_gpu))
    e = rel(y_gpu, y_ref)
    Du = np.stack([u[c] @ wl.D[c].T for c in chans])
    es = rel(y_gpu - Du, y_ref - Du)
    assert e <= tol, f"rel err {e:.3e} > {tol}"
    assert es <= tol, f"state-part rel err {es:.3e} > {tol}"
    return e, es


# ------------------------------------------------------------------ powers (a1)
@pytest.mark.parametrize("m,N", [(16, 11), (64, 13), (100, 15), (256, 5)])
def test_powers_fp64_match_oracle(m, N):
    import paper_2411_17729_b200 as pk
    if m == 100:
        Abar, _ = S.trapezoid(S.hippo(100), None, 5e-4)
    else:
        Abar = S.make_random_mimo(m, 1, 1, 8, 1, 0, rho=0.99).Abar[0]
    pw = pk.powers(torch.from_numpy(Abar).cuda(), N, "fp32")
    torch.cuda.synchronize()
    mm = m * m
    hdr = 256                                                   # header padded to 256 B
    p64 = pw.pack[hdr:hdr + (N + 1) * mm * 8].view(torch.float64).reshape(N + 1, m, m).cpu().numpy()
    ref = oracle.powers(Abar, N)
    for k in range(N + 1):
        scale = max(np.max(np.abs(ref[k])), 1e-300)
        assert np.max(np.abs(p64[k] - ref[k])) <= 1e-12 * max(scale, 1.0) * (1 + k)
    if m == 100:   # the paper's pin: (Abar^(2^15))_11 ~ 5.87548e-15
        assert abs(p64[15][0, 0] / 5.87548e-15 - 1) < 2e-5


@pytest.mark.parametrize("m,N,mode", [(64, 13, "fp32"), (256, 9, "bf16"), (100, 15, "fp32")])
def test_powers_norms_match_oracle(m, N, mode):
    """casc_powers_norms: ||P_k||_F for k <= N and the first neglected power P_{N+1} = P_N P_N
    (the planner's truncation indicator) against the oracle's float64 powers."""
    import paper_2411_17729_b200 as pk
    if m == 100:
        Abar, _ = S.trapezoid(S.hippo(100), None, 5e-4)
        Ns = [N]
    else:
        Abar = np.stack([S.make_random_mimo(m, 1, 1, 8, 1, 0, rho=0.99, seed=s).Abar[0] for s in range(3)])
        Ns = [N, N - 2, 0]
    A = torch.from_numpy(np.ascontiguousarray(Abar)).cuda()
    pw = pk.powers(A, Ns, mode)
    got = pk.powers_norms(pw)
    for s, Ns_ in enumerate(Ns):
        ref = oracle.powers(Abar if Abar.ndim == 2 else Abar[s], Ns_)
        want = [np.linalg.norm(P) for P in ref] + [np.linalg.norm(ref[-1] @ ref[-1])]
        assert np.allclose(got[s, :Ns_ + 2], want, rtol=1e-12, atol=1e-300), (s, got[s], want)
        assert np.all(np.isnan(got[s, Ns_ + 2:]))


# ------------------------------------------------------------------ configs (scaled to oracle-sized runs)
def test_E1_full_size():
    e, es = check_parity(S.make_E1())
    print(f"E1 rel {e:.2e} state {es:.2e}")


def test_E2_reduced_bank():
    wl = S.make_E2(n_ch=12, L=4096, batch=2)
    check_parity(wl)


def test_E2_full_shape_sampled_channels():
    """Full E2 sizes (256 ch, L=16384, batch 4) on the GPU; oracle on 6 channels spanning N."""
    wl = S.make_E2()
    y_gpu, _ = run_gpu(wl)
    order = np.argsort(wl.N)
    pick = [int(order[0]), int(order[len(order) // 3]), int(order[len(order) // 2]),
            int(order[-1]), 0, wl.n_ch - 1]
    y_ref, u = oracle_y(wl, pick)
    for i, c in enumerate(pick):
        e = rel(y_gpu[c], y_ref[i])
        es = rel(y_gpu[c] - u[c] * wl.D[c, 0, 0], y_ref[i] - u[c] * wl.D[c, 0, 0])
        assert e <= 1e-5 and es <= 1e-5, (c, int(wl.N[c]), e, es)


def test_E3_reduced_mimo():
    wl = S.make_E3(L=4096, batch=2)
    check_parity(wl)


def test_E4_reduced_bf16():
    wl = S.make_E4(L=4096, batch=1, N=11)
    check_parity(wl)


@pytest.mark.parametrize("m,p,q,L,batch,N", [(128, 64, 64, 1000, 3, 6), (64, 64, 64, 300, 2, 0),
                                              (256, 128, 64, 4096, 2, 11), (192, 64, 128, 129, 1, 3),
                                              (128, 64, 64, 2, 2, 5), (128, 64, 64, 1, 1, 2),
                                              # Ne = 1 (fused first step only), Ne = 2 (Krylov head,
                                              # no streaming stage), L = 5 (Ne capped at 2 by L)
                                              (128, 64, 64, 500, 2, 1), (128, 64, 64, 500, 2, 2),
                                              (64, 64, 64, 5, 3, 6)])
@pytest.mark.parametrize("mode", ["bf16", "fp32"])
def test_mimo_tensor_core_path(m, p, q, L, batch, N, mode):
    """MIMO systems with m, p, q multiples of 64 take the TMA + tcgen05 GEMM path
    (kind::f16 in bf16 mode, 3xTF32 in fp32 mode): the Krylov head (four lags of u) for Ne >= 2,
    the fused first step for Ne = 1, y directly for Ne = 0."""
    wl = S.make_random_mimo(m, p, q, L=L, batch=batch, N=N, rho=0.98, mode=mode)
    check_parity(wl)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
def test_random_mimo_ragged(mode):
    wl = S.make_random_mimo(48, 5, 7, L=1000, batch=3, N=6, mode=mode)
    check_parity(wl)


# ------------------------------------------------------------------ edge cases
@pytest.mark.parametrize("L", [1, 2, 3, 4, 5, 63, 64, 65, 127, 128, 129, 1023, 1024, 1025])
def test_lengths_and_skipped_stages(L):
    wl = S.make_random_mimo(16, 2, 3, L=L, batch=2, N=12, mode="fp32")
    check_parity(wl)


@pytest.mark.parametrize("m", [16, 32, 64])
@pytest.mark.parametrize("L,N", [(1, 3), (2, 0), (3, 1), (100, 12), (129, 7), (300, 8), (1000, 9), (2049, 11)])
def test_bank_tensor_core_path_edges(m, L, N):
    """SISO systems take the tcgen05 bank path (Krylov head, streaming stages, fused tail)."""
    wl = S.make_random_mimo(m, 1, 1, L=L, batch=2, N=N, rho=0.97, mode="fp32")
    check_parity(wl)


def test_bank_channel_waves_bounded_memory():
    """A workspace for ~3 channels forces the 10-channel bank through 4 waves; results must be
    bitwise those of the single-wave run (each wave is an independent bank)."""
    import paper_2411_17729_b200 as pk
    from paper_2411_17729_b200.runner import DeviceWorkload
    wl = S.make_E2(n_ch=10, L=3000, batch=2)
    one = pk.bank_workspace_bytes(1, wl.m, wl.L, wl.batch, int(wl.N.max()), "fp32")
    dw = DeviceWorkload(wl, ws_budget=3 * one + 4096)
    dw.step()
    torch.cuda.synchronize()
    y_w = dw.y_f64()
    y_full, _ = run_gpu(wl)
    assert np.array_equal(y_w, y_full)
    y_ref, _ = oracle_y(wl)
    assert rel(y_w, y_ref) < 1e-5


def test_bank_mixed_orders_and_ragged_length():
    """Channels with N from 0 to 13 in one bank, L not a multiple of the 128-step tile."""
    wl = S.make_E2(n_ch=14, L=3000, batch=3)
    wl.N[:] = np.arange(14)
    check_parity(wl)


@pytest.mark.parametrize("N", [0, 1, 2, 7])
def test_small_N_and_zero_D(N):
    wl = S.make_random_mimo(32, 3, 2, L=300, batch=1, N=N, zero_D=True)
    check_parity(wl)


def test_impulse_exact_zero_tail():
    """T10 on the GPU: the cascade is a polynomial of degree 2^(N+1)-1, so an impulse at l=0
    produces exactly 0.0 for l >= 2^(N+1) (0 + P 0 = 0 in any arithmetic)."""
    import paper_2411_17729_b200 as pk
    wl = S.make_random_mimo(16, 1, 1, L=600, batch=1, N=5, zero_D=True)
    u = torch.zeros((1, 600, 1), dtype=torch.float32, device="cuda")
    u[0, 0, 0] = 1.0
    pw = pk.powers(torch.from_numpy(wl.Abar[0]).cuda(), 5)
    y = pk.apply(pw, torch.from_numpy(wl.Bbar[0]).cuda(), torch.from_numpy(wl.C[0]).cuda(), None, u)
    yc = y.cpu().double().numpy()[0, :, 0]
    assert np.all(yc[64:] == 0.0)
    assert yc[63] != 0.0
    ref = oracle.cascade(oracle.powers(wl.Abar[0], 5), wl.Bbar[0], wl.C[0], np.zeros((1, 1)),
                         u.cpu().double().numpy(), 5)[0, :, 0]
    assert rel(yc, ref) < 1e-5


def test_effective_stages_reported():
    import paper_2411_17729_b200 as pk
    wl = S.make_random_mimo(8, 1, 1, L=100, batch=1, N=12)
    pw = pk.powers(torch.from_numpy(wl.Abar[0]).cuda(), 12)
    u = torch.randn((1, 100, 1), device="cuda")
    _, eff = pk.apply(pw, torch.from_numpy(wl.Bbar[0]).cuda(), torch.from_numpy(wl.C[0]).cuda(),
                      torch.from_numpy(wl.D[0]).cuda(), u, return_stages=True)
    assert eff == oracle.effective_stages(100, 12) == 7


def test_run_host_matches_device_path():
    import paper_2411_17729_b200 as pk
    from paper_2411_17729_b200.runner import storage_to_torch
    wl = S.make_E2(n_ch=5, L=2048, batch=2)
    y_dev, _ = run_gpu(wl)
    n = wl.n_ch
    u_h = storage_to_torch(wl.u_storage(), "fp32").reshape(n, wl.batch, wl.L, 1).pin_memory()
    y_h = torch.empty_like(u_h).pin_memory()
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    ws = torch.empty(pk.run_host_bytes(n, wl.m, 1, 1, wl.L, wl.batch, int(wl.N.max()), "fp32"),
                     dtype=torch.uint8, device="cuda")
    pk.run_host(f(wl.Abar), f(wl.Bbar), f(wl.C), f(wl.D), u_h, y_h, list(wl.N), "fp32", ws)
    assert np.array_equal(y_h.double().numpy(), y_dev)


def test_determinism_bitwise():
    wl = S.make_E2(n_ch=4, L=2048, batch=2)
    a, _ = run_gpu(wl)
    b, _ = run_gpu(wl)
    assert np.array_equal(a, b)


def test_determinism_full_size_E2_under_load():
    """Repeated full-size E2 steps on one resident workload are bitwise identical. A race between
    the bank pass's roles (e.g. an accumulator released before every reader is done) shows up here
    as a handful of differing outputs in some runs (an early release failed 1 run in 3)."""
    from paper_2411_17729_b200.runner import DeviceWorkload
    dw = DeviceWorkload(S.make_E2())
    dw.step()
    torch.cuda.synchronize()
    ref = dw.y_f64()
    for _ in range(6):
        dw.step()
        torch.cuda.synchronize()
        y = dw.y_f64()
        assert np.array_equal(y, ref), f"{int((y != ref).sum())} outputs differ between identical runs"


@pytest.mark.parametrize("mode", ["bf16", "fp32"])
def test_run_host_mimo_single_chunk_bitwise(mode):
    """casc_run_host for one MIMO system with a small input (1.3 MB: one batch chunk, copies on the
    copy streams): y is bitwise the device-resident path's. The multi-chunk runs are in
    tests/test_gpu_e2e_paths.py."""
    import paper_2411_17729_b200 as pk
    from paper_2411_17729_b200.runner import storage_to_torch
    wl = S.make_random_mimo(128, 64, 64, L=1000, batch=5, N=8, rho=0.97, mode=mode)
    y_dev, _ = run_gpu(wl)
    u_h = storage_to_torch(wl.u_storage(), mode).reshape(1, wl.batch, wl.L, wl.p).pin_memory()
    y_h = torch.empty((1, wl.batch, wl.L, wl.q), dtype=u_h.dtype).pin_memory()
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    ws = torch.empty(pk.run_host_bytes(1, wl.m, wl.p, wl.q, wl.L, wl.batch, int(wl.N.max()), mode),
                     dtype=torch.uint8, device="cuda")
    pk.run_host(f(wl.Abar), f(wl.Bbar), f(wl.C), f(wl.D), u_h, y_h, list(wl.N), mode, ws)
    assert np.array_equal(y_h.float().double().numpy(), y_dev)


# ------------------------------------------------------------------ NEXT-4: exponential discretisation
def test_exponential_scheme_bank():
    """HiPPO channels discretised by the exponential zero-order hold (DESIGN.md
    R27) through the same bank path: N_c planned from the new Abar, parity at 1e-5."""
    wl = S.make_E2(n_ch=12, L=4096, batch=2, scheme="exponential")
    e, es = check_parity(wl)
    print(f"E2x rel {e:.2e} state {es:.2e}")


@pytest.mark.parametrize("m", [16, 32, 64])
def test_bf16_siso_bank_on_tensor_cores(m):
    """bf16 storage of a SISO bank: the library converts u to fp32, runs the tensor-core bank path
    (Krylov head, stage passes, fused output) and rounds y once to bf16; parity at the bf16 bound,
    and the y is the fp32 path's y rounded to bf16 (RN-even), bit for bit."""
    import paper_2411_17729_b200 as pk
    wl = S.make_E2(n_ch=6, L=2048, batch=2, mode="bf16") if m == 64 else \
        S.make_random_mimo(m, 1, 1, L=1500, batch=2, N=9, rho=0.97, mode="bf16")
    check_parity(wl)
    pk.profile_reset()
    pk.profile_enable(True)
    y_bf, _ = run_gpu(wl)
    torch.cuda.synchronize()
    prof = pk.profile_read()
    pk.profile_enable(False)
    assert "direct" not in prof and "stage" not in prof, prof        # no CUDA-core GEMM classes
    from paper_2411_17729_b200.runner import DeviceWorkload
    wl32 = S.Workload(**{**wl.__dict__, "mode": "fp32"})
    u32 = S.bf16_bits_to_f64(wl.u_storage()).astype(np.float32)       # the same (bf16-exact) input values
    dw32 = DeviceWorkload(wl32, u_host=u32)
    dw32.step()
    torch.cuda.synchronize()
    y32 = dw32.y_f64()
    y32_bf = torch.from_numpy(y32).float().to(torch.bfloat16).double().numpy()
    assert np.array_equal(y_bf, y32_bf)


@pytest.mark.parametrize("m,p", [(256, 64), (512, 128), (1024, 256)])
def test_fp32_headroom_grows_with_K(m, p):
    """3xTF32 accuracy vs the contraction length: the fp32 tensor-core accumulator truncates at
    every MMA, so the main chain's error grows with K / 8. With one main accumulator
    the state part measured 1.05e-5 at m = 1024 (K = 1024); contractions longer than 512 therefore
    spread the main chain over three accumulators (mimo_tc3.cu PCfg SPLIT). All three sizes must
    meet the fp32 bound 1e-5."""
    wl = S.make_random_mimo(m, p, p, L=1024, batch=2, N=9, rho=0.98, mode="fp32", seed=m)
    e, es = check_parity(wl)
    print(f"fp32 m={m}: rel {e:.2e} state {es:.2e} (bound 1e-5)")


# ------------------------------------------------------------------ empty inputs (include/cascade.h)
@pytest.mark.parametrize("L,batch", [(0, 3), (200, 0)])
def test_empty_signals_through_the_python_api(L, batch):
    """An empty signal (L = 0 or batch = 0) is a valid call: y comes back empty, nothing launches,
    and a non-empty call on the same pack afterwards is unaffected."""
    import paper_2411_17729_b200 as pk
    rng = np.random.default_rng(11)
    m, p, q, N = 64, 64, 64, 5
    Ab = torch.from_numpy(0.5 * rng.standard_normal((m, m)) / np.sqrt(m)).cuda()
    Bb = torch.from_numpy(rng.standard_normal((m, p))).cuda()
    C = torch.from_numpy(rng.standard_normal((q, m))).cuda()
    pw = pk.powers(Ab, N, "fp32")
    u = torch.empty((batch, L, p), dtype=torch.float32, device="cuda")
    y, eff = pk.apply(pw, Bb, C, None, u, return_stages=True)
    torch.cuda.synchronize()
    assert tuple(y.shape) == (batch, L, q) and pk.last_launch_count() == 0
    assert eff == sum(1 for k in range(N + 1) if (1 << k) < L)
    # bank: 3 channels, empty signals
    Abk = torch.from_numpy(np.stack([0.3 * np.eye(m)] * 3)).cuda()
    pwb = pk.powers(Abk, [2, 3, 4], "fp32")
    ub = torch.empty((3, batch, L), dtype=torch.float32, device="cuda")
    yb = pk.apply_bank(pwb, torch.ones((3, m), dtype=torch.float64, device="cuda"),
                       torch.ones((3, m), dtype=torch.float64, device="cuda"), None, ub)
    torch.cuda.synchronize()
    assert tuple(yb.shape) == (3, batch, L)
    # host entry point
    uh = torch.empty((1, batch, L, p), dtype=torch.float32)
    yh = torch.empty((1, batch, L, q), dtype=torch.float32)
    pk.run_host(Ab.cpu()[None], Bb.cpu()[None], C.cpu()[None], None, uh, yh, N, "fp32",
                torch.empty(0, dtype=torch.uint8, device="cuda"))
    # the same pack on a real signal still matches the oracle
    u2 = torch.from_numpy(rng.standard_normal((2, 300, p)).astype(np.float32)).cuda()
    y2 = pk.apply(pw, Bb, C, None, u2)
    torch.cuda.synchronize()
    P = oracle.powers(Ab.cpu().numpy(), N)
    yref = oracle.cascade(P, Bb.cpu().numpy(), C.cpu().numpy(), np.zeros((q, p)), u2.cpu().numpy().astype(np.float64), N)
    assert rel(y2.cpu().numpy().astype(np.float64), yref) <= TOL["fp32"]
