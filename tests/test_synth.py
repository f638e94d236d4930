"""Input-generator checks (`-m "not gpu"`): determinism, windows, storage rounding, config recipes."""
import math

import numpy as np
import torch

from synth import configs as S
from synth import rng


def test_rng_deterministic_and_windowed():
    a = rng.normal(0, 5, 0, 10000)
    b = rng.normal(0, 5, 0, 10000)
    assert np.array_equal(a, b)
    assert np.array_equal(rng.normal(0, 5, 1234, 100), a[1234:1334])
    assert not np.array_equal(rng.normal(1, 5, 0, 100), a[:100])
    assert not np.array_equal(rng.normal(0, 6, 0, 100), a[:100])
    # roughly standard normal
    big = rng.normal(3, 1, 0, 400000)
    assert abs(big.mean()) < 0.01 and abs(big.std() - 1.0) < 0.01


def test_bf16_rounding_matches_torch():
    x = np.random.default_rng(0).standard_normal(100000).astype(np.float32) * 10.0
    x[:4] = [0.0, -0.0, 1e-40, 3.0e38]
    ours = S.bf16_bits_from_f32(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)


def test_workload_windows_consistent():
    wl = S.make_E2(n_ch=3, L=512, batch=2)
    u = wl.u_all()
    assert u.shape == (3, 2, 512, 1)
    assert np.array_equal(wl.u_window(2, 1, 100, 164), u[2, 1, 100:164])
    w = wl.u_window(1, 0, -5, 10)
    assert np.all(w[:5] == 0.0) and np.array_equal(w[5:], u[1, 0, :10])
    st = wl.u_storage()
    assert st.dtype == np.float32 and np.array_equal(st.astype(np.float64), u)


def test_E1_recipe():
    wl = S.make_E1()
    assert (wl.m, wl.p, wl.q, wl.L, wl.batch, int(wl.N[0])) == (16, 1, 1, 4096, 1, 11)
    assert S.spectral_radius(wl.Abar[0]) <= 0.99 + 1e-12
    assert 2 ** (int(wl.N[0]) + 1) >= wl.L


def test_hippo_bank_recipe_small():
    wl = S.make_E2(n_ch=24, L=16384, batch=1)
    d = wl.meta["delta"]
    assert np.all((d >= 1e-3) & (d <= 1e-1))
    assert np.all((wl.N >= 6) & (wl.N <= 13))        # survey estimate [7, 13]
    for c in range(4):
        N = int(wl.N[c])
        P = np.linalg.matrix_power(wl.Abar[c], 2 ** (N + 1))
        assert np.linalg.norm(P, 2) <= 1e-6 or N == 13
        if N > 0 and N < 13:
            Pm = np.linalg.matrix_power(wl.Abar[c], 2 ** N)
            assert np.linalg.norm(Pm, 2) > 1e-6       # minimality
        assert S.spectral_radius(wl.Abar[c]) < 1.0


def test_E3_recipe_small():
    wl = S.make_E3(L=256, batch=1, m=32, p=8)
    ev = np.sort(np.abs(np.linalg.eigvals(wl.Abar[0])))
    assert ev.min() >= 0.5 - 1e-9 and ev.max() <= 0.999 + 1e-9
    assert abs(0.999 ** (2 ** 14) - 7.6e-8) < 0.1e-8     # BASELINE configs[2] "0.999^(2^14) ~ 7.6e-8"


def test_E4_recipe_small():
    wl = S.make_E4(L=4096, batch=1, m=64, p=16)
    assert abs(S.spectral_radius(wl.Abar[0]) - 0.995) < 1e-12
    assert np.all(wl.D == 0.0) and wl.mode == "bf16"
    u = wl.u_all()
    assert np.array_equal(S.round_to_storage(u, "bf16"), u)   # already bf16-exact
    assert math.isfinite(wl.flops_ns())
