"""GPU checks of the m = 64 bank head on the fp16 tensor path (R33): its operands are
split hi + lo in fp16 after exact power-of-two scaling (per Krylov-weight column, per 128-step
tile), so fp16's narrow exponent range must never show. Two properties pin that:

- scale equivariance: the map u -> y is linear and every kernel on the path computes in binary
  floating point, so scaling u (or Bbar) by 2^k must scale y by exactly 2^k, bit for bit, far
  outside fp16's range (|k| up to 60);
- a sequence whose first half is ~1e-30 and second half ~1e+30 keeps fp32 accuracy on each half
  separately (causality: the first half's outputs depend on the first half's inputs only), against
  the float64 oracle, with the same 1e-5 bound as every fp32 parity test."""
import numpy as np
import pytest
import torch

import oracle
from synth import configs as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2411_17729_b200 as pk
    pk.lib()


def _bank(n_ch=6, L=3000, batch=2):
    wl = S.make_E2(n_ch=n_ch, L=L, batch=batch)
    wl.N[:] = np.array([7, 8, 9, 10, 11, 11][:n_ch])
    return wl


def _run(wl, u64, Bbar=None):
    import paper_2411_17729_b200 as pk
    c = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    n = wl.n_ch
    pw = pk.powers(c(wl.Abar), [int(x) for x in wl.N], "fp32")
    u = c(u64[..., 0].astype(np.float32))
    B = c((wl.Bbar if Bbar is None else Bbar).reshape(n, wl.m))
    y = pk.apply_bank(pw, B, c(wl.C.reshape(n, wl.m)), c(wl.D.reshape(n)), u)
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("k", [-60, -24, 17, 60])
def test_head_scale_equivariance_in_u(k):
    wl = _bank()
    u = wl.u_all()
    y0 = _run(wl, u)
    yk = _run(wl, u * 2.0 ** k)
    assert np.all(np.isfinite(y0))
    assert np.array_equal(yk.astype(np.float64), y0.astype(np.float64) * 2.0 ** k)


@pytest.mark.parametrize("k", [-40, 40])
def test_head_scale_equivariance_in_Bbar(k):
    """Bbar scales the Krylov weights A^j Bbar, i.e. the per-column fp16 scales of the head; D is
    scaled too so that the whole output scales."""
    wl = _bank()
    u = wl.u_all()
    y0 = _run(wl, u)
    wl2 = _bank()
    wl2.D = wl.D * 2.0 ** k
    yk = _run(wl2, u, Bbar=wl.Bbar * 2.0 ** k)
    assert np.array_equal(yk.astype(np.float64), y0.astype(np.float64) * 2.0 ** k)


def test_head_wide_dynamic_range_per_half():
    wl = _bank(n_ch=4, L=4096, batch=2)
    u = wl.u_all().copy()
    h = wl.L // 2
    u[:, :, :h] *= 1e-30
    u[:, :, h:] *= 1e30
    u = u.astype(np.float32).astype(np.float64)        # what the GPU reads
    y = _run(wl, u).astype(np.float64)[..., None]
    ref = oracle.apply_workload(wl, u=u, channels=range(wl.n_ch))
    for sl in (slice(0, h), slice(h, wl.L)):
        a, b = y[:, :, sl], ref[:, :, sl]
        e = float(np.linalg.norm(a - b) / np.linalg.norm(b))
        assert e <= 1e-5, (sl, e)
