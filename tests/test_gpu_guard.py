"""Out-of-bounds write checks (compute-sanitizer is unavailable on this GPU pool): every output is
a view at the front of a larger allocation filled with a sentinel; after the call the bytes past
the view must be untouched. Ragged lengths exercise the partial-tile TMA stores."""
import numpy as np
import pytest
import torch

from synth import configs as S

pytestmark = pytest.mark.gpu


def _padded(shape, dtype, pad=1 << 16):
    n = int(np.prod(shape))
    buf = torch.full((n + pad,), float("nan"), dtype=dtype, device="cuda")
    return buf, buf[:n].view(*shape)


@pytest.mark.parametrize("mode", ["fp32", "bf16"])
@pytest.mark.parametrize("L", [129, 1000, 4097])
def test_mimo_output_guard_band(mode, L):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_2411_17729_b200 as pk
    wl = S.make_random_mimo(128, 64, 64, L=L, batch=3, N=9, mode=mode)
    from paper_2411_17729_b200.runner import DeviceWorkload
    dw = DeviceWorkload(wl)
    pw = pk.powers(dw.Abar, 9, mode)
    buf, y = _padded((3, L, 64), pk.STORAGE[pk.MODES[mode]])
    pk.apply(pw, dw.Bbar, dw.C, dw.D, dw.u, y=y)
    torch.cuda.synchronize()
    assert torch.isnan(buf[y.numel():]).all()
    assert not torch.isnan(y).any()


@pytest.mark.parametrize("L", [129, 3000])
def test_bank_output_guard_band(L):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    import paper_2411_17729_b200 as pk
    from paper_2411_17729_b200.runner import DeviceWorkload
    wl = S.make_E2(n_ch=6, L=L, batch=2)
    dw = DeviceWorkload(wl)
    pw = pk.powers(dw.Abar, [int(x) for x in wl.N], "fp32")
    buf, y = _padded((6, 2, L), torch.float32)
    pk.apply_bank(pw, dw.Bbar, dw.C, dw.D, dw.u, y=y)
    torch.cuda.synchronize()
    assert torch.isnan(buf[y.numel():]).all()
    assert not torch.isnan(y).any()
