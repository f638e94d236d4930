"""GPU self-test of the tcgen05 building block (UMMA descriptors, TMEM, shifted A operand)."""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def tf32_trunc(x):
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def tf32_rna(x):
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x1000)) & np.uint64(0xFFFFE000)
    return b.astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("off", [0, 1, 3, 8, 13])
@pytest.mark.parametrize("prep", [0, 1, 2])
def test_umma_tf32_interleaved_layout(prep, off):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2411_17729_b200 import _lib
    L = _lib.lib()
    g = np.random.default_rng(prep * 100 + off)
    A = g.standard_normal((144, 64)).astype(np.float32)
    B = g.standard_normal((64, 64)).astype(np.float32)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dD = torch.zeros((128, 64), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    rc = L.casc_selftest_umma(prep, off, ctypes.c_void_p(dA.data_ptr()), ctypes.c_void_p(dB.data_ptr()),
                              ctypes.c_void_p(dD.data_ptr()), ctypes.c_void_p(st))
    assert rc == 0
    torch.cuda.synchronize()
    D = dD.cpu().numpy().astype(np.float64)
    conv = tf32_rna if prep == 2 else tf32_trunc
    ref = conv(A[off:off + 128]).astype(np.float64) @ conv(B).astype(np.float64).T
    err = np.max(np.abs(D - ref)) / np.max(np.abs(ref))
    assert err < 1e-6, err
    if prep == 0:
        # raw fp32 operands behave as truncated tf32 (the low 13 mantissa bits are ignored)
        print("raw-vs-trunc max abs diff", np.max(np.abs(D - ref)))
