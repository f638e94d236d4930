"""Sequence-sharded path on one GPU: R emulated ranks in one process (LocalComm) run the CUDA
step functions casc_seq_*; the result must be bitwise the unsharded run (each output row's
accumulation order does not depend on the shard it lives in) and within tolerance
of the float64 oracle. (Separate processes waiting on each other on one GPU are not used.)"""
import numpy as np
import pytest
import torch

import oracle
from synth import configs as S

pytestmark = pytest.mark.gpu
TOL = {"fp32": 1e-5, "bf16": 2e-2}


@pytest.mark.parametrize("mode", ["bf16", "fp32"])
@pytest.mark.parametrize("R,m,p,q,L,N", [(2, 128, 64, 64, 4096, 8), (4, 64, 64, 64, 2048, 9), (8, 128, 64, 128, 8192, 6),
                                         (2, 64, 64, 64, 256, 0)])
def test_emulated_ranks_bitwise_equal_unsharded(mode, R, m, p, q, L, N):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2411_17729_b200 import seqshard
    from paper_2411_17729_b200.runner import DeviceWorkload
    wl = S.make_random_mimo(m, p, q, L=L, batch=2, N=N, rho=0.97, mode=mode)
    dw = DeviceWorkload(wl)
    dw.step()
    y_full = dw.y.clone()
    Ne = seqshard.effective_order(N, L)
    H = seqshard.shard_H(N, L)
    steps = seqshard.CudaSteps(m, p, q, mode)
    steps.prepare(dw.Abar[0], dw.Bbar, dw.C, dw.D, N, Ne)
    L_loc = L // R
    shards = [seqshard.make_shard(dw.u[:, r * L_loc:(r + 1) * L_loc, :], m, q, H) for r in range(R)]
    seqshard.run(steps, seqshard.LocalComm(), shards, N, L)
    torch.cuda.synchronize()
    y = torch.cat([s.y for s in shards], dim=1)
    assert torch.equal(y, y_full)
    ref = oracle.apply_workload(wl)[0]
    yn = y.float().cpu().double().numpy()
    assert np.linalg.norm(yn - ref) / np.linalg.norm(ref) <= TOL[mode]
