"""Small runs of every kernel family, for compute-sanitizer (one tool per invocation)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import configs as S
from paper_2411_17729_b200.runner import DeviceWorkload
from paper_2411_17729_b200 import seqshard

cases = [S.make_E2(n_ch=5, L=1000, batch=2),                                  # bank: head, stage, tail
         S.make_random_mimo(16, 1, 1, L=300, batch=1, N=9),                     # bank m=16 (rp stage)
         S.make_random_mimo(128, 64, 64, L=700, batch=2, N=9, mode="bf16"),     # MIMO bf16 GEMM
         S.make_random_mimo(128, 64, 128, L=700, batch=2, N=9, mode="fp32"),    # MIMO 3xTF32 GEMM
         S.make_random_mimo(48, 5, 7, L=200, batch=2, N=5, mode="fp32")]        # SIMT GEMM
for wl in cases:
    dw = DeviceWorkload(wl)
    dw.step()
    torch.cuda.synchronize()
    print(wl.name, "ok", flush=True)
wl = S.make_random_mimo(64, 64, 64, L=1024, batch=2, N=7, mode="bf16")
dw = DeviceWorkload(wl)
steps = seqshard.CudaSteps(64, 64, 64, "bf16")
steps.prepare(dw.Abar[0], dw.Bbar, dw.C, dw.D, 7, seqshard.effective_order(7, 1024))
H = seqshard.shard_H(7, 1024)
shards = [seqshard.make_shard(dw.u[:, r * 256:(r + 1) * 256, :], 64, 64, H) for r in range(4)]
seqshard.run(steps, seqshard.LocalComm(), shards, 7, 1024)
torch.cuda.synchronize()
print("seqshard ok")
