"""Sequence sharding: the halo-exchange driver (paper_2411_17729_b200/seqshard.py)
checked on CPU. The per-shard steps here are a float64 restatement of the four step contracts of
include/cascade.h (casc_seq_first / stage / last) written in this test, so the driver's halo
bookkeeping and the real torch.distributed exchange (gloo, world_size 2) are verified without a
GPU; the result must equal the unsharded float64 oracle."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from synth import configs as S
from paper_2411_17729_b200 import seqshard


class F64Steps:
    """Step contracts of casc_seq_* in float64 torch (test-side)."""

    def __init__(self, Abar, Bbar, C, D, N, Ne):
        self.P = [torch.from_numpy(x) for x in oracle.powers(Abar, max(N, 0))]
        Ab, Bb, Cm = torch.from_numpy(Abar), torch.from_numpy(Bbar), torch.from_numpy(C)
        Dm = torch.zeros((C.shape[0], Bbar.shape[1]), dtype=torch.float64) if D is None else torch.from_numpy(D)
        self.Bb, self.AB = Bb, Ab @ Bb
        self.C, self.CP, self.D = Cm, Cm @ self.P[Ne], Dm
        self.CBD, self.CAB = Cm @ Bb + Dm, Cm @ (Ab @ Bb)

    def first(self, sh, H):
        u = sh.u_ext
        sh.Va[:, H:, :] = u[:, 1:] @ self.Bb.T + u[:, :-1] @ self.AB.T

    def stage(self, k, sh, src, dst, H):
        L = sh.y.shape[1]
        s = 1 << k
        dst[:, H:, :] = src[:, H:, :] + src[:, H - s:H - s + L, :] @ self.P[k].T

    def last(self, Ne, sh, V, H):
        u = sh.u_ext
        if Ne == 0:
            sh.y[:] = u[:, 1:] @ self.CBD.T + u[:, :-1] @ self.CAB.T
            return
        L = sh.y.shape[1]
        s = 1 << Ne
        sh.y[:] = V[:, H:, :] @ self.C.T + V[:, H - s:H - s + L, :] @ self.CP.T + u[:, 1:] @ self.D.T


def _system(L, N, seed=3):
    wl = S.make_random_mimo(6, 2, 3, L=L, batch=2, N=N, rho=0.97, seed=seed)
    u = torch.from_numpy(wl.u_all()[0])
    return wl, u


@pytest.mark.parametrize("R,L,N", [(4, 256, 5), (2, 100, 3), (4, 64, 4), (3, 90, 0), (2, 2, 3)])
def test_local_emulated_ranks_match_oracle(R, L, N):
    wl, u = _system(L, N)
    Ne = seqshard.effective_order(N, L)
    H = seqshard.shard_H(N, L)
    L_loc = L // R
    if Ne > 0 and (1 << Ne) > L_loc:
        pytest.skip("halo longer than a shard")
    steps = F64Steps(wl.Abar[0], wl.Bbar[0], wl.C[0], wl.D[0], N, Ne)
    shards = [seqshard.make_shard(u[:, r * L_loc:(r + 1) * L_loc, :], wl.m, wl.q, H) for r in range(R)]
    seqshard.run(steps, seqshard.LocalComm(), shards, N, R * L_loc)
    y = torch.cat([s.y for s in shards], dim=1).numpy()
    ref = oracle.cascade(oracle.powers(wl.Abar[0], N), wl.Bbar[0], wl.C[0], wl.D[0], u[:, :R * L_loc].numpy(), N)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, L, N, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl, u = _system(L, N)
        Ne = seqshard.effective_order(N, L)
        H = seqshard.shard_H(N, L)
        L_loc = L // world
        steps = F64Steps(wl.Abar[0], wl.Bbar[0], wl.C[0], wl.D[0], N, Ne)
        sh = seqshard.make_shard(u[:, rank * L_loc:(rank + 1) * L_loc, :].contiguous(), wl.m, wl.q, H)
        seqshard.run(steps, seqshard.DistComm(), [sh], N, L)
        gathered = [torch.empty_like(sh.y) for _ in range(world)]
        dist.all_gather(gathered, sh.y)          # test-side collection only
        if rank == 0:
            np.save(out_path, torch.cat(gathered, dim=1).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L,N", [(512, 6), (200, 3)])
def test_gloo_world2_halo_exchange_matches_oracle(tmp_path, L, N):
    import torch.multiprocessing as mp
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(2, _free_port(), L, N, out), nprocs=2, join=True)
    y = np.load(out)
    wl, u = _system(L, N)
    ref = oracle.cascade(oracle.powers(wl.Abar[0], N), wl.Bbar[0], wl.C[0], wl.D[0], u.numpy(), N)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))
