"""Sequence sharding on the CPU: the halo schedule of the library's
casc_apply_seqsharded (modelled step by step in tests/seqshard_model.py, time-major buffers, one
contiguous halo block per exchange) driven by emulated ranks and by the real torch.distributed
exchange (gloo, world_size 2); the result must equal the unsharded float64 oracle (pin T15). The
NCCL unique-id handshake the library's communicator needs (rank 0 creates the id through the
C ABI, torch broadcasts it) is also checked over gloo."""
import os
import socket
import sys

import numpy as np
import pytest
import torch

import oracle
from synth import configs as S

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import seqshard_model as model  # noqa: E402


def _system(L, N, seed=3):
    wl = S.make_random_mimo(6, 2, 3, L=L, batch=2, N=N, rho=0.97, seed=seed)
    u = torch.from_numpy(wl.u_all()[0]).permute(1, 0, 2).contiguous()      # time-major [L][batch][p]
    return wl, u


def _ref(wl, u, N):
    y = oracle.cascade(oracle.powers(wl.Abar[0], N), wl.Bbar[0], wl.C[0], wl.D[0], u.permute(1, 0, 2).numpy(), N)
    return y.transpose(1, 0, 2)                                          # [L][batch][q]


def _steps(wl, N, L):
    Ne = model.effective_order(N, L)
    return model.F64Steps(oracle.powers(wl.Abar[0], N), wl.Abar[0], wl.Bbar[0], wl.C[0], wl.D[0], Ne)


@pytest.mark.parametrize("R,L,N", [(4, 256, 5), (2, 100, 3), (2, 64, 4), (3, 90, 0), (2, 2, 3), (8, 2048, 7),
                                   (4, 64, 2)])
def test_local_emulated_ranks_match_oracle(R, L, N):
    wl, u = _system(L, N)
    Ne = model.effective_order(N, L)
    H = model.shard_H(N, L)
    L_loc = L // R
    if H > L_loc:
        pytest.skip("halo longer than a shard")
    uh = model.u_halo_rows(Ne)
    if uh > L_loc:
        pytest.skip("u halo longer than a shard")
    shards = [model.make_shard(u[r * L_loc:(r + 1) * L_loc], wl.m, wl.q, H, uh) for r in range(R)]
    model.run(_steps(wl, N, L), model.LocalComm(), shards, N, R * L_loc)
    y = torch.cat([s.y for s in shards], dim=0).numpy()
    ref = _ref(wl, u[:R * L_loc], N)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_effective_order_exact_for_large_L():
    """floor(log2(L - 1)) by integer arithmetic: L - 1 = 2^k - 1 must give k - 1 even where a float
    log2 rounds up."""
    for k in (3, 20, 40, 53, 60):
        L = 1 << k
        assert model.effective_order(99, L) == k - 1
        assert model.effective_order(99, L + 1) == k
        assert model.effective_order(99, L - 1) == k - 1


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
        H = model.shard_H(N, L)
        L_loc = L // world
        uh = model.u_halo_rows(model.effective_order(N, L))
        sh = model.make_shard(u[rank * L_loc:(rank + 1) * L_loc].contiguous(), wl.m, wl.q, H, uh)
        model.run(_steps(wl, N, L), model.DistComm(), [sh], N, L)
        gathered = [torch.empty_like(sh.y) for _ in range(world)]
        dist.all_gather(gathered, sh.y)          # test-side collection only
        if rank == 0:
            np.save(out_path, torch.cat(gathered, dim=0).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L,N", [(512, 6), (200, 3)])
def test_gloo_world2_halo_exchange_matches_oracle(tmp_path, L, N):
    import torch.multiprocessing as mp
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(2, _free_port(), L, N, out), nprocs=2, join=True)
    y = np.load(out)
    wl, u = _system(L, N)
    ref = _ref(wl, u, N)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


def _uid_worker(rank, world, port, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_17729_b200.seqshard import broadcast_unique_id
        uid = broadcast_unique_id()
        np.save(f"{out_path}.{rank}.npy", np.frombuffer(uid, dtype=np.uint8))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_nccl_unique_id_broadcast(tmp_path):
    """Rank 0's casc_nccl_unique_id reaches rank 1 unchanged (128 bytes, not all zero)."""
    import torch.multiprocessing as mp
    import paper_2411_17729_b200 as pk
    try:
        pk.nccl_unique_id()
    except pk.CascadeError as e:
        pytest.skip(f"libnccl not loadable here: {e}")
    out = str(tmp_path / "uid")
    mp.spawn(_uid_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    a, b = np.load(out + ".0.npy"), np.load(out + ".1.npy")
    assert a.shape == (128,) and np.array_equal(a, b) and a.any()


@pytest.mark.parametrize("R,L,N", [(4, 1024, 5), (2, 200, 3), (8, 4096, 8), (3, 90, 0)])
def test_oneshot_u_halo_schedule_matches_oracle(R, L, N):
    """NEXT-2 on the CPU: one exchange of 2^(Ne+1) - 1 rows of u and a rank-local cascade on the
    window give the global outputs (window property, pin T14)."""
    wl, u = _system(L, N)
    L_loc = L // R
    Ne = model.effective_order(N, L)
    if ((2 << Ne) - 1 if Ne else 1) > L_loc:
        pytest.skip("window longer than a shard")
    ys = model.run_oneshot(lambda: _steps(wl, N, L), model.LocalComm(),
                           [u[r * L_loc:(r + 1) * L_loc] for r in range(R)], wl.m, wl.q, N, L)
    y = torch.cat(ys, dim=0).numpy()
    ref = _ref(wl, u[:R * L_loc], N)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))
