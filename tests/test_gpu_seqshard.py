"""Library-owned sequence sharding (casc_apply_seqsharded, csrc/seqshard.cu) on one GPU.

R emulated ranks (casc_comm_init_local: one host thread and one pair of streams per rank, halos as
device copies ordered by events -- ranks never spin on each other inside a kernel) run the same
schedule as the NCCL transport. The result must be bitwise the 1-rank run over an NCCL
communicator (world 1) and bitwise the unsharded casc_apply (each output row's accumulation
order does not depend on the shard or tile it lives in; SURVEY pin T15), and within tolerance of
the float64 oracle."""
import threading

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
    pk.lib()


def _sharded(wl, R, comms, halo="per_stage"):
    """Run R ranks of casc_apply_seqsharded, each on its own thread; returns y [L][batch][q]."""
    import paper_2411_17729_b200 as pk
    md = wl.mode
    N = int(wl.N[0])
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    Abar, Bbar, C = d(wl.Abar[0]), d(wl.Bbar[0]), d(wl.C[0])
    D = d(wl.D[0]) if np.any(wl.D[0]) else None
    u = torch.from_numpy(wl.u_all()[0].transpose(1, 0, 2).copy()).to(pk.STORAGE[pk.api._mode(md)]).cuda()
    L_loc = wl.L // R
    pw = pk.powers(Abar, N, md)
    torch.cuda.synchronize()
    ys = [None] * R
    errs = []

    def rank(r):
        try:
            st, cs = torch.cuda.Stream(), torch.cuda.Stream()
            u_loc = u[r * L_loc:(r + 1) * L_loc].contiguous()
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                ys[r] = pk.apply_seqsharded(comms[r], pw, Bbar, C, D, u_loc, stream=st, comm_stream=cs, halo=halo)
            st.synchronize()
        except Exception as e:                    # reported by the main thread
            errs.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    torch.cuda.synchronize()
    return torch.cat(ys, dim=0)


CASES = [  # (R, m, p, q, L, N)
    (2, 128, 64, 64, 4096, 8),
    (2, 64, 64, 64, 2048, 9),       # output halo 3 * 2^8 = 768 of L_loc = 1024 rows (R31)
    (4, 64, 64, 64, 1024, 2),       # Ne = 2: no fold, head only
    (8, 128, 64, 128, 8192, 6),
    (2, 64, 64, 64, 256, 0),        # Ne = 0: one fused step
    (3, 256, 64, 64, 3000, 7),      # rows not a multiple of the 256-row blocks
]


@pytest.mark.parametrize("mode", ["bf16", "fp32"])
@pytest.mark.parametrize("case", CASES)
def test_emulated_ranks_bitwise(mode, case):
    import paper_2411_17729_b200 as pk
    R, m, p, q, L, N = case
    wl = S.make_random_mimo(m, p, q, L=L, batch=3, N=N, rho=0.97, mode=mode)
    comms = pk.comm_init_local(R)
    try:
        y_R = _sharded(wl, R, comms)
    finally:
        for c in comms:
            c.destroy()
    one = pk.comm_init(0, 1, pk.nccl_unique_id())                   # NCCL transport, one rank
    try:
        y_1 = _sharded(wl, 1, [one])
    finally:
        one.destroy()
    assert torch.equal(y_R, y_1), "R emulated ranks differ from one rank"
    from paper_2411_17729_b200.runner import DeviceWorkload
    dw = DeviceWorkload(wl)
    dw.step()
    torch.cuda.synchronize()
    assert torch.equal(y_1.permute(1, 0, 2), dw.y), "sharded (time-major) differs from unsharded casc_apply"
    ref = oracle.apply_workload(wl)[0]
    yn = y_R.permute(1, 0, 2).float().cpu().double().numpy()
    assert np.linalg.norm(yn - ref) / np.linalg.norm(ref) <= TOL[mode]


def test_halo_longer_than_shard_is_unsupported():
    import paper_2411_17729_b200 as pk
    wl = S.make_random_mimo(64, 64, 64, L=1024, batch=1, N=9, rho=0.9, mode="bf16")   # 2^9 > L/4
    comms = pk.comm_init_local(4)
    try:
        with pytest.raises(pk.CascadeError, match="UNSUPPORTED"):
            _sharded(wl, 4, comms)
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("mode", ["bf16", "fp32"])
@pytest.mark.parametrize("case", [c for c in CASES if c[0] == 1 or ((2 << min(c[5], (c[4] - 1).bit_length() - 1)) - 1)
                                  <= c[4] // c[0]])
def test_oneshot_u_halo_bitwise(mode, case):
    """NEXT-2: one exchange of 2^(Ne+1) - 1 rows of u, then the whole cascade on the window
    [l0 - Hu, l0 + L_loc) (exact by the window property, pin T14): bitwise the per-stage result and
    the unsharded casc_apply, since every output row is computed by the same operations."""
    import paper_2411_17729_b200 as pk
    R, m, p, q, L, N = case
    wl = S.make_random_mimo(m, p, q, L=L, batch=3, N=N, rho=0.97, mode=mode)
    comms = pk.comm_init_local(R)
    try:
        y_one = _sharded(wl, R, comms, halo="oneshot_u")
    finally:
        for c in comms:
            c.destroy()
    comms = pk.comm_init_local(R)
    try:
        y_per = _sharded(wl, R, comms, halo="per_stage")
    finally:
        for c in comms:
            c.destroy()
    assert torch.equal(y_one, y_per)
    from paper_2411_17729_b200.runner import DeviceWorkload
    dw = DeviceWorkload(wl)
    dw.step()
    torch.cuda.synchronize()
    assert torch.equal(y_one.permute(1, 0, 2), dw.y)



PEER_CASES = [  # (R, m, p, q, L, N): the CTA-pair GEMMs (bf16: m % 256 == 0; fp32: m % 128 == 0)
    (2, 256, 64, 64, 4096, 8),
    (4, 256, 64, 128, 8192, 6),
    (3, 256, 64, 64, 3000, 7),      # rows not a multiple of the 256-row blocks
    (2, 256, 64, 64, 2048, 2),      # Ne = 2: the head's rows go straight to the output step
    (2, 256, 64, 64, 256, 0),       # Ne = 0: no state halo (the per-stage schedule)
]


@pytest.mark.parametrize("mode", ["bf16", "fp32"])
@pytest.mark.parametrize("case", PEER_CASES)
def test_peer_halo_bitwise(mode, case):
    """NEXT-2 fused: the GEMM producing v^(k) stores its last 2^k rows into rank r+1's halo rows
    from its epilogue (emulated ranks: into the other rank's workspace on this device), the
    transport only orders the ranks with tokens. Bitwise the per-stage halo and the unsharded
    casc_apply: the halo rows are the same values, read by the same operations."""
    import paper_2411_17729_b200 as pk
    R, m, p, q, L, N = case
    if mode == "fp32" and m % 128:
        pytest.skip("fp32 peer halo needs m % 128 == 0")
    wl = S.make_random_mimo(m, p, q, L=L, batch=3, N=N, rho=0.97, mode=mode)
    comms = pk.comm_init_local(R)
    try:
        y_peer = _sharded(wl, R, comms, halo="peer")
        y_peer2 = _sharded(wl, R, comms, halo="peer")              # a second call on the same comms
    finally:
        for c in comms:
            c.destroy()
    comms = pk.comm_init_local(R)
    try:
        y_per = _sharded(wl, R, comms, halo="per_stage")
    finally:
        for c in comms:
            c.destroy()
    assert torch.equal(y_peer, y_per)
    assert torch.equal(y_peer2, y_per)
    from paper_2411_17729_b200.runner import DeviceWorkload
    dw = DeviceWorkload(wl)
    dw.step()
    torch.cuda.synchronize()
    assert torch.equal(y_peer.permute(1, 0, 2), dw.y)


def test_peer_halo_one_nccl_rank():
    """One NCCL rank: no successor, no IPC mapping; the peer schedule equals the per-stage one."""
    import paper_2411_17729_b200 as pk
    wl = S.make_random_mimo(256, 64, 64, L=2048, batch=2, N=7, rho=0.97, mode="bf16")
    one = pk.comm_init(0, 1, pk.nccl_unique_id())
    try:
        y_peer = _sharded(wl, 1, [one], halo="peer")
        y_per = _sharded(wl, 1, [one], halo="per_stage")
    finally:
        one.destroy()
    assert torch.equal(y_peer, y_per)


def test_peer_halo_needs_pair_gemm():
    """m = 128 in bf16 runs on the one-CTA GEMM, which cannot store into a peer: UNSUPPORTED."""
    import paper_2411_17729_b200 as pk
    wl = S.make_random_mimo(128, 64, 64, L=2048, batch=2, N=6, rho=0.97, mode="bf16")
    comms = pk.comm_init_local(2)
    try:
        with pytest.raises(pk.CascadeError, match="UNSUPPORTED"):
            _sharded(wl, 2, comms, halo="peer")
    finally:
        for c in comms:
            c.destroy()
