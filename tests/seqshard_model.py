"""Test-side model of the library's sequence-sharded schedule (csrc/seqshard.cu), in float64 torch.

It reproduces the schedule the CUDA path runs -- time-major buffers [H + L_loc][batch][dim] with
the halo rows in front, a u halo of uh time rows before the first step (uh = 3 for the Krylov head
v^(2) = sum_{j<4} Abar^j Bbar u_{l-j} when Ne >= 2, R28; uh = 1 for the fused first step),
a halo of the last 2^k time rows of v^(k) before stage k, and before the output step the rows it
reads: 2^Ne of v^(Ne) (R21), or with the output fold for Ne >= 3 (R31) 3*2^(Ne-1) rows of
v^(Ne-1) (stage Ne-1 folded into y); rank 0's halo zero (x_{-1} = 0) -- with the per-step arithmetic written out in
float64, so
the exchange bookkeeping can be checked on the CPU against the oracle: with the real
torch.distributed exchange (gloo, world_size 2, DistComm) and with emulated ranks (LocalComm).
Every halo is one contiguous block of the time-major buffer, as in the library.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


def effective_order(N: int, L: int) -> int:
    """Ne = min(N, floor(log2(L-1))) (R20), exact integer arithmetic."""
    if L <= 2:
        return 0
    return min(N, (L - 1).bit_length() - 1)


@dataclass
class Shard:
    """One rank's buffers: u_ext [uh + L_loc][batch][p] (rows 0..uh-1 = u_{-uh..-1} of this shard),
    Va/Vb [H + L_loc][batch][m] (rows [H - d, H) = the halo of a step with shift d), y [L_loc][batch][q]."""
    u_ext: torch.Tensor
    Va: torch.Tensor
    Vb: torch.Tensor
    y: torch.Tensor


def u_halo_rows(Ne: int) -> int:
    return 3 if Ne >= 2 else 1


def make_shard(u_loc: torch.Tensor, m: int, q: int, H: int, uh: int = 1) -> Shard:
    """u_loc: [L_loc][batch][p]. Halo rows start at zero (rank 0 keeps them)."""
    L_loc, batch, p = u_loc.shape
    dt = u_loc.dtype
    u_ext = torch.zeros((uh + L_loc, batch, p), dtype=dt)
    u_ext[uh:] = u_loc
    Va = torch.zeros((H + L_loc, batch, m), dtype=dt)
    return Shard(u_ext, Va, torch.zeros_like(Va), torch.empty((L_loc, batch, q), dtype=dt))


class DistComm:
    """Halo exchange through torch.distributed P2P: send the last `rows` local rows of `t` to
    rank+1, receive rank-1's into rows [H - rows, H). Both are contiguous in the time-major layout."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def exchange(self, tensors, H: int, rows: int) -> None:
        dist = self.dist
        (t,) = tensors
        ops = []
        if self.rank + 1 < self.world:
            ops.append(dist.P2POp(dist.isend, t[t.shape[0] - rows:], self.rank + 1, self.group))
        if self.rank > 0:
            ops.append(dist.P2POp(dist.irecv, t[H - rows:H], self.rank - 1, self.group))
        for r in dist.batch_isend_irecv(ops) if ops else []:
            r.wait()


class LocalComm:
    """Emulated ranks in one process: shard i's halo is copied from shard i-1's tail."""

    def exchange(self, tensors, H: int, rows: int) -> None:
        for i in range(len(tensors) - 1, 0, -1):
            prev, cur = tensors[i - 1], tensors[i]
            cur[H - rows:H] = prev[prev.shape[0] - rows:]


class F64Steps:
    """The per-step arithmetic of the schedule in float64 (what each GEMM launch computes)."""

    def __init__(self, P, Abar, Bbar, C, D, Ne):
        t = torch.from_numpy
        self.P = [t(x) for x in P]
        Ab, Bb, Cm = t(Abar), t(Bbar), t(C)
        Dm = torch.zeros((C.shape[0], Bbar.shape[1]), dtype=torch.float64) if D is None else t(D)
        self.Bb, self.AB = Bb, Ab @ Bb
        self.Kr = [Bb, self.AB, Ab @ self.AB, Ab @ (Ab @ self.AB)]     # Abar^j Bbar, j < 4 (head)
        self.C, self.CP, self.D = Cm, Cm @ self.P[Ne], Dm
        if Ne >= 3:                                                    # output fold (R31)
            self.CP1, self.CP3 = Cm @ self.P[Ne - 1], (Cm @ self.P[Ne]) @ self.P[Ne - 1]
        self.CBD, self.CAB = Cm @ Bb + Dm, Cm @ (Ab @ Bb)

    def first(self, sh, H):
        u = sh.u_ext                                  # uh = 1
        sh.Va[H:] = u[1:] @ self.Bb.T + u[:-1] @ self.AB.T

    def head(self, sh, H):
        u = sh.u_ext                                  # uh = 3: v^(2) into Vb
        L = sh.y.shape[0]
        sh.Vb[H:] = sum(u[3 - j:3 - j + L] @ self.Kr[j].T for j in range(4))

    def stage(self, k, sh, src, dst, H):
        L = sh.y.shape[0]
        s = 1 << k
        dst[H:] = src[H:] + src[H - s:H - s + L] @ self.P[k].T

    def last(self, Ne, sh, V, H):
        u = sh.u_ext
        uh = u.shape[0] - sh.y.shape[0]
        if Ne == 0:
            sh.y[:] = u[uh:] @ self.CBD.T + u[uh - 1:-1] @ self.CAB.T
            return
        L = sh.y.shape[0]
        if Ne >= 3:                                   # V holds v^(Ne-1): y from four shifts (R31)
            h = 1 << (Ne - 1)
            sh.y[:] = (V[H:] @ self.C.T + V[H - h:H - h + L] @ self.CP1.T + V[H - 2 * h:H - 2 * h + L] @ self.CP.T
                       + V[H - 3 * h:H - 3 * h + L] @ self.CP3.T + u[uh:] @ self.D.T)
            return
        s = 1 << Ne
        sh.y[:] = V[H:] @ self.C.T + V[H - s:H - s + L] @ self.CP.T + u[uh:] @ self.D.T


def run(steps, comm, shards, N: int, L_global: int) -> None:
    """The sharded cascade over `shards` (this process's shards, in rank order)."""
    Ne = effective_order(N, L_global)
    H = out_halo(Ne)
    L_loc = shards[0].y.shape[0]
    if H > L_loc:
        raise NotImplementedError(f"halo {H} exceeds the shard length {L_loc}")
    uh = u_halo_rows(Ne)
    comm.exchange([s.u_ext for s in shards], uh, uh)           # u_{-uh..-1} for the first step
    if Ne == 0:
        for s in shards:
            steps.last(0, s, None, H)
        return
    if Ne >= 2:                                               # Krylov head: v^(2) in Vb
        for s in shards:
            steps.head(s, H)
        src, dst, k0 = [s.Vb for s in shards], [s.Va for s in shards], 2
    else:
        for s in shards:
            steps.first(s, H)
        src, dst, k0 = [s.Va for s in shards], [s.Vb for s in shards], 1
    kl = Ne - 1 if Ne >= 3 else Ne                            # the level the output step reads
    for k in range(k0, kl):
        comm.exchange(src, H, 1 << k)                             # last 2^k rows of v^(k)
        for s, a, b in zip(shards, src, dst):
            steps.stage(k, s, a, b, H)
        src, dst = dst, src
    comm.exchange(src, H, H)
    for s, a in zip(shards, src):
        steps.last(Ne, s, a, H)


def out_halo(Ne: int) -> int:
    """Rows of v the output step reads before l: 3*2^(Ne-1) with the fold (Ne >= 3), else 2^Ne."""
    if Ne <= 0:
        return 0
    return 3 * (1 << (Ne - 1)) if Ne >= 3 else 1 << Ne


def shard_H(N: int, L_global: int) -> int:
    return out_halo(effective_order(N, L_global))


def run_oneshot(steps_factory, comm, u_locs, m: int, q: int, N: int, L_global: int):
    """NEXT-2 schedule (casc_apply_seqsharded, CASC_HALO_ONESHOT_U): one exchange of
    Hu = 2^(Ne+1) - 1 rows of u, then the unsharded cascade on the window [l0 - Hu, l0 + L_loc) of
    each shard (zeros before t = 0) and y kept on the local rows. Returns the local y's."""
    Ne = effective_order(N, L_global)
    Hu = (2 << Ne) - 1 if Ne > 0 else 1
    L_loc, batch, p = u_locs[0].shape
    exts = []
    for u in u_locs:
        e = torch.zeros((Hu + L_loc, batch, p), dtype=u.dtype)
        e[Hu:] = u
        exts.append(e)
    comm.exchange(exts, Hu, Hu)                                   # the only exchange
    ys = []
    for e in exts:
        sh = make_shard(e, m, q, shard_H(N, L_global), u_halo_rows(Ne))
        run(steps_factory(), LocalComm(), [sh], N, L_global)     # one window, no further exchange
        ys.append(sh.y[Hu:])
    return ys
