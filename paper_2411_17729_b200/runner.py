"""Map a synth.Workload onto the C-ABI calls (device upload + powers + apply).

Used by the GPU tests, bench.py and __graft_entry__.smoke(). Marshalling only; no arithmetic
of the method happens here.
"""
from __future__ import annotations

import numpy as np
import torch

from . import api


def storage_to_torch(arr: np.ndarray, mode: str) -> torch.Tensor:
    """synth storage array (float32, or uint16 bf16 bits) -> CPU torch tensor of that dtype."""
    if mode == "fp32":
        return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32))
    return torch.from_numpy(np.ascontiguousarray(arr).view(np.int16)).view(torch.bfloat16)


class DeviceWorkload:
    """Inputs of a workload resident in HBM, plus preallocated outputs / workspace."""

    def __init__(self, wl, device="cuda", u_host: np.ndarray | None = None, channels=None,
                 ws_budget: int | None = None):
        """ws_budget: cap on the workspace bytes (banks then run in channel waves); default is
        the full requirement, capped at 75% of the free device memory after inputs/outputs."""
        self.wl = wl
        self.device = device
        ch = list(range(wl.n_ch)) if channels is None else list(channels)
        self.channels = ch
        self.bank = wl.kind == "bank"
        self.N = [int(wl.N[c]) for c in ch]
        self.N_max = max(self.N)
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
        self.Abar = d(wl.Abar[ch])
        if self.bank:
            self.Bbar, self.C, self.D = d(wl.Bbar[ch, :, 0]), d(wl.C[ch, 0, :]), d(wl.D[ch, 0, 0])
        else:
            self.Bbar, self.C, self.D = d(wl.Bbar[ch[0]]), d(wl.C[ch[0]]), d(wl.D[ch[0]])
            if not np.any(wl.D[ch[0]]):
                self.D = None
        if u_host is None:
            u_host = wl.u_storage(ch[0], ch[-1] + 1) if ch == list(range(ch[0], ch[-1] + 1)) \
                else np.stack([wl.u_storage(c, c + 1)[0] for c in ch])
        u = storage_to_torch(u_host, wl.mode)
        if self.bank:
            u = u.reshape(len(ch), wl.batch, wl.L)
        else:
            u = u.reshape(wl.batch, wl.L, wl.p)
        self.u = u.to(device)
        md = api._mode(wl.mode)
        n = len(ch)
        if self.bank:
            self.y = torch.empty((n, wl.batch, wl.L), dtype=api.STORAGE[md], device=device)
            wsb = api.bank_workspace_bytes(n, wl.m, wl.L, wl.batch, self.N_max, md)
        else:
            self.y = torch.empty((wl.batch, wl.L, wl.q), dtype=api.STORAGE[md], device=device)
            wsb = api.apply_workspace_bytes(wl.m, wl.p, wl.q, wl.L, wl.batch, self.N[0], md)
        self.pack = torch.empty(api.pack_bytes(n, wl.m, self.N_max, md), dtype=torch.uint8, device=device)
        if self.bank:
            free = torch.cuda.mem_get_info(torch.device(device))[0]
            cap = int(0.75 * free) if ws_budget is None else int(ws_budget)
            wsb = min(wsb, max(cap, api.bank_workspace_bytes(1, wl.m, wl.L, wl.batch, self.N_max, md)))
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=device)
        self.pw = None

    def step(self, stream=None):
        """One pass of the hot path: powers (a1) + apply (a2..a6)."""
        self.pw = api.powers(self.Abar, self.N, self.wl.mode, N_max=self.N_max, stream=stream, out=self.pack)
        launches = api.last_launch_count()
        if self.bank:
            api.apply_bank(self.pw, self.Bbar, self.C, self.D, self.u, y=self.y, ws=self.ws, stream=stream)
        else:
            api.apply(self.pw, self.Bbar, self.C, self.D, self.u, y=self.y, ws=self.ws, stream=stream)
        return launches + api.last_launch_count()

    def y_f64(self) -> np.ndarray:
        """y as float64 [n][batch][L][q] (CPU)."""
        y = self.y.float().cpu().double().numpy()
        if self.bank:
            return y[..., None]
        return y[None]


class SeqShardedWorkload:
    """This rank's time shard of a single-system workload (BASELINE configs[3] at N > 1 GPUs):
    rows [rank L_loc, (rank+1) L_loc) of every sequence, time-major [L_loc][batch][p], run by
    casc_apply_seqsharded with the library's own per-stage NCCL halo exchange (comm stream)."""

    def __init__(self, wl, rank: int, world: int, device="cuda", comm=None, group=None, halo="per_stage"):
        if wl.kind != "mimo" or wl.L % world:
            raise ValueError("sequence sharding takes one system with L divisible by the rank count")
        self.wl, self.rank, self.world = wl, rank, world
        self.L_loc = wl.L // world
        self.N = int(wl.N[0])
        md = api._mode(wl.mode)
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
        self.Abar, self.Bbar, self.C = d(wl.Abar[0]), d(wl.Bbar[0]), d(wl.C[0])
        self.D = d(wl.D[0]) if np.any(wl.D[0]) else None
        l0 = rank * self.L_loc
        u = np.stack([wl.u_window(0, b, l0, l0 + self.L_loc) for b in range(wl.batch)], axis=1)   # [L_loc][batch][p]
        self.u = torch.from_numpy(u).to(api.STORAGE[md]).to(device)
        self.y = torch.empty((self.L_loc, wl.batch, wl.q), dtype=api.STORAGE[md], device=device)
        self.pack = torch.empty(api.pack_bytes(1, wl.m, self.N, md), dtype=torch.uint8, device=device)
        self.halo = halo
        self.ws = torch.empty(api.seqsharded_workspace_bytes(wl.m, wl.p, wl.q, self.L_loc, wl.batch, self.N, world, md,
                                                             halo), dtype=torch.uint8, device=device)
        if comm is None:
            if world > 1:
                from .seqshard import comm_from_process_group
                comm = comm_from_process_group(group, device=torch.device(device))
            else:
                comm = api.comm_init(0, 1, api.nccl_unique_id())
        self.comm = comm
        self.comm_stream = torch.cuda.Stream(device=device)

    def step(self, stream=None) -> int:
        """powers + the sharded cascade; returns the number of kernel launches."""
        pw = api.powers(self.Abar, self.N, self.wl.mode, stream=stream, out=self.pack)
        n = api.last_launch_count()
        api.apply_seqsharded(self.comm, pw, self.Bbar, self.C, self.D, self.u, y=self.y, ws=self.ws, stream=stream,
                             comm_stream=self.comm_stream, halo=self.halo)
        return n + api.last_launch_count()

    def run_host(self, u_h: torch.Tensor, y_h: torch.Tensor) -> int:
        """End to end from pinned host buffers: H2D of the local u, step, D2H of the local y."""
        self.u.copy_(u_h, non_blocking=True)
        n = self.step()
        y_h.copy_(self.y, non_blocking=True)
        return n

    def y_f64(self) -> np.ndarray:
        """This shard's y as float64 [batch][L_loc][q] (CPU)."""
        return self.y.float().cpu().double().numpy().transpose(1, 0, 2)
