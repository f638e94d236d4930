"""Torch-facing binding of the C ABI (include/cascade.h). Marshalling only: every step of the
cascade runs inside libcascade_b200.so; torch provides device memory and streams.

Names follow the paper: `powers`, `apply`,
`apply_bank` (per-channel SISO bank, the HiPPO example PAPER.md:253-273).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from ._lib import check, int_array, lib

MODES = {"fp32": 0, "bf16": 1}
PIPES = {0: "none", 1: "tf32", 2: "bf16", 3: "fp64", 4: "fp32"}
STORAGE = {0: torch.float32, 1: torch.bfloat16}


def _mode(mode) -> int:
    return MODES[mode] if isinstance(mode, str) else int(mode)


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _p(t) -> ctypes.c_void_p | None:
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _need(t, dtype, shape, name):
    if t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name}: must be a contiguous CUDA tensor")


@dataclass
class Powers:
    """Opaque pack of Abar^(2^k), k = 0..N_s, per system (float64 + storage rounding)."""
    pack: torch.Tensor
    n_sys: int
    m: int
    N: list
    N_max: int
    mode: int


def pack_bytes(n_sys: int, m: int, N_max: int, mode) -> int:
    return int(lib().casc_pack_bytes(n_sys, m, N_max, _mode(mode)))


def powers(Abar: torch.Tensor, N, mode="fp32", N_max: int | None = None, stream=None,
           out: torch.Tensor | None = None) -> Powers:
    """Abar: float64 CUDA [n_sys][m][m] (or [m][m]); N: int or per-system list."""
    if Abar.dim() == 2:
        Abar = Abar.unsqueeze(0)
    n_sys, m = Abar.shape[0], Abar.shape[1]
    Ns = [int(N)] * n_sys if isinstance(N, int) else [int(x) for x in N]
    N_max = max(Ns) if N_max is None else int(N_max)
    md = _mode(mode)
    _need(Abar, torch.float64, (n_sys, m, m), "Abar")
    nbytes = pack_bytes(n_sys, m, N_max, md)
    pack = torch.empty(nbytes, dtype=torch.uint8, device=Abar.device) if out is None else out
    check(lib().casc_powers(n_sys, m, int_array(Ns), N_max, _p(Abar), md, _p(pack), _stream(stream)),
          "casc_powers")
    return Powers(pack, n_sys, m, Ns, N_max, md)


def powers_norms(pw: Powers, stream=None):
    """||P_k||_F for k = 0..N_s + 1 of each system (the last one the first neglected power, the
    planner's truncation indicator); numpy float64 [n_sys][N_max + 2], NaN past N_s + 1."""
    import numpy as np
    out = np.empty((pw.n_sys, pw.N_max + 2), dtype=np.float64)
    check(lib().casc_powers_norms(pw.n_sys, pw.m, pw.N_max, pw.mode, _p(pw.pack),
                                  out.ctypes.data_as(ctypes.c_void_p), _stream(stream)), "casc_powers_norms")
    return out


def apply_workspace_bytes(m, p, q, L, batch, N, mode) -> int:
    return int(lib().casc_apply_workspace_bytes(m, p, q, L, batch, N, _mode(mode)))


def bank_workspace_bytes(n_ch, m, L, batch, N_max, mode) -> int:
    return int(lib().casc_bank_workspace_bytes(n_ch, m, L, batch, N_max, _mode(mode)))


def apply(pw: Powers, Bbar, C, D, u, y=None, ws=None, stream=None, return_stages=False):
    """One system: u [batch][L][p] (storage dtype) -> y [batch][L][q]."""
    if pw.n_sys != 1:
        raise ValueError("apply() takes a single-system pack; use apply_bank()")
    m, N, md = pw.m, pw.N[0], pw.mode
    batch, L, p = u.shape
    q = C.shape[0]
    _need(u, STORAGE[md], (batch, L, p), "u")
    _need(Bbar, torch.float64, (m, p), "Bbar")
    _need(C, torch.float64, (q, m), "C")
    if D is not None:
        _need(D, torch.float64, (q, p), "D")
    if y is None:
        y = torch.empty((batch, L, q), dtype=STORAGE[md], device=u.device)
    _need(y, STORAGE[md], (batch, L, q), "y")
    wsb = apply_workspace_bytes(m, p, q, L, batch, N, md)
    if ws is None:
        ws = torch.empty(wsb, dtype=torch.uint8, device=u.device)
    eff = ctypes.c_int(0)
    check(lib().casc_apply(m, p, q, L, batch, N, pw.N_max, md, _p(pw.pack), _p(Bbar), _p(C), _p(D),
                           _p(u), _p(y), _p(ws), ws.numel(), ctypes.byref(eff), _stream(stream)),
          "casc_apply")
    return (y, eff.value) if return_stages else y


def apply_bank(pw: Powers, Bbar, C, D, u, y=None, ws=None, stream=None):
    """Bank of SISO channels: u [n_ch][batch][L] (storage dtype) -> y [n_ch][batch][L]."""
    n, m, md = pw.n_sys, pw.m, pw.mode
    _, batch, L = u.shape
    _need(u, STORAGE[md], (n, batch, L), "u")
    _need(Bbar, torch.float64, (n, m), "Bbar")
    _need(C, torch.float64, (n, m), "C")
    if D is not None:
        _need(D, torch.float64, (n,), "D")
    if y is None:
        y = torch.empty((n, batch, L), dtype=STORAGE[md], device=u.device)
    _need(y, STORAGE[md], (n, batch, L), "y")
    wsb = bank_workspace_bytes(n, m, L, batch, pw.N_max, md)
    if ws is None:
        ws = torch.empty(wsb, dtype=torch.uint8, device=u.device)
    check(lib().casc_apply_bank(n, m, L, batch, int_array(pw.N), pw.N_max, md, _p(pw.pack), _p(Bbar),
                                _p(C), _p(D), _p(u), _p(y), _p(ws), ws.numel(), _stream(stream)),
          "casc_apply_bank")
    return y


def run_host_bytes(n_sys, m, p, q, L, batch, N_max, mode) -> int:
    return int(lib().casc_run_host_bytes(n_sys, m, p, q, L, batch, N_max, _mode(mode)))


def run_host(Abar_h, Bbar_h, C_h, D_h, u_h, y_h, N, mode, dev_ws, stream=None):
    """End to end from HOST tensors (pinned for async copies): powers + apply, y written to y_h.
    Abar_h [n][m][m], Bbar_h [n][m][p], C_h [n][q][m], D_h [n][q][p] or None (float64, CPU);
    u_h [n][batch][L][p], y_h [n][batch][L][q] in the storage dtype (CPU)."""
    n, m, _ = Abar_h.shape
    p, q = Bbar_h.shape[2], C_h.shape[1]
    _, batch, L, _ = u_h.shape
    Ns = [int(N)] * n if isinstance(N, int) else [int(x) for x in N]
    md = _mode(mode)
    for t in (Abar_h, Bbar_h, C_h, u_h, y_h) + ((D_h,) if D_h is not None else ()):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("run_host takes contiguous host tensors")
    check(lib().casc_run_host(n, m, p, q, L, batch, int_array(Ns), max(Ns), md, _p(Abar_h), _p(Bbar_h),
                              _p(C_h), _p(D_h), _p(u_h), _p(y_h), _p(dev_ws), dev_ws.numel(),
                              _stream(stream)),
          "casc_run_host")
    return y_h


def last_launch_count() -> int:
    return int(lib().casc_last_launch_count())


# ------------------------------------------------------------------ in-library kernel timing
def profile_enable(on: bool = True) -> None:
    lib().casc_profile_enable(1 if on else 0)


def profile_reset() -> None:
    lib().casc_profile_reset()


def profile_read() -> dict:
    """{class_name: {launches, ms, bytes, flops}} for classes with at least one launch."""
    out = {}
    L = lib()
    for c in range(L.casc_profile_num_classes()):
        n, ms, by, fl = ctypes.c_int(0), ctypes.c_double(0), ctypes.c_double(0), ctypes.c_double(0)
        check(L.casc_profile_read(c, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(by), ctypes.byref(fl)),
              "casc_profile_read")
        if n.value:
            xb, xf, pipe = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_int(0)
            check(L.casc_profile_read_exec(c, ctypes.byref(xb), ctypes.byref(xf), ctypes.byref(pipe)),
                  "casc_profile_read_exec")
            out[L.casc_profile_class_name(c).decode()] = {
                "launches": n.value, "ms": ms.value, "bytes": by.value, "flops": fl.value,
                "exec_bytes": xb.value, "exec_flops": xf.value, "pipe": PIPES.get(pipe.value, "none")}
    return out


# ------------------------------------------------------------------ sequence sharding (a7)
def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it)."""
    buf = ctypes.create_string_buffer(128)
    check(lib().casc_nccl_unique_id(buf), "casc_nccl_unique_id")
    return buf.raw


class Comm:
    """A library communicator (NCCL, or one rank of an in-process emulated group)."""

    def __init__(self, handle: ctypes.c_void_p):
        self.handle = handle
        r, w = ctypes.c_int(0), ctypes.c_int(0)
        check(lib().casc_comm_rank(handle, ctypes.byref(r), ctypes.byref(w)), "casc_comm_rank")
        self.rank, self.world = r.value, w.value

    def destroy(self) -> None:
        if self.handle:
            check(lib().casc_comm_destroy(self.handle), "casc_comm_destroy")
            self.handle = None


def comm_init(rank: int, world: int, unique_id: bytes) -> Comm:
    """NCCL communicator on the current CUDA device (blocks until all ranks joined)."""
    h = ctypes.c_void_p()
    check(lib().casc_comm_init(ctypes.byref(h), rank, world, ctypes.create_string_buffer(unique_id, 128)),
          "casc_comm_init")
    return Comm(h)


def comm_init_local(world: int) -> list:
    """`world` emulated ranks in this process (one device); run each rank's apply on its own thread."""
    hs = (ctypes.c_void_p * world)()
    check(lib().casc_comm_init_local(hs, world), "casc_comm_init_local")
    return [Comm(ctypes.c_void_p(h)) for h in hs]


HALOS = {"per_stage": 0, "oneshot_u": 1, "peer": 2}


def seqsharded_workspace_bytes(m, p, q, L_loc, batch, N, world, mode, halo="per_stage") -> int:
    return int(lib().casc_apply_seqsharded_workspace(m, p, q, L_loc, batch, N, world, _mode(mode), HALOS[halo]))


def apply_seqsharded(comm: Comm, pw: Powers, Bbar, C, D, u_loc, y=None, ws=None, stream=None,
                     comm_stream=None, halo="per_stage"):
    """This rank's shard: u_loc [L_loc][batch][p] (time-major, storage dtype) -> y [L_loc][batch][q].
    The halo exchange with the neighbouring ranks happens inside the library (comm_stream):
    halo='per_stage' (one exchange per step), 'oneshot_u' (2^(Ne+1)-1 rows of u once, NEXT-2) or
    'peer' (the producing GEMM stores the halo rows into rank r+1's buffer; tokens order the ranks)."""
    if pw.n_sys != 1:
        raise ValueError("apply_seqsharded() takes a single-system pack")
    m, N, md = pw.m, pw.N[0], pw.mode
    L_loc, batch, p = u_loc.shape
    q = C.shape[0]
    _need(u_loc, STORAGE[md], (L_loc, batch, p), "u_loc")
    _need(Bbar, torch.float64, (m, p), "Bbar")
    _need(C, torch.float64, (q, m), "C")
    if D is not None:
        _need(D, torch.float64, (q, p), "D")
    if y is None:
        y = torch.empty((L_loc, batch, q), dtype=STORAGE[md], device=u_loc.device)
    _need(y, STORAGE[md], (L_loc, batch, q), "y")
    if ws is None:
        ws = torch.empty(seqsharded_workspace_bytes(m, p, q, L_loc, batch, N, comm.world, md, halo),
                         dtype=torch.uint8, device=u_loc.device)
    if comm_stream is None:
        raise ValueError("apply_seqsharded needs a comm stream distinct from the compute stream")
    check(lib().casc_apply_seqsharded(comm.handle, m, p, q, L_loc, batch, N, pw.N_max, md, HALOS[halo],
                                      _p(pw.pack), _p(Bbar),
                                      _p(C), _p(D), _p(u_loc), _p(y), _p(ws), ws.numel(), _stream(stream),
                                      _stream(comm_stream)),
          "casc_apply_seqsharded")
    return y
