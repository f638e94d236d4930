"""C-ABI checks that need no GPU: the library loads, exports every symbol include/cascade.h
declares, size queries are consistent, and argument validation answers before any device work."""
import ctypes
import os
import re

import pytest

from paper_2411_17729_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "cascade.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(casc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2411_17729_b200 import build
        build.build()
    return _lib.lib()


def test_every_header_symbol_is_exported_and_bound(lib):
    names = header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} missing from the Python binding"


def test_version_and_status_strings(lib):
    assert lib.casc_target_sm() == 100
    assert lib.casc_status_str(0) == b"CASC_OK"
    assert lib.casc_status_str(4) == b"CASC_ERR_UNSUPPORTED"
    assert lib.casc_status_str(99) == b"CASC_ERR_UNKNOWN"


def test_size_queries(lib):
    a = lib.casc_pack_bytes(1, 64, 13, 0)
    b = lib.casc_pack_bytes(1, 64, 13, 1)
    assert b > a > 14 * 64 * 64 * 8           # fp64 powers + tf32 hi/lo (bf16, m <= 64: + bf16 copy)
    a2, b2 = lib.casc_pack_bytes(1, 256, 13, 0), lib.casc_pack_bytes(1, 256, 13, 1)
    assert a2 > b2 > 14 * 256 * 256 * 8       # m > 64: bf16 mode keeps only the bf16 image
    assert lib.casc_pack_bytes(0, 64, 13, 0) == 0
    ws = lib.casc_apply_workspace_bytes(256, 64, 64, 65536, 16, 13, 0)
    assert ws >= 2 * 65536 * 16 * 256 * 4      # two fp32 state buffers
    wsb = lib.casc_bank_workspace_bytes(256, 64, 16384, 4, 13, 0)
    assert wsb >= 2 * 256 * 4 * 16384 * 64 * 4
    assert lib.casc_run_host_bytes(1, 16, 1, 1, 4096, 1, 11, 0) > 0


def test_argument_validation_without_gpu(lib):
    N = _lib.int_array([3])
    # errors are detected before any CUDA call, so these are safe on a CPU-only host
    assert lib.casc_powers(1, 0, N, 3, ctypes.c_void_p(8), 0, ctypes.c_void_p(8), None) == 1
    assert lib.casc_powers(1, 4, N, 2, ctypes.c_void_p(8), 0, ctypes.c_void_p(8), None) == 2   # N > N_max
    assert lib.casc_powers(1, 4, N, 3, ctypes.c_void_p(8), 7, ctypes.c_void_p(8), None) == 1   # bad mode
    v = ctypes.c_void_p(8)
    # p > m
    assert lib.casc_apply(4, 5, 1, 10, 1, 3, 3, 0, v, v, v, None, v, v, v, 1 << 30, None, None) == 2
    # L < 0
    assert lib.casc_apply(4, 1, 1, -1, 1, 3, 3, 0, v, v, v, None, v, v, v, 1 << 30, None, None) == 1
    # workspace too small
    assert lib.casc_apply(4, 1, 1, 10, 1, 3, 3, 0, v, v, v, None, v, v, v, 16, None, None) == 5
    # bank with N_c > N_max
    Nb = _lib.int_array([1, 9])
    assert lib.casc_apply_bank(2, 8, 10, 1, Nb, 3, 0, v, v, v, None, v, v, v, 1 << 30, None) == 2
    # run_host: bank requires SISO
    assert lib.casc_run_host(2, 8, 2, 1, 10, 1, Nb, 9, 0, v, v, v, None, v, v, v, 1 << 40, None) == 4


def test_empty_calls_return_ok_without_touching_buffers(lib):
    """include/cascade.h 'Empty calls': n, L or batch = 0 is a valid call with nothing to compute --
    CASC_OK with every pointer NULL (no device work, so this runs on a CPU-only host), the size
    queries answer 0, and a bad size or mode beside the empty one is still an error."""
    N = _lib.int_array([3])
    e = ctypes.c_int(-1)
    for L, batch in ((0, 4), (100, 0), (0, 0)):
        assert lib.casc_apply(64, 64, 64, L, batch, 3, 3, 0, None, None, None, None, None, None, None, 0,
                              ctypes.byref(e), None) == 0
        assert e.value == 0 or (L > 0 and e.value == 4)      # #{k <= 3 : 2^k < L}
        assert lib.casc_apply_bank(2, 64, L, batch, _lib.int_array([3, 5]), 5, 0, None, None, None, None, None,
                                   None, None, 0, None) == 0
        assert lib.casc_run_host(1, 64, 4, 4, L, batch, N, 3, 1, None, None, None, None, None, None, None, 0,
                                 None) == 0
        assert lib.casc_apply_workspace_bytes(64, 64, 64, L, batch, 3, 0) == 0
        assert lib.casc_run_host_bytes(1, 64, 4, 4, L, batch, 3, 0) == 0
    assert lib.casc_apply_bank(0, 64, 100, 4, None, 5, 0, None, None, None, None, None, None, None, 0, None) == 0
    assert lib.casc_powers(0, 64, None, 5, None, 0, None, None) == 0
    assert lib.casc_apply(64, 64, 64, 0, 4, 3, 3, 9, None, None, None, None, None, None, None, 0, None, None) == 1
    assert lib.casc_apply(64, 65, 64, 0, 4, 3, 3, 0, None, None, None, None, None, None, None, 0, None, None) == 2
    assert lib.casc_apply(64, 64, 64, 0, -1, 3, 3, 0, None, None, None, None, None, None, None, 0, None, None) == 1


def test_sharded_api_validation_without_gpu(lib):
    """The sequence-sharded entry points validate before any CUDA call: an in-process group's
    communicators carry rank / world; bad arguments return CASC_ERR_ARG / _DIM / _UNSUPPORTED."""
    comms = (ctypes.c_void_p * 3)()
    assert lib.casc_comm_init_local(comms, 3) == 0
    r, w = ctypes.c_int(-1), ctypes.c_int(-1)
    for i in range(3):
        assert lib.casc_comm_rank(comms[i], ctypes.byref(r), ctypes.byref(w)) == 0
        assert (r.value, w.value) == (i, 3)
    v = ctypes.c_void_p(8)
    args = lambda comm, m, p, q, L, N, Nmax, halo: (comm, m, p, q, L, 2, N, Nmax, 1, halo,  # noqa: E731
                                                    v, v, v, None, v, v, v, 1 << 40, v, v)
    assert lib.casc_apply_seqsharded(*args(None, 128, 64, 64, 1024, 5, 5, 0)) == 1          # no comm
    assert lib.casc_apply_seqsharded(*args(comms[1], 128, 64, 64, 1024, 5, 5, 7)) == 1      # bad halo mode
    assert lib.casc_apply_seqsharded(*args(comms[1], 128, 64, 64, 1024, 6, 5, 0)) == 2      # N > N_max
    assert lib.casc_apply_seqsharded(*args(comms[1], 96, 64, 64, 1024, 5, 5, 0)) == 4       # m % 64 != 0
    # world 3, L_loc = 100: 2^Ne = 64 fits, the one-shot window 2^(Ne+1) - 1 = 127 does not
    assert lib.casc_apply_seqsharded(*args(comms[1], 128, 64, 64, 100, 6, 6, 1)) == 4
    # workspaces: per-stage halo (2^Ne rows per state buffer) vs one-shot (2^(Ne+1)-1 rows of u and v)
    per = lib.casc_apply_seqsharded_workspace(128, 64, 64, 100, 2, 6, 3, 1, 0)
    one = lib.casc_apply_seqsharded_workspace(128, 64, 64, 100, 2, 6, 3, 1, 1)
    assert per >= 2 * (64 + 100) * 2 * 128 * 2 and one >= 2 * (127 + 100) * 2 * 128 * 2
    for i in range(3):
        assert lib.casc_comm_destroy(comms[i]) == 0
    assert lib.casc_comm_destroy(None) == 1
