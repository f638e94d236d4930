"""ctypes declarations of the C ABI in include/cascade.h (argument marshalling only)."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = _DEFAULT = os.path.join(_HERE, "libcascade_b200.so")
# diagnostics only: A/B two builds of the library within one process launch environment
if os.environ.get("CASC_LIB_OVERRIDE"):
    LIB_PATH = os.path.abspath(os.environ["CASC_LIB_OVERRIDE"])

c_int, c_size_t, c_int64, c_void_p, c_char_p = ctypes.c_int, ctypes.c_size_t, ctypes.c_int64, ctypes.c_void_p, ctypes.c_char_p
P_int = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes); the list is also the symbol export check of tests/test_abi.py
SIGNATURES = {
    "casc_status_str": (c_char_p, [c_int]),
    "casc_version": (c_int, []),
    "casc_target_sm": (c_int, []),
    "casc_last_launch_count": (c_int, []),
    "casc_pack_bytes": (c_size_t, [c_int, c_int, c_int, c_int]),
    "casc_powers": (c_int, [c_int, c_int, P_int, c_int, c_void_p, c_int, c_void_p, c_void_p]),
    "casc_powers_norms": (c_int, [c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "casc_apply_workspace_bytes": (c_size_t, [c_int, c_int, c_int, c_int64, c_int, c_int, c_int]),
    "casc_apply": (c_int, [c_int, c_int, c_int, c_int64, c_int, c_int, c_int, c_int,
                           c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                           c_void_p, c_size_t, P_int, c_void_p]),
    "casc_bank_workspace_bytes": (c_size_t, [c_int, c_int, c_int64, c_int, c_int, c_int]),
    "casc_apply_bank": (c_int, [c_int, c_int, c_int64, c_int, P_int, c_int, c_int,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_size_t, c_void_p]),
    "casc_run_host_bytes": (c_size_t, [c_int, c_int, c_int, c_int, c_int64, c_int, c_int, c_int]),
    "casc_run_host": (c_int, [c_int, c_int, c_int, c_int, c_int64, c_int, P_int, c_int, c_int,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                              c_void_p, c_size_t, c_void_p]),
    "casc_selftest_umma": (c_int, [c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "casc_nccl_unique_id": (c_int, [c_void_p]),
    "casc_comm_init": (c_int, [ctypes.POINTER(c_void_p), c_int, c_int, c_void_p]),
    "casc_comm_init_local": (c_int, [ctypes.POINTER(c_void_p), c_int]),
    "casc_comm_destroy": (c_int, [c_void_p]),
    "casc_comm_rank": (c_int, [c_void_p, P_int, P_int]),
    "casc_apply_seqsharded_workspace": (c_size_t, [c_int, c_int, c_int, c_int64, c_int, c_int, c_int, c_int,
                                                   c_int]),
    "casc_apply_seqsharded": (c_int, [c_void_p, c_int, c_int, c_int, c_int64, c_int, c_int, c_int, c_int, c_int,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_size_t, c_void_p, c_void_p]),
    "casc_profile_enable": (c_int, [c_int]),
    "casc_profile_reset": (c_int, []),
    "casc_profile_num_classes": (c_int, []),
    "casc_profile_class_name": (c_char_p, [c_int]),
    "casc_profile_read": (c_int, [c_int, P_int, ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "casc_profile_read_exec": (c_int, [c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                       P_int]),
}

_lib = None


class CascadeError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Load the in-tree CUDA library; fails loudly if it is missing (there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CascadeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the cascade has no CPU fallback)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if LIB_PATH != _DEFAULT and not hasattr(l, name):
                continue                     # A/B against an older build: only what it exports
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        name = lib().casc_status_str(status).decode()
        raise CascadeError(f"{what} failed: {name} ({status})")


def int_array(vals):
    arr = (ctypes.c_int * len(vals))(*[int(v) for v in vals])
    return arr
