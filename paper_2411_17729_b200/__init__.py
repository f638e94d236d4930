"""B200-native (sm_100a) fast cascade for LTI/SSM transfer functions (Beylkin, arXiv 2411.17729).

The compute lives in libcascade_b200.so (C ABI: include/cascade.h); this package is the thin
torch-facing binding. There is no CPU fallback.
"""
from .api import (MODES, STORAGE, Comm, Powers, apply, apply_bank, apply_seqsharded,  # noqa: F401
                  apply_workspace_bytes, bank_workspace_bytes, comm_init, comm_init_local,
                  last_launch_count, nccl_unique_id, pack_bytes, powers, powers_norms, profile_enable, profile_read,
                  profile_reset, run_host, run_host_bytes, seqsharded_workspace_bytes)
from ._lib import CascadeError, LIB_PATH, lib  # noqa: F401
