"""ctypes binding of libpip.so (the C ABI declared in include/pip.h).

Loading is lazy and LOUD: there is no CPU fallback anywhere in the product
path.  If the shared library is missing or cannot be loaded, every operation
raises ``RuntimeError``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libpip.so"
_lib = None

u64 = C.c_uint64
u32 = C.c_uint32
vp = C.c_void_p
i32 = C.c_int
sz = C.c_size_t

# status codes (include/pip.h)
PIP_OK = 0
PIP_ERR_INVALID_ARG = 1
PIP_ERR_INVALID_SWAPS = 2
PIP_ERR_LIVELOCK = 3
PIP_ERR_OOM = 4
PIP_ERR_CUDA = 5
PIP_ERR_UNSORTED = 6
PIP_ERR_UNSUPPORTED = 7
PIP_ERR_TABLE = 8
PIP_ERR_DEBUG_SWEEP = 9
PIP_ERR_STALLED = 10

OP_ADD, OP_MAX, OP_MIN, OP_XOR = 0, 1, 2, 3
RP_NAIVE, RP_FLAT, RP_ONERES, RP_FINAL = 0, 1, 2, 3

PRED_ALL, PRED_MASK_EQ, PRED_MOD_EQ, PRED_LT, PRED_LE, PRED_GT, PRED_GE, PRED_EQ = range(8)


class PipPred(C.Structure):
    _fields_ = [("kind", u32), ("negate", u32), ("a", u64), ("b", u64)]


class PipRpStats(C.Structure):
    _fields_ = [
        ("rounds", u64),
        ("total_committed", u64),
        ("n_iterates", u64),
        ("peak_table_count", u64),
        ("table_capacity", u64),
        ("prefix", u64),
        ("workspace_words", u64),
        ("rounds_recorded", u64),
    ]


class PipShardPiece(C.Structure):
    _fields_ = [("peer", u32), ("reserved", u32), ("local_offset", u64), ("length", u64)]


# name -> (restype, argtypes); the full export list of include/pip.h
SIGNATURES = {
    "pip_version": (i32, []),
    "pip_status_string": (C.c_char_p, [i32]),
    "pip_last_cuda_error": (C.c_char_p, []),
    "pip_scratch_bytes": (sz, [i32]),
    "pip_scratch_status": (i32, [vp, vp]),
    "pip_scan_u64": (i32, [vp, u64, i32, u64, i32, vp, vp, sz, vp]),
    "pip_scan_u64_carry": (i32, [vp, u64, i32, u64, i32, vp, vp, vp, sz, vp]),
    "pip_reduce_u64": (i32, [vp, u64, i32, vp, vp, sz, vp]),
    "pip_scan_u64_host": (i32, [vp, u64, i32, u64, i32, C.POINTER(u64), i32]),
    "pip_filter_u64": (i32, [vp, u64, C.POINTER(PipPred), vp, vp, sz, vp]),
    "pip_count_u64": (i32, [vp, u64, C.POINTER(PipPred), vp, vp, sz, vp]),
    "pip_filter_u64_host": (i32, [vp, u64, C.POINTER(PipPred), C.POINTER(u64), i32]),
    "pip_rotate_u64": (i32, [vp, u64, u64, vp, sz, vp]),
    "pip_reverse_u64": (i32, [vp, u64, vp]),
    "pip_move_u64": (i32, [vp, u64, u64, u64, vp, sz, vp]),
    "pip_compact_by_mask_u64": (i32, [vp, u64, vp, vp, vp, sz, vp]),
    "pip_rt_workspace_bytes": (sz, [u64]),
    "pip_rt_reserve_max_u64": (i32, [vp, vp, u64, vp, vp, u64, vp, sz, C.POINTER(u64), vp]),
    "pip_rt_lookup_u64": (i32, [vp, vp, u64, vp, u64, vp, vp, vp]),
    "pip_rt_delete_u64": (i32, [vp, u64, vp, u64, vp, sz, C.POINTER(u64), vp]),
    "pip_partition_workspace_bytes": (sz, [u64]),
    "pip_partition_u64": (i32, [vp, u64, C.POINTER(PipPred), vp, vp, sz, vp]),
    "pip_partition_u64_host": (i32, [vp, u64, C.POINTER(PipPred), C.POINTER(u64), i32]),
    "pip_partition_segments_u64": (i32, [vp, vp, vp, vp, C.c_uint32, vp, u64, vp, sz, vp]),
    "pip_sort_segments_u64": (i32, [vp, vp, vp, u64, vp]),
    "pip_sort_segments_grid_u64": (i32, [vp, vp, vp, u64, u64, vp]),
    "pip_list_contract_workspace_bytes": (sz, [u64, u64, i32]),
    "pip_tree_contract_workspace_bytes": (sz, [u64, u64]),
    "pip_tree_contract_u64": (i32, [vp, vp, vp, vp, vp, u64, u64, i32, i32, vp, u64, C.POINTER(u64), vp,
                                    vp, C.POINTER(u64), C.POINTER(u64), vp, sz, vp]),
    "pip_tree_round_u64": (i32, [i32, vp, vp, vp, vp, vp, u64, u64, vp, u64, vp, vp, vp, i32, vp]),
    "pip_list_contract_u64": (i32, [vp, vp, vp, u64, u64, i32, vp, u64, vp, vp, vp, vp, sz, vp]),
    "pip_merge_u64": (i32, [vp, u64, u64, i32, vp, sz, vp, sz, vp]),
    "pip_merge_workspace_bytes": (sz, [u64, u64, u64]),
    "pip_merge_u64_host": (i32, [vp, u64, u64, u64, i32]),
    "pip_merge_host_workspace_bytes": (sz, [u64, u64, u64]),
    "pip_rp_workspace_bytes": (sz, [u64, u64, i32]),
    "pip_random_permutation_u64": (
        i32, [vp, vp, u64, u64, i32, i32, vp, u64, vp, vp, sz, C.POINTER(PipRpStats), vp]),
    "pip_validate_swaps_u64": (i32, [vp, u64, vp, vp, sz, vp]),
    "pip_random_permutation_u64_host": (
        i32, [vp, vp, u64, u64, i32, C.POINTER(PipRpStats), i32]),
    "pip_rng_words_u64": (i32, [vp, u64, u64, u64, u32, vp]),
    "pip_make_swaps_u64": (i32, [vp, u64, u64, u64, vp]),
    "pip_bench_random_rmw": (i32, [vp, u64, u64, u64, C.POINTER(C.c_float), vp]),
    "pip_bench_random_update": (i32, [vp, u64, u64, u64, i32, C.POINTER(C.c_float), vp]),
    "pip_sharded_workspace_bytes": (sz, [i32]),
    "pip_nccl_available": (i32, []),
    "pip_scan_u64_sharded": (i32, [vp, u64, i32, u64, i32, vp, i32, i32, vp, sz, vp, vp, sz, vp]),
    "pip_filter_shard_plan": (i32, [C.POINTER(u64), i32, i32, u64, C.POINTER(PipShardPiece),
                                    C.POINTER(i32), C.POINTER(u64), C.POINTER(u64),
                                    C.POINTER(PipShardPiece), C.POINTER(i32)]),
    "pip_filter_u64_sharded": (i32, [vp, u64, u64, C.POINTER(PipPred), vp, i32, i32, vp, sz,
                                     C.POINTER(u64), C.POINTER(u64), vp, sz, vp]),
}


def lib_path() -> Path:
    return _LIB_PATH


def load() -> C.CDLL:
    """Load libpip.so (building it first if it is absent and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        if os.environ.get("PIP_NO_AUTOBUILD") != "1":
            from . import _build

            try:
                _build.build()
            except Exception as exc:  # pragma: no cover - depends on toolchain
                raise RuntimeError(f"libpip.so is missing and could not be built: {exc}") from exc
        if not _LIB_PATH.exists():
            raise RuntimeError(f"libpip.so not found at {_LIB_PATH}; run __graft_entry__.build()")
    lib = C.CDLL(str(_LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class PipError(RuntimeError):
    """A CUDA-side failure reported by libpip (status PIP_ERR_CUDA / OOM / ...)."""

    def __init__(self, status: int, where: str):
        lib = load()
        msg = lib.pip_status_string(status).decode()
        if status == PIP_ERR_CUDA:
            msg += f" ({lib.pip_last_cuda_error().decode()})"
        super().__init__(f"{where}: {msg} [status {status}]")
        self.status = status


def check_stall(scratch_ptr: int, stream: int, where: str) -> None:
    """Synchronize ``stream`` and raise if a look-back op queued on this
    scratch gave up waiting (PIP_ERR_STALLED: its output is incomplete)."""
    check(load().pip_scratch_status(scratch_ptr, stream), where)


def check(status: int, where: str) -> None:
    """Map a pip_status onto the reference's exception types."""
    if status == PIP_OK:
        return
    if status in (PIP_ERR_INVALID_ARG, PIP_ERR_INVALID_SWAPS, PIP_ERR_UNSORTED):
        from . import detres  # noqa: F401  (keeps import order simple)

        lib = load()
        raise ValueError(lib.pip_status_string(status).decode())
    if status == PIP_ERR_LIVELOCK:
        from .detres import LivelockError

        raise LivelockError("no iterate committed for 64 rounds; the commit rule cannot make progress")
    raise PipError(status, where)
