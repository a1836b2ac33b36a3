"""ctypes binding of the C ABI in include/lars_b200.h (liblars_b200.so).

There is deliberately no fallback: if the library is missing or fails to
load, importing the step API raises.  `build.py` produces the library in-tree.
"""

import ctypes
import os

from .errors import NativeError

_LIB_NAME = os.environ.get("LARS_B200_LIB", "liblars_b200.so")  # liblars_b200_trace.so: profiling
_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", _LIB_NAME)

LARS_OK = 0
LARS_ERR_INVALID = 1
LARS_ERR_ALIGNMENT = 2
LARS_ERR_LAYOUT = 3
LARS_ERR_TOO_MANY_PIECES = 4
LARS_ERR_NO_DEVICE = 5
LARS_ERR_HOST_ONLY_PLAN = 6
LARS_ERR_HOST_MEMORY = 7
LARS_SEG_TRUST = 1
LARS_SEG_SHARED = 2
LARS_STEP_EXPLICIT_LR = 1
LARS_STEP_USE_WCARRY = 2
LARS_STEP_ADVANCE_ITER = 4
LARS_STATUS_EXHAUSTED = 1
LARS_STATUS_RANK_TIMEOUT = 2
LARS_PLAN_HOST_ONLY = 1
INT32_MAX = 2**31 - 1

EXPORTED = (
    "lars_plan_create", "lars_plan_info", "lars_plan_partition", "lars_plan_destroy",
    "lars_workspace_init", "lars_step", "lars_partial_norms", "lars_update", "lars_step_peer",
    "lars_step_peer_stream", "lars_peer_barrier", "lars_host_register", "lars_host_unregister", "lars_host_copy_in", "lars_host_copy_out",
    "lars_strerror", "lars_abi_version",
)


class Segment(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("length", ctypes.c_int64),
                ("layer", ctypes.c_int32), ("flags", ctypes.c_int32)]


class HParams(ctypes.Structure):
    _fields_ = [("base_lr", ctypes.c_double), ("momentum", ctypes.c_double),
                ("weight_decay", ctypes.c_double), ("poly_power", ctypes.c_double),
                ("trust", ctypes.c_double), ("grad_scale", ctypes.c_double),
                ("lr", ctypes.c_double), ("warmup_iters", ctypes.c_int64),
                ("max_iters", ctypes.c_int64), ("lars_enabled", ctypes.c_int32),
                ("flags", ctypes.c_int32)]


class StepInfo(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("iteration", ctypes.c_int64),
                ("nonfinite_layer", ctypes.c_int32), ("status", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("grid", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("nseg", ctypes.c_int32), ("nlayers", ctypes.c_int32),
                ("npieces", ctypes.c_int64), ("nbatches", ctypes.c_int64),
                ("elements", ctypes.c_int64), ("max_pieces_cta", ctypes.c_int32),
                ("max_slots_cta", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("workspace_bytes", ctypes.c_int64)]


MAX_RANKS = 8


class Peer(ctypes.Structure):
    _fields_ = [("w_peer", ctypes.c_void_p * MAX_RANKS), ("g_peer", ctypes.c_void_p * MAX_RANKS),
                ("x_peer", ctypes.c_void_p * MAX_RANKS), ("f_peer", ctypes.c_void_p * MAX_RANKS),
                ("g_shard", ctypes.c_void_p), ("m", ctypes.c_void_p),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32)]


class HostSpan(ctypes.Structure):
    _fields_ = [("host", ctypes.c_void_p), ("offset", ctypes.c_int64), ("numel", ctypes.c_int64)]


STEP_INFO_BYTES = ctypes.sizeof(StepInfo)

_lib = None


def lib_path():
    return _LIB_PATH


def load():
    """Load liblars_b200.so (once).  Raises if it is missing: no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} not found: build it with `python -m paper_1709_05011_b200.build` "
            "(the LARS step has no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.lars_plan_create.argtypes = [ctypes.POINTER(Segment), i32, i32, i32, i32,
                                     ctypes.POINTER(vp)]
    lib.lars_plan_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    lib.lars_plan_partition.argtypes = [vp, vp, vp, vp]
    lib.lars_plan_destroy.argtypes = [vp]
    lib.lars_plan_destroy.restype = None
    lib.lars_workspace_init.argtypes = [vp, vp, vp]
    lib.lars_step.argtypes = [vp, vp, vp, vp, ctypes.POINTER(HParams), vp, vp, vp, vp, vp, vp]
    lib.lars_partial_norms.argtypes = [vp, vp, vp, ctypes.POINTER(HParams), vp, vp, vp, vp, vp]
    lib.lars_update.argtypes = [vp, vp, vp, vp, ctypes.POINTER(HParams), vp, vp, vp, vp, vp]
    lib.lars_step_peer.argtypes = [vp, ctypes.POINTER(Peer), ctypes.POINTER(HParams), vp, vp, vp,
                                   vp, vp, vp]
    lib.lars_step_peer_stream.argtypes = lib.lars_step_peer.argtypes
    lib.lars_peer_barrier.argtypes = [ctypes.POINTER(Peer), vp, vp, vp]
    lib.lars_host_register.argtypes = [vp, i64]
    lib.lars_host_unregister.argtypes = [vp]
    lib.lars_host_copy_in.argtypes = [ctypes.POINTER(HostSpan), i32, vp, vp, i64, vp]
    lib.lars_host_copy_out.argtypes = [vp, vp, i64, ctypes.POINTER(HostSpan), i32, vp]
    lib.lars_strerror.argtypes = [ctypes.c_int]
    lib.lars_strerror.restype = ctypes.c_char_p
    lib.lars_abi_version.argtypes = []
    for name in ("lars_plan_create", "lars_plan_info", "lars_plan_partition",
                 "lars_workspace_init", "lars_step", "lars_partial_norms", "lars_update", "lars_step_peer",
                 "lars_step_peer_stream", "lars_peer_barrier", "lars_host_register", "lars_host_unregister", "lars_host_copy_in",
                 "lars_host_copy_out", "lars_abi_version"):
        getattr(lib, name).restype = ctypes.c_int
    if lib.lars_abi_version() != 1:
        raise ImportError(f"liblars_b200 ABI {lib.lars_abi_version()} != 1")
    _lib = lib
    return lib


def check(rc):
    if rc != LARS_OK:
        lib = load()
        raise NativeError(rc, lib.lars_strerror(rc).decode())
    return rc
