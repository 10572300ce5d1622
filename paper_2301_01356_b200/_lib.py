"""ctypes binding of ``libfastbcc_b200.so`` (the C ABI in include/fastbcc_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every entry point raises.
"""

import ctypes
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
# FBCC_LIB: an experiment build (tools/build_variant.py); default the in-tree library
LIB_PATH = Path(os.environ["FBCC_LIB"]) if os.environ.get("FBCC_LIB") else _HERE / "libfastbcc_b200.so"

FBCC_OK = 0
FBCC_ERR_ARG = 1
FBCC_ERR_TOO_LARGE = 2
FBCC_ERR_WORKSPACE = 3
FBCC_ERR_CUDA = 4
FBCC_ERR_CYCLE = 5
FBCC_ERR_COVER = 6
FBCC_FLAG_TIMING = 1
FBCC_FLAG_PROFILE = 2
FBCC_FLAG_HOST_OFFSETS32 = 4
FBCC_MAX_PROFILE = 512

# every symbol the header declares (checked by tests/test_abi.py)
EXPORTS = ("fbcc_workspace_bytes", "fbcc_run", "fbcc_run_host", "fbcc_strerror", "fbcc_last_cuda_error", "fbcc_version",
           "fbcc_kernel_name", "fbcc_plan_create", "fbcc_plan_run", "fbcc_plan_launch", "fbcc_plan_stats", "fbcc_plan_destroy",
           "fbcc_set_option", "fbcc_get_option")

OPTIONS = {"sample_rounds": 0, "giant_skip": 1, "s0": 3, "sl": 4, "compress_mask": 8, "pdl": 11, "stream_chunks": 12, "skel_parent": 13, "giant_fold": 14, "eb_staged": 15, "max_rounds": 16, "skel_max_rounds": 17, "accept_fold": 18, "detach": 19, "witness": 20}


def set_option(name: str, value: int) -> None:
    check(load().fbcc_set_option(OPTIONS[name], int(value)))


def get_option(name: str) -> int:
    return int(load().fbcc_get_option(OPTIONS[name]))


class FbccOutputs(ctypes.Structure):
    _fields_ = [("label", ctypes.c_void_p), ("head", ctypes.c_void_p), ("edge_label", ctypes.c_void_p),
                ("is_ap", ctypes.c_void_p), ("comp", ctypes.c_void_p)]


class FbccHostIO(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in ("offsets", "edges", "label", "head", "edge_label", "is_ap")]


class FbccDebug(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in
                ("forest", "parent", "first", "last", "w1", "w2", "low", "high", "fence")]


class FbccStats(ctypes.Structure):
    _fields_ = [("num_bccs", ctypes.c_int64), ("num_components", ctypes.c_int64),
                ("num_edges", ctypes.c_int64), ("stage_ms", ctypes.c_float * 6), ("total_ms", ctypes.c_float),
                ("launches", ctypes.c_int32), ("nprof", ctypes.c_int32),
                ("prof_kind", ctypes.c_int32 * 512), ("prof_ms", ctypes.c_float * 512)]


_lock = threading.Lock()
_lib = None


def load():
    """Load the extension (building it first if the .so is missing)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            from . import build

            build.build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        L.fbcc_workspace_bytes.restype = ctypes.c_int
        L.fbcc_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_size_t)]
        L.fbcc_run.restype = ctypes.c_int
        L.fbcc_run.argtypes = [P, P, ctypes.c_int64, ctypes.c_int64, P, ctypes.c_size_t,
                               ctypes.POINTER(FbccOutputs), ctypes.POINTER(FbccDebug),
                               ctypes.POINTER(FbccStats), P, ctypes.c_uint32]
        L.fbcc_run_host.restype = ctypes.c_int
        L.fbcc_run_host.argtypes = [ctypes.POINTER(FbccHostIO), ctypes.c_int64, ctypes.c_int64, P, P, P,
                                    ctypes.c_size_t, ctypes.POINTER(FbccOutputs), ctypes.POINTER(FbccStats), P,
                                    ctypes.c_uint32]
        L.fbcc_strerror.restype = ctypes.c_char_p
        L.fbcc_strerror.argtypes = [ctypes.c_int]
        L.fbcc_last_cuda_error.restype = ctypes.c_char_p
        L.fbcc_version.restype = ctypes.c_int
        L.fbcc_kernel_name.restype = ctypes.c_char_p
        L.fbcc_kernel_name.argtypes = [ctypes.c_int]
        _bind_plan(L)
        bind_ops(L)
        _lib = L
        return L


def check(rc: int) -> None:
    if rc == FBCC_OK:
        return
    L = load()
    msg = L.fbcc_strerror(rc).decode()
    if rc == FBCC_ERR_CUDA:
        raise RuntimeError(f"{msg}: {L.fbcc_last_cuda_error().decode()}")
    if rc == FBCC_ERR_WORKSPACE:
        raise MemoryError(msg)
    raise ValueError(msg)


def all_exports():
    return EXPORTS + OP_EXPORTS


def workspace_bytes(n: int, m: int) -> int:
    out = ctypes.c_size_t(0)
    check(load().fbcc_workspace_bytes(n, m, ctypes.byref(out)))
    return int(out.value)


def kernel_name(kind: int) -> str:
    return load().fbcc_kernel_name(int(kind)).decode()


def _bind_plan(L):
    P = ctypes.c_void_p
    L.fbcc_plan_create.restype = ctypes.c_int
    L.fbcc_plan_create.argtypes = [P, P, ctypes.c_int64, ctypes.c_int64, P, ctypes.c_size_t,
                                   ctypes.POINTER(FbccOutputs), ctypes.c_uint32, ctypes.POINTER(ctypes.c_void_p)]
    L.fbcc_plan_run.restype = ctypes.c_int
    L.fbcc_plan_run.argtypes = [P, ctypes.POINTER(FbccStats), P]
    L.fbcc_plan_launch.restype = ctypes.c_int
    L.fbcc_plan_launch.argtypes = [P, P]
    L.fbcc_plan_stats.restype = ctypes.c_int
    L.fbcc_plan_stats.argtypes = [P, ctypes.POINTER(FbccStats)]
    L.fbcc_plan_destroy.restype = ctypes.c_int
    L.fbcc_plan_destroy.argtypes = [P]


FBCC_ERR_RANGE = 7
FBCC_ERR_LABELS = 8
FBCC_ERR_NOT_FOREST = 9
OP_CONNECTED_COMPONENTS = 1
OP_LIST_RANKING = 2
OP_BUILD_EULER_TOUR = 3
OP_COMPUTE_TAGS = 4
OP_EXTRACT_BCCS = 5
OP_SYMMETRIZE = 6
OP_CLASSIFY_EDGES = 7
OP_EXPORTS = ("fbcc_op_workspace_bytes", "fbcc_connected_components", "fbcc_list_ranking",
              "fbcc_build_euler_tour", "fbcc_compute_tags", "fbcc_extract_bccs", "fbcc_symmetrize",
              "fbcc_classify_edges")


def bind_ops(L):
    P = ctypes.c_void_p
    I64 = ctypes.c_int64
    L.fbcc_op_workspace_bytes.restype = ctypes.c_int
    L.fbcc_op_workspace_bytes.argtypes = [ctypes.c_int, I64, I64, ctypes.POINTER(ctypes.c_size_t)]
    L.fbcc_connected_components.argtypes = [P, P, I64, I64, P, P, ctypes.c_size_t, P, P, ctypes.POINTER(I64), P]
    L.fbcc_list_ranking.argtypes = [P, I64, P, I64, P, P, ctypes.c_size_t, P]
    L.fbcc_build_euler_tour.argtypes = [I64, P, I64, P, P, P, P, P, ctypes.c_size_t, P]
    L.fbcc_compute_tags.argtypes = [P, P, I64, I64, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]
    L.fbcc_extract_bccs.argtypes = [P, P, I64, P, P, ctypes.POINTER(I64), P, ctypes.c_size_t, P]
    L.fbcc_symmetrize.argtypes = [P, P, I64, I64, P, P, ctypes.POINTER(I64), P, ctypes.c_size_t, P]
    L.fbcc_classify_edges.argtypes = [P, P, I64, I64, P, P, P, P, P, P, P, ctypes.c_size_t, P]
    for name in OP_EXPORTS[1:]:
        getattr(L, name).restype = ctypes.c_int


def op_workspace_bytes(op: int, a: int, b: int = 0) -> int:
    out = ctypes.c_size_t(0)
    check(load().fbcc_op_workspace_bytes(op, int(a), int(b), ctypes.byref(out)))
    return int(out.value)
