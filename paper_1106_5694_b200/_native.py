"""ctypes binding of the C-ABI in include/lsapgpu.h (liblsapgpu.so, built in-tree).

The shared library is the product: it holds the sm_100a kernels and the host
orchestration.  There is no fallback: if the library is missing the import of
this module raises, and if no sm_100 device is present ``Context()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "lib", "liblsapgpu.so")

OK, ERR_INVALID, ERR_CUDA, ERR_INTERNAL, ERR_STATE = 0, 1, 2, 3, 4
F64, F32, I32, I16 = 0, 1, 2, 3
STORAGE_NAMES = {0: "int16", 1: "int32", 2: "fp32", 3: "fp64"}
STORAGE_BYTES = {0: 2, 1: 4, 2: 4, 3: 8}
GEN = {"int": 1, "f32": 2, "unit": 3, "p2p": 4, "geom": 5}

EXPORTS = [
    "lsapgpu_version", "lsapgpu_device_count", "lsapgpu_create", "lsapgpu_destroy",
    "lsapgpu_last_error", "lsapgpu_stream", "lsapgpu_set_matrix", "lsapgpu_set_matrix_device",
    "lsapgpu_generate", "lsapgpu_n", "lsapgpu_storage", "lsapgpu_read_rows", "lsapgpu_solve",
    "lsapgpu_evaluate_all", "lsapgpu_check_conflicts", "lsapgpu_apply_parallel_switches",
    "lsapgpu_random_perm", "lsapgpu_objective", "lsapgpu_counters", "lsapgpu_solve_dist",
    "lsapgpu_dist_exchange_bytes", "lsapgpu_set_scan_timing", "lsapgpu_scan_timing", "lsapgpu_scan_plan",
    "lsapgpu_set_placement",
    "lsapgpu_set_timeline", "lsapgpu_timeline", "lsapgpu_auction_solve",
    "lsapgpu_greedy_assignment",
    "lsapgpu_dist_p2p_bytes", "lsapgpu_ipc_handle", "lsapgpu_ipc_open", "lsapgpu_ipc_close",
    "lsapgpu_dev_alloc", "lsapgpu_dev_free",
]


class Params(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("eps", C.c_double),
        ("reeval", C.c_int32),
        ("use_graph", C.c_int32),
        ("deadline_ns", C.c_int64),
        ("init_sigma", C.c_void_p),
        ("init_mode", C.c_int32),
        ("pad_", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("outer_iterations", C.c_int64),
        ("switches_applied", C.c_int64),
        ("terminated_by", C.c_int32),
        ("value", C.c_double),
        ("elapsed_ms", C.c_double),
        ("inner_iterations", C.c_int64),
        ("pair_items", C.c_int64),
        ("agent_scans", C.c_int64),
        ("job_scans", C.c_int64),
        ("lfmm_rounds", C.c_int64),
        ("scan_launches", C.c_int64),
        ("bytes_scanned", C.c_int64),
        ("storage", C.c_int32),
        ("scan_filter", C.c_int32),
        ("filter_kept", C.c_int64),
        ("filter_overflows", C.c_int64),
        ("host_log_orders", C.c_int64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}


class AuctionParams(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double),
        ("has_epsilon", C.c_int32),
        ("scaling", C.c_int32),
        ("scale_factor", C.c_double),
        ("deadline_ns", C.c_int64),
    ]


class AuctionStats(C.Structure):
    _fields_ = [
        ("outer_iterations", C.c_int64),
        ("switches_applied", C.c_int64),
        ("terminated_by", C.c_int32),
        ("completed_greedily", C.c_int32),
        ("value", C.c_double),
        ("elapsed_ms", C.c_double),
        ("bids", C.c_int64),
        ("phases", C.c_int64),
        ("epsilon", C.c_double),
        ("bytes_scanned", C.c_int64),
        ("storage", C.c_int32),
        ("scan_filter", C.c_int32),
        ("filter_kept", C.c_int64),
        ("filter_overflows", C.c_int64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class Dist(C.Structure):
    _fields_ = [
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("allgather", ALLGATHER_FN),
        ("user", C.c_void_p),
        ("send_dev", C.c_void_p),
        ("recv_dev", C.c_void_p),
        ("peer_recv", C.POINTER(C.c_void_p)),
        ("peer_flags", C.POINTER(C.c_void_p)),
    ]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    sig = {
        "lsapgpu_version": (C.c_char_p, []),
        "lsapgpu_device_count": (C.c_int, []),
        "lsapgpu_create": (C.c_int, [C.POINTER(vp), C.c_int]),
        "lsapgpu_destroy": (None, [vp]),
        "lsapgpu_last_error": (C.c_char_p, [vp]),
        "lsapgpu_stream": (vp, [vp]),
        "lsapgpu_set_matrix": (C.c_int, [vp, vp, i32, i32]),
        "lsapgpu_set_matrix_device": (C.c_int, [vp, vp, i32, i32]),
        "lsapgpu_generate": (C.c_int, [vp, i32, i32, u64, dbl]),
        "lsapgpu_n": (i32, [vp]),
        "lsapgpu_storage": (i32, [vp]),
        "lsapgpu_read_rows": (C.c_int, [vp, vp, i32, vp]),
        "lsapgpu_solve": (C.c_int, [vp, C.POINTER(Params), vp, vp, C.POINTER(Stats), vp, vp, i64,
                                    C.POINTER(i64)]),
        "lsapgpu_evaluate_all": (C.c_int, [vp, vp, dbl, vp, vp, vp, vp]),
        "lsapgpu_check_conflicts": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                              C.POINTER(i32)]),
        "lsapgpu_apply_parallel_switches": (C.c_int, [vp, vp, vp, C.POINTER(dbl), vp, vp, vp, vp, vp,
                                                      vp, vp, vp, dbl, vp, vp, vp, vp, vp,
                                                      C.POINTER(i32)]),
        "lsapgpu_random_perm": (None, [i32, u64, vp]),
        "lsapgpu_objective": (C.c_int, [vp, vp, C.POINTER(dbl)]),
        "lsapgpu_counters": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
        "lsapgpu_solve_dist": (C.c_int, [vp, C.POINTER(Params), C.POINTER(Dist), vp, vp, C.POINTER(Stats), vp, vp,
                                         i64, C.POINTER(i64)]),
        "lsapgpu_dist_exchange_bytes": (C.c_size_t, [i32, i32]),
        "lsapgpu_dist_p2p_bytes": (C.c_size_t, [i32, i32]),
        "lsapgpu_ipc_handle": (C.c_int, [vp, vp]),
        "lsapgpu_dev_alloc": (C.c_int, [C.c_int, C.c_size_t, C.POINTER(vp)]),
        "lsapgpu_dev_free": (C.c_int, [C.c_int, vp]),
        "lsapgpu_ipc_open": (C.c_int, [vp, C.POINTER(vp)]),
        "lsapgpu_ipc_close": (C.c_int, [vp]),
        "lsapgpu_set_scan_timing": (C.c_int, [vp, C.c_int]),
        "lsapgpu_set_timeline": (C.c_int, [vp, C.c_int32]),
        "lsapgpu_timeline": (C.c_int32, [vp, C.c_void_p, C.c_int32]),
        "lsapgpu_auction_solve": (C.c_int, [vp, C.POINTER(AuctionParams), vp, vp, C.POINTER(AuctionStats),
                                            vp, vp, i64]),
        "lsapgpu_greedy_assignment": (C.c_int, [vp, vp, C.POINTER(i64)]),
        "lsapgpu_scan_plan": (C.c_int, [vp, vp, C.c_int32]),
        "lsapgpu_set_placement": (C.c_int, [vp, C.c_int32, C.c_int32]),
        "lsapgpu_scan_timing": (C.c_int, [vp, C.POINTER(dbl), C.POINTER(i64), C.POINTER(dbl),
                                          C.POINTER(i64), C.POINTER(dbl), C.POINTER(i64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
