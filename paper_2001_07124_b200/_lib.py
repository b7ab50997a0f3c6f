"""ctypes declarations of librtucker (include/rtucker.h).  Argument marshalling only.

The product path has no fallback: if the in-tree CUDA library is missing this
module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "librtucker.so")

RT_OK, RT_EINVAL, RT_ERANK, RT_ENOMEM, RT_ECUDA, RT_ENCCL, RT_ENUMERIC, RT_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "RT_OK", -1: "RT_EINVAL", -2: "RT_ERANK", -3: "RT_ENOMEM", -4: "RT_ECUDA", -5: "RT_ENCCL",
                -6: "RT_ENUMERIC", -7: "RT_EUNSUPPORTED"}
RT_F32, RT_F64 = 0, 1
RT_OMEGA_GAUSS, RT_OMEGA_KRON, RT_OMEGA_KR, RT_OMEGA_COUNT = 0, 1, 2, 3
RT_OPT_TTM_IMPL, RT_OPT_PROFILE, RT_OPT_QR_FALLBACK, RT_OPT_OMEGA_TF32, RT_OPT_TC_SEGMENT, RT_OPT_TC_SKEW = 0, 1, 2, 3, 4, 5
RT_OPT_FORCE_COLLECTIVES = 6
RT_OPT_TC_ABLATE = 100          # profiling / A-B switches (210/211: fp16-split power product off/on)

EXPORTS = ["rt_get_unique_id", "rt_create", "rt_loopback_group_create", "rt_loopback_group_destroy",
           "rt_create_loopback", "rt_destroy", "rt_last_error", "rt_sync", "rt_set_option", "rt_profile_read",
           "rtucker_sketch", "rtucker_qr", "rtucker_core", "rtucker_hosvd", "rtucker_sthosvd", "rtucker_pet", "rtucker_rp_hooi"]


class rt_tensor(C.Structure):
    _fields_ = [("dtype", C.c_int), ("order", C.c_int), ("dims", C.c_int64 * 5),
                ("last_offset", C.c_int64), ("last_global", C.c_int64), ("data", C.c_void_p)]


class rt_profile_entry(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("count", C.c_int64), ("ms", C.c_double)]


class RtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"librtucker.so not built ({LIB_PATH}); run `python -m paper_2001_07124_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    P, I64, I, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
    PP = C.POINTER(C.c_void_p)
    PI64 = C.POINTER(C.c_int64)
    sig = {
        "rt_get_unique_id": (I, [C.POINTER(C.c_uint8)]),
        "rt_create": (I, [C.POINTER(P), P, C.POINTER(C.c_uint8), I, I]),
        "rt_loopback_group_create": (I, [C.POINTER(P), I]),
        "rt_loopback_group_destroy": (I, [P]),
        "rt_create_loopback": (I, [C.POINTER(P), P, P, I]),
        "rt_destroy": (I, [P]),
        "rt_last_error": (C.c_char_p, [P]),
        "rt_sync": (I, [P]),
        "rt_set_option": (I, [P, I, I64]),
        "rt_profile_read": (I, [P, C.POINTER(rt_profile_entry), I, C.POINTER(I), C.POINTER(I64)]),
        "rtucker_sketch": (I, [P, C.POINTER(rt_tensor), I, I, PP, PI64, PI64, I, P, I64]),
        "rtucker_qr": (I, [P, I64, I64, I, P, I64, P, I64, P, I]),
        "rtucker_core": (I, [P, C.POINTER(rt_tensor), PP, PI64, P, P, P]),
        "rtucker_hosvd": (I, [P, C.POINTER(rt_tensor), PI64, I, I, I, PP, PI64, PI64, PP, P, P, P]),
        "rtucker_sthosvd": (I, [P, C.POINTER(rt_tensor), PI64, I, I, I, PP, PI64, PI64, C.POINTER(C.c_int), PP, P,
                                P, P]),
        "rtucker_pet": (I, [P, C.POINTER(rt_tensor), PI64, PP, PI64, PI64, PP, PI64, PI64, PP, P, P, P]),
        "rtucker_rp_hooi": (I, [P, C.POINTER(rt_tensor), PI64, I, PP, PP, PI64, PP, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()
