"""B200-native randomized Tucker / HOSVD hot path (arXiv 2001.07124, §V).

C-ABI library ``lib/librtucker.so`` (include/rtucker.h) + a thin ctypes binding
(``api``).  Build with ``python -m paper_2001_07124_b200.build``.  Attribute access
loads the CUDA library; there is no CPU fallback (ImportError if it is missing).
"""
__all__ = ["Handle", "LoopbackGroup", "get_unique_id", "tensor_desc", "colmajor", "new_colmajor",
           "rtucker_sketch", "rtucker_qr", "rtucker_core", "rtucker_hosvd", "rtucker_sthosvd",
           "core_to_numpy", "RtError"]


def __getattr__(name):
    if name in __all__:
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
