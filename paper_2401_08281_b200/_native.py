"""ctypes binding of libflatknn.so (the C ABI in ``include/flatknn.h``).

ctypes releases the GIL for the duration of every call, matching the
reference's nogil Cython loops (``_ckernels.pyx:149,157,173``).  There is no
CPU fallback: if the library is missing, importing the index raises.
"""

from __future__ import annotations

import ctypes
import os

from .build import DEV_LIB_PATH, LIB_PATH

FK_METRIC_IP = 0
FK_METRIC_L2 = 1
FK_F32, FK_F16, FK_BF16 = 0, 1, 2

FK_OK = 0
FK_E_INVALID = -1
FK_E_CUDA = -2
FK_E_NOMEM = -3
FK_E_UNSUPPORTED = -4
FK_E_NOTFOUND = -5

# every symbol include/flatknn.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "fk_create", "fk_add", "fk_search", "fk_merge_shards", "fk_reconstruct", "fk_remove_ids",
    "fk_reset", "fk_ntotal", "fk_dim", "fk_get_ids", "fk_destroy", "fk_last_error",
    "fk_set_profiling", "fk_kernel_times", "fk_last_plan", "fk_kmeans_rescore",
    "fk_range_search", "fk_range_fetch", "fk_range_total", "fk_range_free", "fk_set_option",
    "fk_positions", "fk_refine", "fk_gate",
    "fk_xchg_handle_bytes", "fk_xchg_create", "fk_xchg_connect", "fk_xchg_acquire", "fk_xchg_put",
    "fk_xchg_merge", "fk_xchg_status", "fk_xchg_destroy",
)

FK_OPT_PLAN_ROWS = 1
FK_OPT_BLAS_THRESHOLD = 2

_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_INT = ctypes.c_int

_SIGS = {
    "fk_create": (_INT, [_INT, _INT, _INT, _INT, ctypes.POINTER(_P)]),
    "fk_add": (_INT, [_P, _P, _I64, _INT, _P, _INT, _P]),
    "fk_search": (_INT, [_P, _P, _I64, _INT, _INT, _P, _P, _P, _INT, _P]),
    "fk_merge_shards": (_INT, [_INT, _INT, _I64, _INT, _P, _P, _P, _P, _P, _P]),
    "fk_reconstruct": (_INT, [_P, _P, _I64, _P, _INT, _P]),
    "fk_remove_ids": (_INT, [_P, _P, _I64, _INT, ctypes.POINTER(_I64), _P]),
    "fk_reset": (_INT, [_P]),
    "fk_ntotal": (_I64, [_P]),
    "fk_dim": (_INT, [_P]),
    "fk_get_ids": (_INT, [_P, _P]),
    "fk_destroy": (None, [_P]),
    "fk_last_error": (ctypes.c_char_p, []),
    "fk_set_profiling": (_INT, [_P, _INT]),
    "fk_kernel_times": (_INT, [_P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(_INT)]),
    "fk_last_plan": (_INT, [_P, ctypes.POINTER(_INT)]),
    "fk_range_search": (_INT, [_P, _P, _I64, _INT, ctypes.c_float, _P, ctypes.POINTER(_I64), ctypes.POINTER(_P),
                               _INT, _P]),
    "fk_range_fetch": (_INT, [_P, _P, _P, _I64, _INT, _P]),
    "fk_range_total": (_I64, [_P]),
    "fk_range_free": (None, [_P]),
    "fk_set_option": (_INT, [_P, _INT, _I64]),
    "fk_gate": (_INT, [_P, ctypes.c_double, _P]),
    "fk_xchg_handle_bytes": (_INT, []),
    "fk_xchg_create": (_INT, [_INT, _INT, _INT, _I64, _INT, ctypes.POINTER(_P), _P]),
    "fk_xchg_connect": (_INT, [_P, _P]),
    "fk_xchg_acquire": (_INT, [_P, _P]),
    "fk_xchg_put": (_INT, [_P, _I64, _INT, _P, _P, _P, _P]),
    "fk_xchg_merge": (_INT, [_P, _INT, _I64, _INT, _P, _P, _P]),
    "fk_xchg_status": (_INT, [_P]),
    "fk_xchg_destroy": (None, [_P]),
    "fk_positions": (_INT, [_P, _P, _I64, _P, _INT, _P]),
    "fk_refine": (_INT, [_P, _INT, _P, _I64, _P, _INT, _INT, _P, _P, _INT, _P]),
    "fk_kmeans_rescore": (_INT, [_P, _I64, _INT, _P, _P, _I64, _P, _INT, _INT, _P, ctypes.c_double,
                                 ctypes.c_double, _P, _P, _P, _P]),
    "fk_debug_set_ip_dump": (_INT, [_P, _P]),
    "fk_debug_set_trace": (_INT, [_P, _P]),
}


class NativeError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Load (once) and return the CUDA library; raises if it was not built."""
    global _lib
    if _lib is None:
        path = DEV_LIB_PATH if os.environ.get("FK_DEV_LIB") == "1" else LIB_PATH
        if os.environ.get("FK_LIB_VARIANT"):  # experiment builds (scripts only)
            from .build import variant_path
            path = variant_path(os.environ["FK_LIB_VARIANT"])
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: the CUDA extension is not built "
                "(run `python -m paper_2401_08281_b200.build`). There is no CPU fallback.")
        L = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a C-ABI return code to the reference's exception types."""
    if rc == FK_OK:
        return
    msg = lib().fk_last_error().decode(errors="replace")
    if rc == FK_E_INVALID:
        raise ValueError(msg)
    if rc == FK_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == FK_E_NOTFOUND:
        raise KeyError(msg)
    if rc == FK_E_NOMEM:
        raise MemoryError(msg)
    raise NativeError(msg)
