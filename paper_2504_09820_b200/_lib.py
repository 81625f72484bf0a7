"""ctypes binding of libfpmimo_b200.so (C ABI: include/fpmimo_b200.h).

The library is REQUIRED: there is no CPU fallback anywhere in this package.
If the shared object is missing or no CUDA device is present, calls raise.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ContractViolation

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FPM_LIB") or os.path.join(_HERE, "libfpmimo_b200.so")  # FPM_LIB: dev variants

FPM_OK, FPM_EINVAL, FPM_ENOTPD, FPM_ECUDA, FPM_EUNSUPPORTED = range(5)
FPM_RHO = {"as_written": 0, "textbook": 1}
FPM_ALG = {"lmmse": 0, "cg": 1, "fp_cg": 2, "fp_bj_cg": 3}
FPM_FLAG_GRAM_FP32 = 0x100
COUNTERS = ("bit_errors", "symbol_errors", "diverged", "breakdown", "trials", "nonpd")
NCOUNTERS = 8

# every symbol include/fpmimo_b200.h declares
EXPORTS = ("fpm_version", "fpm_strerror", "fpm_limits", "fpm_gram", "fpm_bj_setup", "fpm_cg", "fpm_cg_ex", "fpm_residual_gaps", "fpm_herm_norm2", "fpm_lmmse", "fpm_gen_trials", "fpm_simulate", "fpm_gram32",
           "fpm_slice_count", "fpm_detect", "fpm_detect_host", "fpm_launch_count", "fpm_last_kernel", "fpm_probe_fp64",
           "fpm_debug_set_trace")


class Format(ctypes.Structure):
    _fields_ = [("sig_bits", ctypes.c_int32), ("exp_bits", ctypes.c_int32), ("subnormals", ctypes.c_int32)]


class Precision(ctypes.Structure):
    _fields_ = [("work", Format), ("matvec", Format), ("inner", Format)]


class CgHistory(ctypes.Structure):
    """fpm_cg_history (include/fpmimo_b200.h): device pointers, NULL = skip."""
    _fields_ = [("residual_norms", ctypes.c_void_p), ("iterate_norms", ctypes.c_void_p),
                ("alphas", ctypes.c_void_p), ("betas", ctypes.c_void_p), ("converged_at", ctypes.c_void_p),
                ("rtol", ctypes.c_double), ("iterates", ctypes.c_void_p), ("residual_vectors", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double

_SIGS = {
    "fpm_version": (ctypes.c_int, []),
    "fpm_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "fpm_limits": (ctypes.c_int, [_P, _P, _P]),
    "fpm_gram": (ctypes.c_int, [_P, _P, _I64, _I32, _I32, _D, _P, _P, _P]),
    "fpm_bj_setup": (ctypes.c_int, [_P, _I64, _I32, _I32, _I32, _P, _P, _P]),
    "fpm_cg": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _I32, ctypes.POINTER(Precision), _I32,
                              _P, _P, _P, _P]),
    "fpm_cg_ex": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _I32, ctypes.POINTER(Precision), _I32,
                                 _P, _P, _P, ctypes.POINTER(CgHistory), _P]),
    "fpm_residual_gaps": (ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I32, _I32, _P, _P]),
    "fpm_herm_norm2": (ctypes.c_int, [_P, _I64, _I32, _P, _P]),
    "fpm_lmmse": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P, _P]),
    "fpm_gram32": (ctypes.c_int, [_P, _P, _I64, _I32, _I32, _D, _P, _P, _P]),
    "fpm_gen_trials": (ctypes.c_int, [ctypes.c_uint64, _I32, _I32, _I64, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P]),
    "fpm_simulate": (ctypes.c_int, [ctypes.c_uint64, _I32, _I32, _I64, _I64, _I32, _I32, _D, _D, _I32, _I32, _I32,
                                    _D, _D, _P, _P, _P, _P, _P, _P]),
    "fpm_slice_count": (ctypes.c_int, [_P, _P, _I64, _I32, _I32, _P, _P, _P]),
    "fpm_detect": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _D, _I32, _I32, _I32,
                                  ctypes.POINTER(Precision), _I32, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "fpm_detect_host": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _D, _I32, _I32, _I32,
                                       ctypes.POINTER(Precision), _I32, _I32, _P, _P, _P, _P, _P, _P, _I64]),
    "fpm_launch_count": (ctypes.c_int64, []),
    "fpm_last_kernel": (ctypes.c_char_p, []),
    "fpm_probe_fp64": (ctypes.c_int, [_I64, ctypes.POINTER(ctypes.c_double)]),
    "fpm_debug_set_trace": (ctypes.c_int, [_P]),
}

_lib = None


def load():
    """Load (once) and return the CDLL; raises if the library is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built (run `python -c 'import __graft_entry__ as g; "
                               f"g.build()'`); this package has no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str):
    if rc == FPM_OK:
        return
    msg = load().fpm_strerror(rc).decode()
    if rc in (FPM_EINVAL, FPM_ENOTPD):
        raise ContractViolation(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg} (code {rc})")


def precision_struct(prec) -> Precision:
    """prec: object with .work/.matvec/.inner FloatFormat-likes."""
    def f(x):
        return Format(int(x.sig_bits), int(x.exp_bits), 1 if getattr(x, "subnormals_enabled", True) else 0)
    return Precision(f(prec.work), f(prec.matvec), f(prec.inner))
