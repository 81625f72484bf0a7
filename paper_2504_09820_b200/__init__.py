"""B200-native batched FP-CG / FP-BJ-CG massive-MIMO detector.

Drop-in for the hot path of the reference package `fpmimo`
(Gram/matched filter -> block-Jacobi -> mixed-precision CG -> QAM slicing ->
error counts).  All computation runs in hand-written sm_100a CUDA kernels
(libfpmimo_b200.so, C ABI in include/fpmimo_b200.h); this package is the
host-side mirror of the reference's detector API.
"""

from .errors import ContractViolation, FormatError  # noqa: F401
from .formats import BFLOAT16, FP16, FP32, FP64, FloatFormat, get_format, make_format  # noqa: F401

__version__ = "1.0.0"


def __getattr__(name):
    # lazy: importing the package must not require torch / CUDA
    if name in ("solvers", "detect", "parallel"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
