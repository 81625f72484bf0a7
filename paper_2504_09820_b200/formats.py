"""Floating-point format descriptors (host-side knobs only).

Mirrors the reference's FloatFormat / make_format / get_format registry
(formats.py:51-188) so detector configurations read the same.  No arithmetic
happens here: the formats are passed to the CUDA library as
(sig_bits, exp_bits, subnormals) and every rounding runs on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import FormatError

__all__ = ["FloatFormat", "make_format", "get_format", "registered_formats",
           "BFLOAT16", "FP16", "FP32", "FP64"]


@dataclass(frozen=True)
class FloatFormat:
    name: str
    sig_bits: int
    exp_bits: int
    subnormals_enabled: bool = True
    unit_roundoff: float = field(init=False, compare=False)
    x_min: float = field(init=False, compare=False)   # smallest positive normal, 2**(1 - bias)
    x_max: float = field(init=False, compare=False)   # largest finite, (2 - 2**(1 - sig)) * 2**bias

    def __post_init__(self):
        if self.sig_bits < 2 or self.exp_bits < 2:
            raise FormatError(f"need sig_bits >= 2 and exp_bits >= 2, got ({self.sig_bits}, {self.exp_bits})")
        if self.sig_bits > 53 or self.exp_bits > 11:
            raise FormatError(f"({self.sig_bits}, {self.exp_bits}) exceeds the binary64 substrate (53, 11)")
        object.__setattr__(self, "unit_roundoff", 2.0 ** (-self.sig_bits))
        bias = (1 << (self.exp_bits - 1)) - 1
        object.__setattr__(self, "x_min", 2.0 ** (1 - bias))
        object.__setattr__(self, "x_max", (2.0 - 2.0 ** (1 - self.sig_bits)) * 2.0 ** bias)

    @property
    def is_native(self) -> bool:
        return self.sig_bits == 53 and self.exp_bits == 11 and self.subnormals_enabled

    def triple(self):
        return (self.sig_bits, self.exp_bits, 1 if self.subnormals_enabled else 0)


def make_format(sig_bits: int, exp_bits: int, *, subnormals_enabled: bool = True,
                name: str | None = None) -> FloatFormat:
    return FloatFormat(name or f"p{sig_bits}e{exp_bits}", int(sig_bits), int(exp_bits),
                       subnormals_enabled=subnormals_enabled)


BFLOAT16 = make_format(8, 8, name="bfloat16")
FP16 = make_format(11, 5, name="fp16")
FP32 = make_format(24, 8, name="fp32")
FP64 = make_format(53, 11, name="fp64")
_REGISTRY = {f.name: f for f in (BFLOAT16, FP16, FP32, FP64)}


def registered_formats() -> dict:
    return dict(_REGISTRY)


def get_format(name) -> FloatFormat:
    if isinstance(name, FloatFormat):
        return name
    if hasattr(name, "sig_bits") and hasattr(name, "exp_bits"):   # a reference FloatFormat
        return make_format(name.sig_bits, name.exp_bits,
                           subnormals_enabled=getattr(name, "subnormals_enabled", True),
                           name=getattr(name, "name", None))
    try:
        return _REGISTRY[name]
    except KeyError:
        raise FormatError(f"unknown format {name!r}; registry has: {', '.join(sorted(_REGISTRY))}") from None
