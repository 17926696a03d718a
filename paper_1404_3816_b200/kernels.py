"""Kernel (generalized covariance function) description.

Mirror of the reference KernelSpec (kernels.py:25-69): same fields, the same
validation and ValueError messages.  The kernel is evaluated only on the GPU
(inside the P2P / M2L operator kernels of libhikf_b200.so); this module only
describes it and converts it to the C-ABI struct.  Reference KernelSpec
objects are accepted anywhere a KernelSpec is (duck-typed on the fields).
"""

from __future__ import annotations

from dataclasses import dataclass

from ._lib import FAMILY_CODE, HikfKernel

_FAMILIES = ("gaussian", "exponential", "logarithm")
_DEFAULT_POWER = {"gaussian": 2.0, "exponential": 1.0}


@dataclass(frozen=True)
class KernelSpec:
    family: str
    variance: float = 1.0
    length_scale: float = 1.0
    power: float | None = None
    log_amplitude: float | None = None

    def __post_init__(self):
        if self.family not in _FAMILIES:
            raise ValueError(f"unknown kernel family {self.family!r}; expected one of {_FAMILIES}")
        if self.family == "logarithm":
            if self.log_amplitude is None or not self.log_amplitude < 0:
                raise ValueError("logarithm family requires log_amplitude < 0")
        else:
            if not self.variance >= 0:
                raise ValueError("variance must be >= 0")
            if not self.length_scale > 0:
                raise ValueError("length_scale must be > 0")
            if not (0 < self.effective_power <= 2):
                raise ValueError("power must lie in (0, 2]")

    @property
    def effective_power(self) -> float:
        if self.family == "logarithm":
            raise ValueError("logarithm family has no power parameter")
        return _DEFAULT_POWER[self.family] if self.power is None else float(self.power)


def value_at_zero(spec) -> float:
    """kernels.py:91-95: K(0), with the logarithm diagonal 0 by convention."""
    return 0.0 if spec.family == "logarithm" else float(spec.variance)


def to_c(spec) -> HikfKernel:
    """C-ABI kernel struct from a KernelSpec (ours or the reference's)."""
    fam = spec.family
    if fam not in FAMILY_CODE:
        raise ValueError(f"unknown kernel family {fam!r}")
    if fam == "logarithm":
        return HikfKernel(FAMILY_CODE[fam], 0.0, 1.0, 1.0, float(spec.log_amplitude))
    power = _DEFAULT_POWER[fam] if spec.power is None else float(spec.power)
    return HikfKernel(FAMILY_CODE[fam], float(spec.variance), float(spec.length_scale), power, 0.0)
