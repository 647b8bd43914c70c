"""Pluggable base kernels, mirroring ``mgksolver.basekernels``.

The classes keep the reference names, constructor arguments, ``flop_count``
(the cost model's X contribution) and ``with_role`` (reference
``basekernels.py:28-261``).  They carry no arithmetic on the host: each one
lowers to a small descriptor (``device_descriptor``) that the CUDA solver
evaluates in-kernel for every fused contribution.  Variants the device does
not implement raise ``NotImplementedError`` at lowering time rather than
silently falling back to the CPU.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

# descriptor kind codes shared with csrc/mgk_types.h
K_CONST1, K_DELTA, K_SE, K_POLY = 0, 1, 2, 3
MAX_POLY = 8


class KernelShapeError(ValueError):
    """Label payload does not match what the kernel variant expects."""


class KernelRangeError(ValueError):
    """Kernel evaluated outside its admissible range in validation mode."""


class BaseKernel:
    role: str = "edge"
    flop_count: int = 1

    def with_role(self, role: str) -> "BaseKernel":
        if role not in ("vertex", "edge"):
            raise ValueError(f"unknown kernel role {role!r}")
        self.role = role
        return self

    def device_descriptor(self) -> tuple[int, list[float]]:
        raise NotImplementedError(f"{type(self).__name__} has no device lowering yet")


@dataclass
class ConstantOne(BaseKernel):
    """kappa = 1 (basekernels.py:60-70)."""

    flop_count: int = 0

    def device_descriptor(self):
        return K_CONST1, []


@dataclass
class KroneckerDelta(BaseKernel):
    """1 if labels equal (all components for vectors) else h (basekernels.py:73-95)."""

    h: float
    flop_count: int = 1

    def __post_init__(self):
        if not (0 < self.h <= 1):
            raise ValueError(f"delta baseline h must be in (0, 1], got {self.h}")

    def device_descriptor(self):
        return K_DELTA, [float(self.h)]


@dataclass
class SquareExponential(BaseKernel):
    """exp(-alpha |a-b|^2) (basekernels.py:98-125)."""

    alpha: float
    flop_count: int = 4

    def __post_init__(self):
        if self.alpha <= 0:
            raise ValueError("alpha must be positive")

    def device_descriptor(self):
        return K_SE, [float(self.alpha)]


@dataclass
class CompactPolynomial(BaseKernel):
    """Horner on |a-b| of scalar labels, clamped to [0,1] (basekernels.py:128-172)."""

    coeffs: Sequence[float]
    validate: bool = False

    def __post_init__(self):
        self.coeffs = tuple(float(c) for c in self.coeffs)
        if not self.coeffs:
            raise ValueError("need at least one coefficient")
        self.flop_count = max(len(self.coeffs) - 1, 1)

    def device_descriptor(self):
        if self.validate:
            raise NotImplementedError("CompactPolynomial(validate=True) has no device lowering")
        if len(self.coeffs) > MAX_POLY:
            raise NotImplementedError(f"at most {MAX_POLY} polynomial coefficients on device")
        return K_POLY, list(self.coeffs)


SCALAR_KERNELS = (ConstantOne, KroneckerDelta, SquareExponential, CompactPolynomial)
MAX_COMPONENTS = 4


def _scalar_spec(k: BaseKernel) -> str:
    if isinstance(k, ConstantOne):
        return "const1"
    if isinstance(k, KroneckerDelta):
        return f"delta:{k.h!r}"
    if isinstance(k, SquareExponential):
        return f"se:{k.alpha!r}"
    if isinstance(k, CompactPolynomial):
        k.device_descriptor()  # raises for unsupported variants
        return "poly:" + ",".join(repr(c) for c in k.coeffs)
    raise NotImplementedError(f"{type(k).__name__} is not a scalar kernel; the device composes scalar kernels only")


@dataclass
class ProductComposite(BaseKernel):
    """Product of one scalar sub-kernel per label component (basekernels.py:175-211).

    Lowers to the device spec ``prod:K1|K2|...`` (evaluated in-kernel, csrc/mgk_dev.cuh)."""

    components: Sequence[BaseKernel]

    def __post_init__(self):
        self.components = tuple(self.components)
        self.flop_count = sum(k.flop_count for k in self.components) + max(len(self.components) - 1, 0)

    def spec(self) -> str:
        if not 1 <= len(self.components) <= MAX_COMPONENTS:
            raise NotImplementedError(f"1..{MAX_COMPONENTS} composite components on device")
        if sum(isinstance(k, CompactPolynomial) for k in self.components) > 1:
            raise NotImplementedError("at most one polynomial component on device")
        return "prod:" + "|".join(_scalar_spec(k) for k in self.components)


@dataclass
class RConvolution(BaseKernel):
    """sum_i sum_j inner(a_i, b_j) over label components (basekernels.py:214-244).

    Lowers to the device spec ``rconv:K`` (evaluated in-kernel, csrc/mgk_dev.cuh)."""

    inner: BaseKernel

    def __post_init__(self):
        self.flop_count = self.inner.flop_count + 1

    def spec(self) -> str:
        return "rconv:" + _scalar_spec(self.inner)


def kernel_from_spec(spec: str) -> BaseKernel:
    """``const1 | delta:H | se:ALPHA | poly:C0,C1,...`` (basekernels.py:247-261), plus the
    composite forms ``prod:K1|K2|...`` and ``rconv:K`` of the class-only kernels."""
    head, _, rest = spec.partition(":")
    if head == "prod":
        return ProductComposite([kernel_from_spec(p) for p in rest.split("|")])
    if head == "rconv":
        return RConvolution(kernel_from_spec(rest))
    if head == "const1":
        return ConstantOne()
    if head == "delta":
        return KroneckerDelta(h=float(rest))
    if head == "se":
        return SquareExponential(alpha=float(rest))
    if head == "poly":
        return CompactPolynomial(coeffs=[float(c) for c in rest.split(",")])
    raise ValueError(f"unknown kernel spec {spec!r}")


def as_kernel(k, role: str):
    """Accept a BaseKernel, a SPEC string or None."""
    if k is None:
        return None
    if isinstance(k, str):
        k = kernel_from_spec(k)
    if not isinstance(k, BaseKernel):
        raise TypeError(f"expected a BaseKernel or spec string, got {type(k).__name__}")
    return k.with_role(role)
