"""Quantizer / sign-policy configuration of the drop-in API.

``QuantSpec`` and ``SignPolicy`` take the reference's constructor arguments
and validation (lioncomm/quant.py:102-153).  On the CUDA path the quantizer
itself runs inside the fused interpolate kernel (csrc/kernels.cu, K1) and the
per-layer L1 norm in csrc/l1norm.cu; only the finite-p=1 nearest-rounding
quantizer (the paper's Lion Cub p-bit scheme) is on the hot path, other
variants raise ``ConfigError`` from the step.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError

PACKABLE_WIDTHS = (1, 2, 4, 8)
INF = float("inf")
ZERO_MODES = ("exact-ternary", "alternating")
ROUNDINGS = ("nearest", "stochastic")


@dataclass(frozen=True)
class QuantSpec:
    """Levels in [-qmax, qmax] with qmax = 2**(bits-1) - 1; scale by the mean
    p-norm ``norm_p`` (0 = geometric mean, inf = max norm)."""

    bits: int = 8
    norm_p: float = 1.0
    rounding: str = "nearest"
    log_transform: bool = False
    no_zero: bool = False

    def __post_init__(self):
        if self.bits < 1:
            raise ConfigError(f"bits must be >= 1, got {self.bits}")
        p = self.norm_p
        if p != 0 and not p > 0:
            raise ConfigError(f"norm_p must be 0, positive, or inf: {p}")
        if self.rounding not in ROUNDINGS:
            raise ConfigError(f"unknown rounding mode {self.rounding!r}")

    @property
    def qmax(self) -> int:
        return (1 << (self.bits - 1)) - 1

    def cuda_supported(self) -> bool:
        """The quantizer variants the fused CUDA encoder implements."""
        return self.bits == 1 or (self.norm_p == 1.0 and self.rounding == "nearest"
                                  and not self.log_transform and not self.no_zero)


@dataclass(frozen=True)
class SignPolicy:
    """Zero handling when reducing to signs: ``exact-ternary`` keeps 0,
    ``alternating`` substitutes +1 on odd iterations and -1 on even ones."""

    mode: str = "alternating"
    iteration: int = 0

    def __post_init__(self):
        if self.mode not in ZERO_MODES:
            raise ConfigError(f"unknown sign policy mode {self.mode!r}")
        if self.iteration < 0:
            raise ConfigError("iteration must be non-negative")

    def zero_fill(self) -> int:
        return -1 if self.iteration % 2 == 0 else 1

    def kernel_fill(self) -> int:
        """The ``fill`` argument of the C ABI: +-1, or 0 for exact-ternary."""
        return 0 if self.mode == "exact-ternary" else self.zero_fill()
