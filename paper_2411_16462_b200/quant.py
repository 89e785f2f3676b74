"""Quantizer / sign-policy configuration of the drop-in API.

``QuantSpec`` and ``SignPolicy`` take the reference's constructor arguments
and validation (lioncomm/quant.py:102-153).  On the CUDA path the quantizer
itself runs inside the fused interpolate kernel (csrc/kernels.cu, K1) and the
per-layer mean p-norm in csrc/l1norm.cu.  Every variant of the reference is
implemented: norm_p 1 (the paper's Lion Cub p-bit scheme), any finite p,
0 (geometric mean) and inf (max norm); nearest or stochastic rounding;
log_transform; no_zero.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError

LC_Q_STOCHASTIC = 1 << 0   # include/lioncub.h
LC_Q_NO_ZERO = 1 << 1


def draw_seed(rng) -> int:
    """A 64-bit seed for the counter-based stochastic-rounding stream."""
    if rng is None:
        raise ConfigError("stochastic rounding needs an rng")
    if isinstance(rng, int):
        return rng & 0xFFFFFFFFFFFFFFFF
    if hasattr(rng, "integers"):         # numpy Generator
        return int(rng.integers(0, 1 << 63, dtype="int64"))
    import torch
    if isinstance(rng, torch.Generator):
        return int(torch.randint(0, 1 << 62, (1,), generator=rng).item())
    raise ConfigError(f"unsupported rng {type(rng).__name__}")


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

    def kernel_flags(self) -> int:
        """``lc_segments.qflags`` of this spec (include/lioncub.h LC_Q_*)."""
        return ((LC_Q_STOCHASTIC if self.rounding == "stochastic" else 0)
                | (LC_Q_NO_ZERO if self.no_zero else 0))

    def draw_seed(self, rng) -> int:
        """This call's stochastic-rounding stream seed, drawn from ``rng``
        (0 for nearest rounding).  ``rng``: a ``numpy.random.Generator`` (as
        the reference takes, quant.py:127-128), a CPU ``torch.Generator``, or
        an int (a fixed stream).  Missing rng -> ConfigError like the
        reference (quant.py:163-165)."""
        if self.rounding != "stochastic":
            return 0
        return draw_seed(rng)


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
