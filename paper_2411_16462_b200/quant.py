"""Quantizer / sign-policy configuration of the drop-in API.

``QuantSpec`` and ``SignPolicy`` take the reference's constructor arguments
and validation (lioncomm/quant.py:27-78).  On the CUDA path the quantizer
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
        return int(torch.randint(0, 1 << 62, (1,), generator=rng, device=rng.device).item())
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


# ---------------------------------------------------------------------------
# Standalone operators over CUDA tensors (quant.py:81-300).  Each runs our
# sm_100a kernels (csrc/quant.cu, csrc/l1norm.cu, csrc/kernels.cu); there is
# no CPU path -- CPU arrays raise ConfigError.
# ---------------------------------------------------------------------------

import ctypes as _C  # noqa: E402
import struct as _struct  # noqa: E402
import threading as _threading  # noqa: E402

from . import _lib  # noqa: E402
from .errors import PackFormatError, PackRangeError  # noqa: E402

_IDENTITY = None        # lc_hyper with c = 0*x + 1*x = x (exact, -0.0 kept)
_plans: dict = {}       # (device, n) -> single-segment norm plan
_plans_lock = _threading.Lock()


def _identity_hyper():
    global _IDENTITY
    if _IDENTITY is None:
        _IDENTITY = _lib.Hyper(0.0, 1.0, 0.0, 1.0, 0.0, 0.0)
    return _IDENTITY


def _stream(dev):
    import torch
    return torch.cuda.current_stream(dev).cuda_stream


def _as_cuda_f32(x, what: str):
    """Flat, 16-byte aligned fp32 CUDA view of ``x``.  float64 input must be
    fp32-representable (the optimizer state is fp32; the operators compute
    in float64 from fp32 values)."""
    import torch
    if not isinstance(x, torch.Tensor) or x.device.type != "cuda":
        raise ConfigError(f"{what}: expected a CUDA tensor (no CPU path)")
    x = x.reshape(-1)
    if x.dtype == torch.float32:
        x = x.contiguous()
        return x if x.data_ptr() % 16 == 0 else x.clone()
    x64 = x.to(torch.float64).contiguous()
    out = torch.empty(x64.numel(), dtype=torch.float32, device=x.device)
    flags = torch.zeros(1, dtype=torch.int32, device=x.device)
    _lib.call("lc_f64_to_f32_exact", x64.data_ptr(), x64.numel(), out.data_ptr(),
              flags.data_ptr(), _stream(x.device))
    if int(flags.item()):
        raise ConfigError(f"{what}: values are not exactly representable in float32")
    return out


def _plan(dev, n: int):
    if n == 0:
        raise ConfigError("lp_mean_norm of an empty vector")
    key = (dev.index, n)
    with _plans_lock:
        p = _plans.get(key)
        if p is None:
            if len(_plans) >= 64:      # bounded cache of device plans
                _plans.clear()
            import torch
            from .optimizer import _L1Plan

            class _One:
                seg_start = [0, n]
                names = ["x"]
            with torch.cuda.device(dev):
                p = _plans[key] = (_L1Plan(_One), torch.tensor([0, n], dtype=torch.int64,
                                                               device=dev))
        return p


def scale_tables(plan_handle: int, g, m, mask, hyp, spec: QuantSpec, norms, scales,
                 logs, stream) -> None:
    """Per-segment quantizer scalars (quant.py:143-161) into device arrays:
    ``logs`` (2*nseg doubles; first half M1(c)) when log_transform, then the
    norm M_p of y in ``norms`` and the scale in ``scales``."""
    args = (plan_handle, g.data_ptr(), m.data_ptr(), _lib.ptr(mask), _C.byref(hyp))
    nseg = norms.numel()
    lg = None
    if spec.log_transform:
        lg = logs[:nseg]
        _lib.call("lc_l1_scales", *args, spec.qmax, lg.data_ptr(), logs[nseg:].data_ptr(),
                  stream)
    if spec.norm_p == 1.0 and lg is None:
        _lib.call("lc_l1_scales", *args, spec.qmax, norms.data_ptr(), scales.data_ptr(),
                  stream)
    else:
        ns = _lib.NormSpec(float(spec.norm_p), spec.qmax, 0, _lib.ptr(lg))
        _lib.call("lc_norm_scales", *args, _C.byref(ns), norms.data_ptr(), scales.data_ptr(),
                  stream)


def lp_mean_norm(x, p: float) -> float:
    """``lp_mean_norm`` (quant.py:81-104) of a CUDA tensor: p = inf max|x|,
    p = 0 geometric mean of the nonzero |x|, finite p numpy's
    max * mean((|x|/max)**p)**(1/p) in numpy's pairwise summation order."""
    import torch
    if not (p == 0 or p > 0):
        raise ConfigError(f"invalid norm order {p}")
    x32 = _as_cuda_f32(x, "lp_mean_norm")
    plan, _ = _plan(x32.device, x32.numel())
    norms = torch.zeros(2, dtype=torch.float64, device=x32.device)
    ns = _lib.NormSpec(float(p), 0, 0, None)
    _lib.call("lc_norm_scales", plan.handle, x32.data_ptr(), x32.data_ptr(), None,
              _C.byref(_identity_hyper()), _C.byref(ns), norms.data_ptr(),
              norms[1:].data_ptr(), _stream(x32.device))
    return float(norms[0].item())


def quantize(x, spec: QuantSpec, rng=None):
    """``quantize`` (quant.py:127-173) of a CUDA tensor -> int64 tensor of
    x's shape in [-qmax, qmax].  Stochastic rounding draws its stream seed
    from ``rng`` (see QuantSpec.draw_seed)."""
    import torch
    shape = tuple(x.shape) if isinstance(x, torch.Tensor) else None
    x32 = _as_cuda_f32(x, "quantize")
    n = x32.numel()
    if n == 0:
        raise ConfigError("quantize of an empty vector")
    dev = x32.device
    plan, start = _plan(dev, n)
    tabs = torch.zeros(4, dtype=torch.float64, device=dev)   # norm, scale, M1, -
    s = _stream(dev)
    scale_tables(plan.handle, x32, x32, None, _identity_hyper(), spec, tabs[0:1], tabs[1:2],
                 tabs[2:4], s)
    seed = 0
    if spec.rounding == "stochastic":
        if rng is None and float(tabs[1].item()) != 0.0:
            raise ConfigError("stochastic rounding needs an rng")
        seed = draw_seed(rng) if rng is not None else 0
    segs = _lib.Segments(start.data_ptr(), tabs[1:2].data_ptr(), 1, spec.qmax,
                         tabs[2:3].data_ptr() if spec.log_transform else None,
                         spec.kernel_flags(), 0, seed)
    q = torch.empty(n, dtype=torch.int64, device=dev)
    _lib.call("lc_quantize_values", x32.data_ptr(), n, _C.byref(segs), q.data_ptr(), s)
    return q.view(shape) if shape is not None else q


def dequantize(q, spec: QuantSpec, norm: float, log_scale: float | None = None):
    """``dequantize`` (quant.py:176-195): q * (norm/qmax) for p = inf, else
    q * (2 norm/qmax); the log map undone with ``log_scale``.  float64."""
    import torch
    if not isinstance(q, torch.Tensor) or q.device.type != "cuda":
        raise ConfigError("dequantize: expected a CUDA tensor (no CPU path)")
    shape = tuple(q.shape)
    qmax = spec.qmax
    if qmax == 0 or norm == 0:
        return torch.zeros(shape, dtype=torch.float64, device=q.device)
    mult = norm / qmax if spec.norm_p == INF else 2.0 * norm / qmax
    if spec.log_transform and log_scale is None:
        raise ConfigError("dequantize of a log-transformed vector needs log_scale")
    qi = q.reshape(-1).to(torch.int64).contiguous()
    out = torch.empty(qi.numel(), dtype=torch.float64, device=q.device)
    _lib.call("lc_dequantize", qi.data_ptr(), qi.numel(), float(mult),
              float(log_scale or 0.0), int(spec.log_transform), out.data_ptr(),
              _stream(q.device))
    return out.view(shape)


def apply_sign(x, policy: SignPolicy):
    """``apply_sign`` (quant.py:198-204): elementwise sign, zeros (and -0.0)
    resolved by the policy.  int8 tensor of x's shape (values as the
    reference's int64)."""
    import torch
    if not isinstance(x, torch.Tensor) or x.device.type != "cuda":
        raise ConfigError("apply_sign: expected a CUDA tensor (no CPU path)")
    shape = tuple(x.shape)
    f64 = x.dtype == torch.float64
    xf = x.reshape(-1).contiguous() if x.dtype in (torch.float32, torch.float64) else \
        x.reshape(-1).to(torch.float64).contiguous()
    out = torch.empty(xf.numel(), dtype=torch.int8, device=x.device)
    _lib.call("lc_apply_sign_values", xf.data_ptr(), int(f64 or xf.dtype == torch.float64),
              xf.numel(), policy.kernel_fill(), out.data_ptr(), _stream(x.device))
    return out.view(shape)


def _payload_len(count: int, width: int) -> int:
    return (count * width + 7) // 8


def _check_width(width: int):
    if width not in PACKABLE_WIDTHS:
        raise ConfigError(f"width must be one of {PACKABLE_WIDTHS}, got {width}")


def _is_sign_map(width: int, offset: int) -> bool:
    return width == 1 and offset == 1


class PackedBits:
    """``PackedBits`` (quant.py:208-239): ``count`` fields of ``width`` bits,
    element 0 in the low bits, value + ``offset`` stored (width 1 with
    offset 1 is the sign map {-1,+1} -> {0,1}).  ``payload`` is a CUDA uint8
    tensor; ``to_bytes``/``from_bytes`` speak the reference's wire format
    (header ``<IBi`` count, width, offset)."""

    HEADER = _struct.Struct("<IBi")

    def __init__(self, width: int, count: int, offset: int, payload):
        self.width, self.count, self.offset, self.payload = width, count, offset, payload

    def __repr__(self):
        return f"PackedBits(width={self.width}, count={self.count}, offset={self.offset})"

    def __eq__(self, other):
        import torch
        return (isinstance(other, PackedBits) and
                (self.width, self.count, self.offset) == (other.width, other.count,
                                                          other.offset) and
                torch.equal(self.payload.cpu(), other.payload.cpu()))

    def to_bytes(self) -> bytes:
        return self.HEADER.pack(self.count, self.width, self.offset) + \
            self.payload.cpu().numpy().tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes, device="cuda") -> "PackedBits":
        import torch
        if len(raw) < cls.HEADER.size:
            raise PackFormatError(f"truncated header: {len(raw)} bytes")
        count, width, offset = cls.HEADER.unpack_from(raw)
        payload = raw[cls.HEADER.size:]
        expected = _payload_len(count, width)
        if len(payload) != expected:
            raise PackFormatError(
                f"payload is {len(payload)} bytes, expected {expected} "
                f"for count={count} width={width}")
        t = torch.frombuffer(bytearray(payload), dtype=torch.uint8) if payload else \
            torch.zeros(0, dtype=torch.uint8)
        return cls(width=width, count=count, offset=offset, payload=t.to(device))


def pack(values, width: int, offset: int = 0) -> PackedBits:
    """``pack`` (quant.py:255-281) of a CUDA integer tensor (raveled).
    PackRangeError names the first value that does not fit."""
    import torch
    _check_width(width)
    if not isinstance(values, torch.Tensor) or values.device.type != "cuda":
        raise ConfigError("pack: expected a CUDA tensor (no CPU path)")
    v = values.reshape(-1).to(torch.int64).contiguous()
    count = v.numel()
    sign_map = _is_sign_map(width, offset)
    words = torch.zeros(max(1, -(-count * width // 32)), dtype=torch.int32, device=v.device)
    flags = torch.zeros(1, dtype=torch.int32, device=v.device)
    if count:
        _lib.call("lc_pack_i64_fields", v.data_ptr(), count, width, 0 if sign_map else offset,
                  int(sign_map), words.data_ptr(), flags.data_ptr(), _stream(v.device))
        if int(flags.item()):
            if sign_map:
                bad = v.abs() != 1
            else:
                st = v + offset
                bad = (st < 0) | (st > (1 << width) - 1)
            i = int(torch.nonzero(bad)[0, 0].item())
            raise PackRangeError(i, int(v[i].item()), width)
    payload = words.view(torch.uint8)[:_payload_len(count, width)].clone()
    return PackedBits(width=width, count=count, offset=offset, payload=payload)


def unpack(packed: PackedBits):
    """``unpack`` (quant.py:284-300): exact inverse of ``pack`` -> int64."""
    import torch
    _check_width(packed.width)
    expected = _payload_len(packed.count, packed.width)
    if packed.payload.numel() != expected:
        raise PackFormatError(f"payload is {packed.payload.numel()} bytes, expected {expected}")
    dev = packed.payload.device
    if dev.type != "cuda":
        raise ConfigError("unpack: payload must be a CUDA tensor (no CPU path)")
    words = torch.zeros(max(1, -(-expected // 4)), dtype=torch.int32, device=dev)
    words.view(torch.uint8)[:expected].copy_(packed.payload)
    out = torch.empty(packed.count, dtype=torch.int64, device=dev)
    sign_map = _is_sign_map(packed.width, packed.offset)
    if packed.count:
        _lib.call("lc_fields_decode", words.data_ptr(), packed.count, packed.width, 1,
                  0 if sign_map else packed.offset, int(sign_map), out.data_ptr(),
                  _stream(dev))
    return out
