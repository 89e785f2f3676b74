"""CPU oracle for the Lion Cub distributed optimizer step.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2411_16462_b200`` imports
this module; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it,
and only as the checker / the timed CPU baseline, never as a product path.

It is a single-process numpy restatement of the reference package
``lioncomm`` (``/root/reference/pkg/src/lioncomm``): every P-rank
collective is evaluated on the gathered per-rank inputs, exactly like the
reference tests' ``sum_oracle`` (``pkg/tests/test_collectives.py:14-15``).
Each function cites the reference lines it restates.  Arithmetic follows the
reference operation by operation (float64 numpy, the same operand order), so
for fp32-representable inputs the outputs are bit-identical to the
reference's.

Parity of this restatement is PINNED against vectors produced by the real
reference (``tests/golden/make_golden.py`` imports ``lioncomm`` from
``/root/reference`` and writes ``tests/golden/*.npz``); see
``tests/test_oracle.py``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np


class OracleConfigError(ValueError):
    """Raised where the reference raises ``ConfigError`` (errors.py:8)."""


class OracleCapacityError(OracleConfigError):
    """Raised where the reference raises ``CapacityError`` (errors.py:12-16)."""


# ---------------------------------------------------------------------------
# quant.py
# ---------------------------------------------------------------------------

def zero_fill(iteration: int) -> int:
    """``SignPolicy.zero_fill`` (quant.py:76-78): +1 on odd t, -1 on even."""
    return 1 if iteration % 2 == 1 else -1


def apply_sign(x, mode: str, iteration: int) -> np.ndarray:
    """``apply_sign`` (quant.py:198-204).  -0.0 == 0 so it takes the fill."""
    x = np.asarray(x)
    s = np.sign(x).astype(np.int64)
    if mode == "alternating":
        s = np.where(x == 0, zero_fill(iteration), s)
    return s


def pairwise_sum(a: np.ndarray) -> float:
    """numpy's float64 pairwise summation order (the order ``np.mean`` uses
    inside ``lp_mean_norm``, quant.py:104).  Blocks of <=128 elements use 8
    strided accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7));
    larger blocks split at n/2 rounded down to a multiple of 8.  Kept here
    as executable documentation of the order the CUDA norm kernel mirrors;
    ``tests/test_oracle.py`` checks it against ``np.sum``."""
    a = np.asarray(a, dtype=np.float64)

    def rec(lo: int, n: int) -> float:
        if n < 8:
            res = 0.0
            for i in range(n):
                res += float(a[lo + i])
            return res
        if n <= 128:
            r = [float(a[lo + k]) for k in range(8)]
            i = 8
            while i < n - (n % 8):
                for k in range(8):
                    r[k] += float(a[lo + i + k])
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += float(a[lo + i])
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return rec(0, a.size)


def lp_mean_norm_l1(x) -> float:
    """``lp_mean_norm(x, 1)`` (quant.py:81-104, finite-p branch):
    M1 = max|x| * mean(|x|/max|x|)."""
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        raise OracleConfigError("lp_mean_norm of an empty vector")
    a = np.abs(x)
    m = a.max()
    if m == 0:
        return 0.0
    return float(m * np.mean((a / m) ** 1.0) ** (1.0 / 1.0))


def quantize_l1(x, bits: int) -> np.ndarray:
    """``quantize`` with ``QuantSpec(bits, norm_p=1, rounding="nearest")``
    (quant.py:127-173): q = clip(round_half_even(qmax/(2 M1) * x), +-qmax)."""
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        raise OracleConfigError("quantize of an empty vector")
    qmax = 2 ** (bits - 1) - 1
    m = lp_mean_norm_l1(x)
    if m == 0 or qmax == 0:
        return np.zeros(x.shape, dtype=np.int64)
    scaled = (qmax / (2.0 * m)) * x
    q = np.round(scaled).astype(np.int64)
    return np.clip(q, -qmax, qmax)


INF = float("inf")


def lp_mean_norm(x, p: float) -> float:
    """``lp_mean_norm`` (quant.py:81-104), every order: p = inf -> max|x|;
    p = 0 -> exp(mean(log|x_j|)) over the nonzero entries (0 if none);
    finite p -> max * mean((|x|/max)**p)**(1/p)."""
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        raise OracleConfigError("lp_mean_norm of an empty vector")
    a = np.abs(x)
    if p == INF:
        return float(a.max())
    if p == 0:
        nz = a[a > 0]
        if nz.size == 0:
            return 0.0
        return float(np.exp(np.mean(np.log(nz))))
    if p <= 0:
        raise OracleConfigError(f"invalid norm order {p}")
    m = a.max()
    if m == 0:
        return 0.0
    return float(m * np.mean((a / m) ** p) ** (1.0 / p))


def stream_uniforms(seed: int, index) -> np.ndarray:
    """The CUDA path's stochastic-rounding stream (csrc/common.cuh
    ``lc::uniform01``): element e draws u = x * 2**-32 with x =
    lowbias32(lo32(e)*0x9E3779B9 + lo32(seed) ^ hi32(e)*0x85EBCA6B ^
    hi32(seed)) in wrapping uint32 arithmetic, a counter-based stream (no
    sequential state, so any element range of any rank can be drawn
    independently).  The reference draws from numpy's PCG64
    (quant.py:107-116); parity of stochastic rounding with the reference is
    statistical, with this stream exact."""
    e = np.asarray(index, dtype=np.uint64)
    s = int(seed) & 0xFFFFFFFFFFFFFFFF
    u32 = np.uint32
    with np.errstate(over="ignore"):
        x = (e & np.uint64(0xFFFFFFFF)).astype(u32) * u32(0x9E3779B9) + u32(s & 0xFFFFFFFF)
        x ^= (e >> np.uint64(32)).astype(u32) * u32(0x85EBCA6B) ^ u32(s >> 32)
        x ^= x >> u32(16)
        x *= u32(0x7FEB352D)
        x ^= x >> u32(15)
        x *= u32(0x846CA68B)
        x ^= x >> u32(16)
    return x.astype(np.float64) * (2.0 ** -32)


def sround(v, u) -> np.ndarray:
    """``sround`` (quant.py:107-116) with the uniforms supplied: floor(v) +
    (u < v - floor(v))."""
    v = np.asarray(v, dtype=np.float64)
    lo = np.floor(v)
    frac = v - lo
    return (lo + (np.asarray(u) < frac)).astype(np.int64)


def quantize(x, spec: "Spec", uniforms=None) -> np.ndarray:
    """``quantize`` (quant.py:127-173), every variant: optional log map
    y = sign(x) log1p(|x|/M1(x)) (:146-150, :119-120), scale qmax/M_inf
    (p = inf, :153-161) or qmax/(2 M_p) (:162-170), nearest (half-even) or
    stochastic rounding (``uniforms`` = the per-element draws), clip,
    then no_zero (:171-173)."""
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        raise OracleConfigError("quantize of an empty vector")
    qmax = spec.qmax
    y = x
    if spec.log_transform:
        s = lp_mean_norm(x, 1.0)
        if s > 0:
            y = np.sign(x) * np.log1p(np.abs(x) / s)
    m = lp_mean_norm(y, spec.norm_p)
    if m == 0 or qmax == 0:
        q = np.zeros(x.shape, dtype=np.int64)
    else:
        scaled = (qmax / m) * y if spec.norm_p == INF else (qmax / (2.0 * m)) * y
        if spec.rounding == "stochastic":
            if uniforms is None:
                raise OracleConfigError("stochastic rounding needs an rng")
            q = sround(scaled, np.asarray(uniforms).reshape(x.shape))
        else:
            q = np.round(scaled).astype(np.int64)
        q = np.clip(q, -qmax, qmax)
    if spec.no_zero:
        fix = (q == 0) & (x != 0)
        q = np.where(fix, np.sign(x).astype(np.int64), q)
    return q


def quant_scale(x, spec: "Spec") -> tuple:
    """(scale, log_scale) the quantizer multiplies by: the per-layer scalars
    the CUDA norm kernels produce (quant.py:143-161)."""
    x = np.asarray(x, dtype=np.float64)
    y, s = x, None
    if spec.log_transform:
        s = lp_mean_norm(x, 1.0)
        if s > 0:
            y = np.sign(x) * np.log1p(np.abs(x) / s)
    m = lp_mean_norm(y, spec.norm_p)
    if m == 0 or spec.qmax == 0:
        return 0.0, s, m
    return (spec.qmax / m if spec.norm_p == INF else spec.qmax / (2.0 * m)), s, m


def dequantize(q, spec: "Spec", norm: float, log_scale: float | None = None) -> np.ndarray:
    """``dequantize`` (quant.py:176-195)."""
    q = np.asarray(q, dtype=np.float64)
    qmax = spec.qmax
    if qmax == 0 or norm == 0:
        return np.zeros_like(q)
    y = q * (norm / qmax) if spec.norm_p == INF else q * (2.0 * norm / qmax)
    if spec.log_transform:
        if log_scale is None:
            raise OracleConfigError("dequantize of a log-transformed vector needs log_scale")
        return np.sign(y) * log_scale * np.expm1(np.abs(y))
    return y


def pack_words(stored, width: int) -> np.ndarray:
    """``pack(values, width)`` payload (quant.py:255-281) viewed as
    little-endian uint32 words: element i sits at bits
    ``width*(i % (32//width))`` of word ``i // (32//width)``.  Widths 16/32
    extend the same layout (the B200 wire uses them for wide p-bit sums)."""
    stored = np.asarray(stored, dtype=np.uint64).ravel()
    per = 32 // width
    nw = -(-stored.size // per)
    pad = np.zeros(nw * per, dtype=np.uint64)
    pad[: stored.size] = stored
    lanes = pad.reshape(nw, per)
    shifts = (np.arange(per, dtype=np.uint64) * np.uint64(width))
    return (lanes << shifts).sum(axis=1).astype(np.uint32)


def pack_signs(s) -> np.ndarray:
    """``pack(s, 1, 1)`` (quant.py:261-266): {-1,+1} -> {0,1}, 1 bit each."""
    s = np.asarray(s, dtype=np.int64)
    return pack_words((s + 1) >> 1, 1)


def unpack_words(words, width: int, count: int) -> np.ndarray:
    """Inverse of ``pack_words`` (``unpack``, quant.py:284-300)."""
    words = np.asarray(words, dtype=np.uint32).astype(np.uint64)
    per = 32 // width
    shifts = np.arange(per, dtype=np.uint64) * np.uint64(width)
    mask = np.uint64((1 << width) - 1)
    f = ((words[:, None] >> shifts) & mask).ravel()
    return f[:count].astype(np.int64)


# ---------------------------------------------------------------------------
# collectives.py (single-process restatements of the P-rank results)
# ---------------------------------------------------------------------------

@dataclass
class Vote:
    """``VoteResult`` (collectives.py:67-73)."""
    values: np.ndarray
    range: tuple
    ties: int


def choose_lane_bits(workers: int, q_max: int, binary_signs: bool = False) -> int:
    """collectives.py:168-176."""
    max_stored = 1 if binary_signs else 2 * q_max
    need = workers * max_stored
    for bits in (8, 16, 32):
        if need <= (1 << bits) - 1:
            return bits
    raise OracleCapacityError(
        f"sum of {workers} values up to {max_stored} exceeds a 32-bit lane")


def direct_sum(qs: Sequence[np.ndarray], q_max: int, binary_signs: bool = False,
               lane_bits: int | None = None) -> Vote:
    """``direct_allreduce`` result (collectives.py:179-249): the exact
    elementwise sum of offset values, de-offset, plus the tie count.  The
    ring RS+AG is order-free integer addition, so the gathered sum is it."""
    p = len(qs)
    max_stored = 1 if binary_signs else 2 * q_max
    if lane_bits is None:
        lane_bits = choose_lane_bits(p, q_max, binary_signs)
    if lane_bits not in (8, 16, 32):
        raise OracleConfigError("lane_bits must be one of [8, 16, 32]")
    if p * max_stored > (1 << lane_bits) - 1:
        raise OracleCapacityError("capacity")
    stored = []
    for q in qs:
        q = np.ascontiguousarray(np.asarray(q).ravel(), dtype=np.int64)
        if binary_signs:
            if np.any(np.abs(q) != 1):
                raise OracleConfigError("binary_signs requires values in {-1, +1}")
            stored.append((q + 1) >> 1)
        else:
            if np.any(np.abs(q) > q_max):
                raise OracleConfigError(f"values exceed declared q_max={q_max}")
            stored.append(q + q_max)
    summed = np.sum(np.stack(stored), axis=0).astype(np.int64)
    if binary_signs:
        signed = 2 * summed - p
        bound = p
    else:
        signed = summed - p * q_max
        bound = p * q_max
    ties = int(np.count_nonzero(signed == 0))
    return Vote(values=signed, range=(-float(bound), float(bound)), ties=ties)


def vote_1bit(cs: Sequence[np.ndarray], mode: str, iteration: int) -> Vote:
    """``compressed_allreduce_1bit`` result (collectives.py:252-310).
    Per rank s = apply_sign(c) (zeros rejected, :263-267); owners sum the P
    sign chunks and take apply_sign again (:288-293); the +1 padding
    (:269-271) sums to P != 0 so it never ties and is stripped (:309), which
    makes the result independent of the chunking."""
    signs = []
    for c in cs:
        s = apply_sign(np.asarray(c, dtype=np.float64).ravel(), mode, iteration)
        if np.any(s == 0):
            raise OracleConfigError(
                "1-bit path cannot carry exact zeros; use the alternating policy")
        signs.append(s)
    tally = np.sum(np.stack(signs), axis=0)
    ties = int(np.count_nonzero(tally == 0))
    voted = apply_sign(tally, mode, iteration)
    if np.any(voted == 0):
        raise OracleConfigError(
            "1-bit path cannot carry exact zeros; use the alternating policy")
    return Vote(values=voted, range=(-1.0, 1.0), ties=ties)


def ps_sum(cs: Sequence[np.ndarray], efficient: bool = False) -> Vote:
    """``ps_gather_broadcast`` for float vectors (collectives.py:132-165).
    Flat: rank 0 adds ranks 1..P-1 in order (:153-158).  Efficient: the
    binomial-tree reduce order of ``_tree_reduce_to_root`` (:96-109)."""
    vecs = [np.asarray(c, dtype=np.float64).ravel() for c in cs]
    p = len(vecs)
    if not efficient:
        total = vecs[0].copy()
        for src in range(1, p):
            total = total + vecs[src]
    else:
        acc = [v.copy() for v in vecs]
        mask = 1
        while mask < p:
            for r in range(0, p, 2 * mask):
                partner = r + mask
                if partner < p:
                    acc[r] = acc[r] + acc[partner]
            mask <<= 1
        total = acc[0]
    ties = int(np.count_nonzero(total == 0))
    bound = float(np.max(np.abs(total))) if total.size else 0.0
    return Vote(values=total, range=(-bound, bound), ties=ties)


def mean_f32(xs: Sequence[np.ndarray]) -> np.ndarray:
    """``allreduce_mean_f32`` (collectives.py:319-344): float32 payloads,
    float64 accumulation in rank order at rank 0, one rounding to f32."""
    vecs = [np.asarray(x, dtype=np.float32).ravel() for x in xs]
    acc = vecs[0].astype(np.float64)
    for src in range(1, len(vecs)):
        acc += vecs[src].astype(np.float64)
    return (acc / len(vecs)).astype(np.float32)


# ---------------------------------------------------------------------------
# optimizer.py
# ---------------------------------------------------------------------------

@dataclass
class Hyper:
    """``LionHyper`` (optimizer.py:43-60) with a constant learning rate."""
    beta1: float = 0.9
    beta2: float = 0.99
    lr: float = 1e-4
    weight_decay: float = 0.0


@dataclass
class Spec:
    """``QuantSpec`` (quant.py:28-55): bits, norm order, rounding, log map,
    no_zero."""
    bits: int = 8
    norm_p: float = 1.0
    rounding: str = "nearest"
    log_transform: bool = False
    no_zero: bool = False

    @property
    def qmax(self) -> int:
        return 2 ** (self.bits - 1) - 1


def _vote_layer(cs: Sequence[np.ndarray], spec: Spec | None, algo: str,
                mode: str, t: int, uniforms=None):
    """``_vote`` (optimizer.py:137-169): returns (sign, Vote).  ``uniforms``:
    per-rank stochastic-rounding draws of this layer."""
    if algo == "compressed1bit":
        v = vote_1bit(cs, mode, t)
        return v.values, v
    if spec is None:
        if algo == "direct":
            raise OracleConfigError("direct allreduce needs an integer QuantSpec")
        qs = cs
    elif spec.bits == 1:
        qs = [apply_sign(c, mode, t) for c in cs]
    else:
        qs = [quantize(c, spec, None if uniforms is None else uniforms[r])
              for r, c in enumerate(cs)]
    if algo in ("ps", "ps_efficient"):
        if spec is None:
            v = ps_sum(qs, efficient=algo == "ps_efficient")
        else:
            total = np.sum(np.stack([np.asarray(q, np.int64) for q in qs]), axis=0)
            v = Vote(values=total, range=(0, 0), ties=int(np.count_nonzero(total == 0)))
    elif algo == "direct":
        binary = spec.bits == 1
        v = direct_sum(qs, q_max=spec.qmax if not binary else 1, binary_signs=binary)
    else:
        raise OracleConfigError(f"unknown vote algorithm {algo!r}")
    return apply_sign(v.values, mode, t), v


def distributed_step(thetas: Sequence[Mapping[str, np.ndarray]],
                     moms: Sequence[Mapping[str, np.ndarray]],
                     grads: Sequence[Mapping[str, np.ndarray]],
                     h: Hyper, spec: Spec | None, algo: str, iteration: int,
                     zero_mode: str = "alternating",
                     masks: Mapping[str, np.ndarray] | Sequence | None = None,
                     seeds: Sequence[int] | None = None):
    """``distributed_lion_step`` for all P ranks at once
    (optimizer.py:172-210).  Per layer in sorted order: c = b1*m + (1-b1)*g
    (:199), optional mask (:200-201), vote (:202), theta' (:204), m' (:205).

    ``masks`` is one mapping shared by all ranks or a per-rank sequence.
    ``seeds``: per-rank stochastic-rounding seeds of this step (the CUDA
    path's stream is indexed by the element's offset in the sorted-name flat
    buffer).
    Returns (thetas', moms', vote_sign{layer}, ties{layer}, c{rank}{layer},
    vote{layer})."""
    p = len(thetas)
    t = iteration + 1
    eta = float(h.lr)
    new_t = [dict() for _ in range(p)]
    new_m = [dict() for _ in range(p)]
    signs, ties, votes = {}, {}, {}
    cs_all = [dict() for _ in range(p)]
    offset = 0
    for name in sorted(thetas[0]):
        cs = []
        for r in range(p):
            m = np.asarray(moms[r][name], dtype=np.float64)
            g = np.asarray(grads[r][name], dtype=np.float64)
            c = h.beta1 * m + (1.0 - h.beta1) * g
            mk = None
            if masks is not None:
                mk = masks[r] if isinstance(masks, (list, tuple)) else masks
            if mk is not None and name in mk:
                c = np.where(mk[name], c, 0.0)
            cs.append(c)
            cs_all[r][name] = c
        flat = [c.ravel() for c in cs]
        uni = None
        if seeds is not None:
            idx = offset + np.arange(flat[0].size)
            uni = [stream_uniforms(seeds[r], idx) for r in range(p)]
        offset += flat[0].size
        sign, vote = _vote_layer(flat, spec, algo, zero_mode, t, uniforms=uni)
        sign = np.asarray(sign).reshape(cs[0].shape)
        for r in range(p):
            theta = np.asarray(thetas[r][name], dtype=np.float64)
            m = np.asarray(moms[r][name], dtype=np.float64)
            g = np.asarray(grads[r][name], dtype=np.float64)
            new_t[r][name] = theta - eta * (sign + h.weight_decay * theta)
            new_m[r][name] = h.beta2 * m + (1.0 - h.beta2) * g
        signs[name] = sign
        ties[name] = vote.ties
        votes[name] = vote
    return new_t, new_m, signs, ties, cs_all, votes


def signsgd_step(thetas: Sequence[Mapping[str, np.ndarray]],
                 grads: Sequence[Mapping[str, np.ndarray]], lr: float, algo: str,
                 iteration: int, zero_mode: str = "alternating"):
    """``signsgd_majority_step`` for all P ranks (optimizer.py:213-241):
    theta' = theta - lr * majority(sign(g_r)), momentum untouched."""
    t = iteration + 1
    out = {}
    for name in sorted(thetas[0]):
        gs = [np.asarray(g[name], dtype=np.float64).ravel() for g in grads]
        if algo == "compressed1bit":
            maj = vote_1bit(gs, zero_mode, t).values
        else:
            ss = [apply_sign(g, zero_mode, t) for g in gs]
            if algo == "direct":
                v = direct_sum(ss, q_max=1, binary_signs=True)
            else:
                v = ps_sum([s.astype(np.float64) for s in ss],
                           efficient=algo == "ps_efficient")
            maj = apply_sign(v.values, zero_mode, t)
        th = np.asarray(thetas[0][name], dtype=np.float64)
        out[name] = th - lr * np.asarray(maj).reshape(th.shape)
    return out


def divergence(moms: Sequence[Mapping[str, np.ndarray]]) -> dict:
    """``divergence_from_momenta`` (optimizer.py:270-276): per layer, max over
    elements of the population std across ranks."""
    return {name: float(np.stack([np.asarray(m[name], np.float64) for m in moms])
                        .std(axis=0, ddof=0).max())
            for name in sorted(moms[0])}


def lion_step(theta: Mapping[str, np.ndarray], mom: Mapping[str, np.ndarray],
              grad: Mapping[str, np.ndarray], h: Hyper):
    """``lion_step`` (optimizer.py:114-131): single worker, np.sign (zeros
    contribute no update)."""
    nt, nm = {}, {}
    for name in theta:
        g = np.asarray(grad[name], dtype=np.float64)
        m = np.asarray(mom[name], dtype=np.float64)
        th = np.asarray(theta[name], dtype=np.float64)
        c = h.beta1 * m + (1.0 - h.beta1) * g
        nt[name] = th - float(h.lr) * (np.sign(c) + h.weight_decay * th)
        nm[name] = h.beta2 * m + (1.0 - h.beta2) * g
    return nt, nm


def sync_fires(period: int, t: int) -> bool:
    """``SyncPolicy.fires`` (optimizer.py:95-96)."""
    return period > 0 and t % period == 0


def sync_selects(layers, name: str) -> bool:
    """``SyncPolicy.selects`` (optimizer.py:98-103)."""
    if layers == "all":
        return True
    if layers == "none":
        return False
    return name in layers


def sync_momentum(moms: Sequence[Mapping[str, np.ndarray]], period: int, layers,
                  iteration: int):
    """``maybe_sync_momentum`` (optimizer.py:244-258): at firing iterations
    every selected layer's momentum becomes the f32 mean (then f64)."""
    out = [dict(m) for m in moms]
    if not sync_fires(period, iteration):
        return out
    for name in sorted(moms[0]):
        if sync_selects(layers, name):
            mean = mean_f32([m[name] for m in moms])
            for r in range(len(moms)):
                out[r][name] = mean.astype(np.float64).reshape(
                    np.asarray(moms[r][name]).shape)
    return out


def hash_params(params: Mapping[str, np.ndarray]) -> str:
    """``hash_params`` (optimizer.py:34-40)."""
    import hashlib
    hs = hashlib.sha256()
    for name in sorted(params):
        hs.update(name.encode())
        hs.update(np.ascontiguousarray(params[name], dtype="<f8").tobytes())
    return hs.hexdigest()


# ---------------------------------------------------------------------------
# Synthetic inputs (runner.py:289-297 make_worker_updates; workloads.py:154-175)
# ---------------------------------------------------------------------------

def synth_rank_inputs(seed: int, world: int, sizes: Mapping[str, tuple],
                      kind: str = "laplace", beta1: float = 0.9):
    """Seeded fp32 per-rank (theta, m, g) dicts.  theta is shared across
    ranks (data-parallel replicas); g_r = base + Laplace noise with a shared
    Laplace base (runner.py:289-297), m_r ~ 0.1 N(0,1).  Kinds add the edge
    cases the reference tests exercise: ``ties`` (iid +-1 grads, m = 0:
    test_collectives.py:174-186), ``zeros`` (exact zeros and -0.0, the
    alternating fill), ``outliers`` (laplace_with_outliers, workloads.py:165-
    171), ``cancel`` (m = -(1-b1)/b1 g, near-cancelling c)."""
    base_rng = np.random.default_rng(np.random.SeedSequence([seed, 10_000]))
    theta, base = {}, {}
    for name, shape in sizes.items():
        n = int(np.prod(shape)) if len(shape) else 1
        theta[name] = base_rng.normal(size=shape).astype(np.float32)
        b = base_rng.laplace(0.0, 1.0, size=n)
        if kind == "outliers":
            k = min(4, n)
            idx = base_rng.choice(n, size=k, replace=False)
            b[idx] = 1e3 * base_rng.choice([-1.0, 1.0], size=k)
        base[name] = b.reshape(shape)
    ranks = []
    for r in range(world):
        rng = np.random.default_rng(np.random.SeedSequence([seed, r]))
        g, m = {}, {}
        for name, shape in sizes.items():
            if kind == "ties":
                gg = rng.choice([-1.0, 1.0], size=shape)
                mm = np.zeros(shape)
            else:
                gg = base[name] + rng.laplace(0.0, 1.0, size=shape)
                mm = 0.1 * rng.normal(size=shape)
            gg = np.asarray(gg, dtype=np.float32)
            mm = np.asarray(mm, dtype=np.float32)
            if kind == "zeros":
                z = rng.random(size=shape) < 0.05
                gg = np.where(z, np.float32(0.0), gg)
                mm = np.where(z, np.float32(0.0), mm)
                negz = rng.random(size=shape) < 0.02
                gg = np.where(negz, np.float32(-0.0), gg)
                mm = np.where(negz, np.float32(-0.0), mm)
            if kind == "cancel":
                mm = (-(1.0 - beta1) / beta1 * gg.astype(np.float64)).astype(np.float32)
            g[name] = np.ascontiguousarray(gg, dtype=np.float32)
            m[name] = np.ascontiguousarray(mm, dtype=np.float32)
        ranks.append({"theta": {k: v.copy() for k, v in theta.items()},
                      "m": m, "g": g})
    return ranks


def f32_ulp_diff(a, b) -> np.ndarray:
    """|a-b| in units of float32 ulps (for tolerance statements)."""
    a = np.asarray(a, dtype=np.float32).view(np.int32).astype(np.int64)
    b = np.asarray(b, dtype=np.float32).view(np.int32).astype(np.int64)
    a = np.where(a < 0, -(a & 0x7FFFFFFF), a)
    b = np.where(b < 0, -(b & 0x7FFFFFFF), b)
    return np.abs(a - b)


def fsum_mean(xs: Sequence[np.ndarray]) -> np.ndarray:
    """Compensated mean oracle of the reference tests
    (test_collectives.py:210-224)."""
    cast = [np.asarray(x, dtype=np.float32).astype(np.float64).ravel() for x in xs]
    n = cast[0].size
    return np.array([math.fsum(c[i] for c in cast) / len(cast) for i in range(n)])
