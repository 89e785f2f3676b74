"""Case table shared by the golden generator and the parity tests."""

import zlib

# Sorted-name layer layout of every step case (flat vectors, as the
# reference votes return raveled values): a weight, a tiny bias,
# a word-sized layer and an odd-sized layer so flat offsets are unaligned.
SIZES = {
    "a.weight": (1000,),
    "b.bias": (7,),
    "c": (64,),
    "d": (1501,),
}


def _c(name, algo, world, kind, iteration=0, wd=0.0, bits=None,
       zero_mode="alternating", seed=None, lr=1e-3, **extra):
    d = dict(name=name, algo=algo, world=world, kind=kind, iteration=iteration,
             wd=wd, bits=bits, zero_mode=zero_mode,
             seed=seed if seed is not None else zlib.crc32(name.encode()) % 10_000,
             lr=lr)
    d.update(extra)
    return d


STEP_CASES = [
    # 1-bit compressed vote (collectives.py:252-310)
    _c("c1", "compressed1bit", 1, "laplace", seed=11),
    _c("c2", "compressed1bit", 2, "ties", iteration=1, wd=0.1, seed=12),
    _c("c3", "compressed1bit", 3, "zeros", seed=13),
    _c("c4", "compressed1bit", 4, "laplace", iteration=1, seed=14),
    _c("c5", "compressed1bit", 8, "cancel", wd=0.1, seed=15),
    _c("c6", "compressed1bit", 4, "ties", seed=16, mask="a.weight"),
    _c("c7", "compressed1bit", 8, "ties", iteration=1, seed=17),
    # sum-of-signs p-bit (direct, QuantSpec(bits=1))
    _c("d1", "direct", 1, "laplace", iteration=1, bits=1, seed=21),
    _c("d2", "direct", 2, "ties", bits=1, seed=22),
    _c("d3", "direct", 3, "zeros", iteration=1, bits=1, seed=23),
    _c("d4", "direct", 8, "laplace", wd=0.1, bits=1, seed=24),
    _c("d5", "direct", 4, "ties", iteration=1, bits=1, seed=25),
    # L1 p-bit (direct, QuantSpec(bits=b, norm_p=1))
    _c("q1", "direct", 1, "outliers", bits=5, seed=31),
    _c("q2", "direct", 2, "laplace", iteration=1, bits=5, seed=32),
    _c("q3", "direct", 8, "outliers", bits=5, seed=33),
    _c("q4", "direct", 4, "laplace", iteration=1, wd=0.1, bits=8, seed=34),
    _c("q5", "direct", 3, "zeros", bits=8, zero_mode="exact-ternary", seed=35),
    _c("q6", "direct", 4, "laplace", bits=2, seed=36),
    _c("q7", "direct", 2, "ties", bits=3, iteration=1, seed=37, mask="d"),
    # quantizer variants (quant.py:127-173): max norm, other p, geometric
    # mean, log map, no_zero (nearest rounding; stochastic is statistical)
    _c("x1", "direct", 4, "outliers", bits=5, seed=61, quant=dict(norm_p=float("inf"))),
    _c("x2", "direct", 2, "laplace", iteration=1, bits=4, seed=62, quant=dict(norm_p=2.0)),
    _c("x3", "direct", 3, "zeros", bits=8, seed=63, quant=dict(norm_p=0.0)),
    _c("x4", "direct", 8, "laplace", bits=5, seed=64, quant=dict(log_transform=True)),
    _c("x5", "direct", 4, "ties", bits=3, seed=65, quant=dict(no_zero=True)),
    _c("x6", "direct", 1, "outliers", bits=5, seed=66, quant=dict(norm_p=3.0)),
    _c("x7", "direct", 2, "laplace", bits=5, seed=67, mask="d",
       quant=dict(norm_p=0.5, no_zero=True)),
    _c("x8", "direct", 4, "laplace", iteration=1, wd=0.1, bits=6, seed=68,
       quant=dict(norm_p=float("inf"), log_transform=True)),
    # full precision (ps / ps_efficient, spec=None)
    _c("p1", "ps", 1, "zeros", zero_mode="exact-ternary", seed=41),
    _c("p2", "ps", 2, "laplace", seed=42),
    _c("p3", "ps_efficient", 3, "cancel", zero_mode="exact-ternary", seed=43),
    _c("p4", "ps_efficient", 8, "laplace", iteration=1, seed=44),
    _c("p5", "ps", 4, "ties", zero_mode="exact-ternary", seed=45),
    _c("p6", "ps_efficient", 5, "ties", iteration=1, seed=46),
    # ps / ps_efficient over a QuantSpec: the int64 sum of apply_sign or
    # quantize outputs (optimizer.py:151-158), ternary zeros included
    _c("ps1", "ps", 4, "ties", bits=1, zero_mode="exact-ternary", seed=71),
    _c("ps2", "ps_efficient", 3, "zeros", bits=1, seed=72),
    _c("ps3", "ps", 2, "laplace", iteration=1, bits=5, seed=73),
    _c("ps4", "ps_efficient", 8, "outliers", bits=3, zero_mode="exact-ternary", seed=74),
    _c("ps5", "ps", 1, "zeros", bits=1, zero_mode="exact-ternary", seed=75),
    # selective momentum sync (optimizer.py:244-258) after the step
    _c("s1", "compressed1bit", 4, "laplace", iteration=9, seed=51,
       sync=(10, ["a.weight", "d"])),
    _c("s2", "direct", 3, "laplace", bits=1, seed=52, sync=(1, "all")),
    _c("s3", "ps", 8, "laplace", iteration=1, seed=53, sync=(2, "all")),
    _c("s4", "compressed1bit", 2, "laplace", iteration=4, seed=54,
       sync=(10, "all")),  # t=5: does not fire
]

COLLECTIVE_CASES = []
for _w in (2, 3, 4, 8):
    for _n in (1, 7, 64, 1000):
        COLLECTIVE_CASES.append(dict(name=f"dir_w{_w}_n{_n}", kind="direct",
                                     world=_w, n=_n, q_max=7, seed=_w * 7 + _n))
        COLLECTIVE_CASES.append(dict(name=f"cmp_w{_w}_n{_n}", kind="compressed",
                                     world=_w, n=_n, t=1 + (_n % 2),
                                     seed=_w + _n))
        COLLECTIVE_CASES.append(dict(name=f"mean_w{_w}_n{_n}", kind="mean",
                                     world=_w, n=_n, seed=_w * 31 + _n))
COLLECTIVE_CASES.append(dict(name="dirbin_w4_n100", kind="direct", world=4,
                             n=100, q_max=1, binary=True, seed=3))
COLLECTIVE_CASES.append(dict(name="dir15_w8_n257", kind="direct", world=8,
                             n=257, q_max=15, seed=5))


def quant_kwargs(case: dict) -> dict | None:
    """QuantSpec keyword arguments of a step case (None: spec=None)."""
    if case["bits"] is None:
        return None
    kw = dict(bits=case["bits"], norm_p=1.0)
    kw.update(case.get("quant") or {})
    return kw
