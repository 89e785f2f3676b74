"""ctypes front end of oracle/lioncub_oracle.c (the C restatement used for
large parity checks).  TEST INFRASTRUCTURE ONLY -- see lioncub_oracle.py.

``build()`` compiles ``oracle/_build/liblcoracle.so`` with gcc (OpenMP,
``-ffp-contract=off``); ``__graft_entry__.build()`` calls it, and ``load()``
builds on first use when the library is missing or stale.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "lioncub_oracle.c")
LIB = os.path.join(HERE, "_build", "liblcoracle.so")

ALGOS = {"compressed1bit": 0, "direct_signs": 1, "direct_l1": 2, "ps": 3,
         "ps_efficient": 4, "ps_signs": 5}
ERRORS = {-1: "zero sign on a binary path", -2: "tie in exact-ternary 1-bit vote",
          -3: "bad arguments"}


class Hyper(C.Structure):
    _fields_ = [("beta1", C.c_double), ("one_minus_beta1", C.c_double),
                ("beta2", C.c_double), ("one_minus_beta2", C.c_double),
                ("lr", C.c_double), ("weight_decay", C.c_double)]


def hyper(beta1=0.9, beta2=0.99, lr=1e-4, wd=0.0) -> Hyper:
    return Hyper(beta1, 1.0 - beta1, beta2, 1.0 - beta2, lr, wd)


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
           "-shared", "-fPIC", SRC, "-o", tmp, "-lm"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"gcc failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


_lock = threading.Lock()
_lib = None


def load():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build())
            P = C.c_void_p
            lib.lco_step.restype = C.c_int
            lib.lco_step.argtypes = [C.c_int, C.c_int64, C.c_int, P, P, P, P, P, P, C.c_int,
                                     C.c_int, C.c_int, P, P, P, P]
            lib.lco_pairwise_sum.restype = C.c_double
            lib.lco_pairwise_sum.argtypes = [P, C.c_int64]
            lib.lco_l1_scales.restype = C.c_int
            lib.lco_l1_scales.argtypes = [C.c_int64, C.c_int, P, P, P, P, P, C.c_int, P]
            _lib = lib
        return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def step(theta, ms, gs, seg_start, h: Hyper, algo: str, fill: int, bits: int = 0,
         mask=None):
    """All P ranks' Lion Cub step on flat fp32 buffers (layers at
    ``seg_start``).  Returns (theta' f32, [m'_r f32], sign int8, ties
    int64[nseg]).  Raises ValueError for the reference's ConfigError cases."""
    P = len(ms)
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    n = theta.size
    ms = [np.ascontiguousarray(x, dtype=np.float32) for x in ms]
    gs = [np.ascontiguousarray(x, dtype=np.float32) for x in gs]
    seg = np.ascontiguousarray(seg_start, dtype=np.int64)
    nseg = seg.size - 1
    th_out = np.empty(n, np.float32)
    m_out = [np.empty(n, np.float32) for _ in range(P)]
    sign = np.empty(n, np.int8)
    ties = np.zeros(nseg, np.int64)
    arr = lambda xs: (C.c_void_p * P)(*[x.ctypes.data for x in xs])  # noqa: E731
    mk = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    rc = load().lco_step(P, n, nseg, _p(seg), _p(theta), arr(ms), arr(gs), _p(mk),
                         C.byref(h), ALGOS[algo], bits, fill, _p(th_out), arr(m_out),
                         _p(sign), _p(ties))
    if rc != 0:
        raise ValueError(ERRORS.get(rc, f"lco_step rc={rc}"))
    return th_out, m_out, sign, ties


def pairwise_sum(x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(load().lco_pairwise_sum(_p(x), x.size))


def algo_name(algo: str, spec_bits, zero_mode: str = "alternating") -> str:
    """The C oracle's mode of a reference (algo, QuantSpec.bits) pair
    (optimizer.py:137-169; L1 norms only)."""
    if algo == "compressed1bit":
        return "compressed1bit"
    if spec_bits is None:
        return algo
    if spec_bits == 1:
        return "direct_signs" if algo == "direct" else "ps_signs"
    return "direct_l1"
