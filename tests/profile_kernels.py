"""Single-GPU driver for ncu captures of the step kernels (one process).

    python tests/profile_kernels.py [--n N] [--P P] [--reps R]

Runs the owner-blocked encode (K1, 1-bit, P blocks into a local buffer), the
1-bit vote (K4) and the theta update (K5) on an N-param buffer, timing each
with CUDA events; prints one JSON line.  Under ncu, pick a kernel with
`-k regex:k_encode` etc.
"""

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2411_16462_b200 import _lib  # noqa: E402
from paper_2411_16462_b200.collectives import owner_elems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    n, P = args.n, args.P
    dev = torch.device("cuda", 0)
    g = torch.randn(n, device=dev)
    m = torch.randn(n, device=dev) * 0.1
    th = torch.randn(n, device=dev)
    L = owner_elems(n, P)
    cw = L // 32
    send = torch.zeros(P * cw, dtype=torch.int32, device=dev)
    full = torch.zeros(P * cw, dtype=torch.int32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    hyp = _lib.Hyper(0.9, 1.0 - 0.9, 0.99, 1.0 - 0.99, 1e-4, 0.0)
    dst = _lib.table([send.data_ptr() + j * cw * 4 for j in range(P)])
    vout = _lib.table([full.data_ptr()])
    s = torch.cuda.current_stream().cuda_stream
    res = {"n": n, "P": P}

    def timed(name, fn, nbytes):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        res[name] = {"ms": ms, "GBps": nbytes / ms / 1e6}

    timed("encode_1bit", lambda: _lib.call(
        "lc_encode", g.data_ptr(), m.data_ptr(), None, n, C.byref(hyp), 1,
        _lib.LC_ENC_SIGN1, 1, None, dst, P, L, 0, flags.data_ptr(), None, s), 12 * n + n / 8)
    timed("vote_bits", lambda: _lib.call(
        "lc_vote_bits", send.data_ptr(), P, cw, L, 1, 0, vout, None, None, 1,
        flags.data_ptr(), None, s), (P + 1) * cw * 4)
    timed("apply_update", lambda: _lib.call(
        "lc_apply_update", th.data_ptr(), n, _lib.table([send.data_ptr()]), None, 1,
        P * cw, 0, 1e-4, 0.0, None, s),
        8 * n + n / 8)
    # allgather exchange: K1 replicating into P local rows, K5v over P rows
    row = -(-n // 1024) * 32
    rows = torch.zeros(P * row, dtype=torch.int32, device=dev)
    rdst = _lib.table([rows.data_ptr() + j * row * 4 for j in range(P)])
    timed("encode_replicate", lambda: _lib.call(
        "lc_encode", g.data_ptr(), m.data_ptr(), None, n, C.byref(hyp), 1,
        _lib.LC_ENC_SIGN1 | _lib.LC_ENC_REPLICATE, 1, None, rdst, P, row * 32, 0,
        flags.data_ptr(), None, s), 12 * n + P * n / 8)
    timed("vote_update", lambda: _lib.call(
        "lc_vote_update", rows.data_ptr(), row, P, th.data_ptr(), n, 1, 0, 1e-4, 0.0,
        flags.data_ptr(), None, s), 8 * n + P * n / 8)
    timed("fused_local", lambda: _lib.call(
        "lc_fused_local_step", th.data_ptr(), m.data_ptr(), g.data_ptr(), None, n,
        C.byref(hyp), 1, _lib.LC_LOCAL_BINARY, None, None, None, None, flags.data_ptr(), s),
        20 * n)
    # per-layer numpy-exact L1 norm on the GPT-2-small layout (148 layers)
    sys.path.insert(0, ROOT)
    from bench import gpt2_small_layout
    import paper_2411_16462_b200 as lc
    lay = lc.Layout(gpt2_small_layout())
    nl = lay.n
    gl = torch.randn(nl, device=dev)
    ml = torch.randn(nl, device=dev) * 0.1
    arr = (C.c_int64 * len(lay.seg_start))(*lay.seg_start)
    plan = C.c_void_p()
    _lib.check(_lib.load().lc_l1_plan_create(C.byref(plan), arr, len(lay.names)))
    norms = torch.zeros(len(lay.names), dtype=torch.float64, device=dev)
    scales = torch.zeros_like(norms)
    timed("l1_scales_gpt2", lambda: _lib.call(
        "lc_l1_scales", plan.value, gl.data_ptr(), ml.data_ptr(), None, C.byref(hyp), 15,
        norms.data_ptr(), scales.data_ptr(), s), 16 * nl)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
