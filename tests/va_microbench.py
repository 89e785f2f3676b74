"""Single-GPU microbenchmark of the 1-bit owner-vote step kernels at the
TinyLlama 1.1B size (a tuning tool, not a test): one rank's K1
(``lc_encode`` into its local slots), ``lc_vote_apply`` with every peer
flag pre-published (no waiting: the kernel's own throughput, without the
cross-rank skew a multi-GPU run adds), ``lc_apply_update`` (the NCCL-path
K5 over the same words) and the P = 1 fused step, each timed with CUDA
events over ``--iters`` launches.  Prints one JSON line.

    python tests/va_microbench.py [--n 1100048384] [--P 4] [--iters 20]
"""

import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_16462_b200 import _lib  # noqa: E402
from paper_2411_16462_b200.collectives import owner_elems, owner_valid  # noqa: E402


def timed(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_100_048_384)
    ap.add_argument("--P", type=int, default=4)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    lib = _lib.load()
    n, P, r = args.n, args.P, 0
    dev = "cuda"
    L = owner_elems(n, P)
    cw = L // 32
    theta = torch.randn(n, device=dev)
    m = torch.randn(n, device=dev)
    g = torch.randn(n, device=dev)
    recv = torch.randint(-2**31, 2**31 - 1, (P * cw,), dtype=torch.int32, device=dev)
    full = torch.randint(-2**31, 2**31 - 1, (P * cw,), dtype=torch.int32, device=dev)
    flags = [torch.full((P,), 1 << 40, dtype=torch.int64, device=dev) for _ in range(P)]
    counter = torch.zeros(32, dtype=torch.int32, device=dev)
    err = torch.zeros(2, dtype=torch.int32, device=dev)
    kflags = torch.zeros(1, dtype=torch.int32, device=dev)
    hyp = _lib.Hyper(0.9, 0.1, 0.99, 0.01, 1e-4, 0.1)
    s = torch.cuda.current_stream().cuda_stream

    def sync(wait, arrive, ctr):
        sy = _lib.Sync()
        for j in range(P):
            sy.peer_flags[j] = flags[j].data_ptr()
        sy.my_flags = flags[r].data_ptr()
        sy.counter = counter.data_ptr() + 32 * ctr
        sy.err = err.data_ptr()
        sy.wait_epoch, sy.arrive_epoch = wait, arrive
        sy.P, sy.rank, sy.timeout_s = P, r, 5.0
        return sy

    # peer flags never drop below the epochs waited on (arrivals store 2^40)
    sy1 = sync(0, 1 << 40, 0)
    sy2 = sync(1 << 40, 1 << 40, 1)
    dst = _lib.table([recv.data_ptr() + j * cw * 4 for j in range(P)])
    vout = _lib.table([full.data_ptr() + r * cw * 4 for _ in range(P)])
    out = {"n": n, "P": P}

    def enc():
        _lib.call("lc_encode", g.data_ptr(), m.data_ptr(), None, n, C.byref(hyp), 1,
                  _lib.LC_ENC_SIGN1, 1, None, dst, P, L, 0, kflags.data_ptr(), C.byref(sy1), s)

    def va():
        _lib.call("lc_vote_apply", recv.data_ptr(), P, cw, owner_valid(n, P, r), 1, 0, vout,
                  None, P, kflags.data_ptr(), C.byref(sy2), theta.data_ptr(), n,
                  full.data_ptr(), None, 1e-4, 0.1, s)

    bits = _lib.table([full.data_ptr()])

    def au():
        _lib.call("lc_apply_update", theta.data_ptr(), n, bits, None, 1, P * cw, 0, 1e-4, 0.1,
                  None, s)

    def fused():
        _lib.call("lc_fused_local_step", theta.data_ptr(), m.data_ptr(), g.data_ptr(), None, n,
                  C.byref(hyp), 1, _lib.LC_LOCAL_BINARY, None, None, None, None,
                  kflags.data_ptr(), s)

    bytes_ = {"encode": 12.125 * n, "vote_apply": 8.125 * n + P * cw * 4 / P,
              "apply_update": 8.125 * n, "fused_local": 20.0 * n}
    fns = {"encode": enc, "vote_apply": va, "apply_update": au, "fused_local": fused}
    sel = [k for k in fns if not args.only or k in args.only.split(",")]
    for k in sel:
        ms = timed(fns[k], args.iters)
        out[k] = {"ms": round(ms, 4), "GBs": round(bytes_[k] / ms / 1e6, 1)}
    e = err.cpu().tolist()
    out["err"] = e
    print(json.dumps(out))


if __name__ == "__main__":
    main()
