"""The production peer-memory kernels driven directly through the C ABI on
ONE GPU: ``lc_vote_apply`` (owner vote + push to every rank + theta update
with per-owner waits), ``lc_vote_update`` (allgather exchange: vote + update
from P replicated rows) and ``lc_encode`` in ``LC_ENC_REPLICATE`` mode --
P simulated ranks whose buffers all live on this GPU (k_vote_apply of the
P ranks runs concurrently on P streams and synchronises through the real
epoch flags), compared bit-exactly with the oracle (reference collectives.py:252-310 and optimizer.py:199-205).  Also
the failure contract: a flag that never arrives makes every kernel give up
after the timeout, write nothing, and name the missing rank.
"""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import lioncub_oracle as O
from tests.gpu_helpers import assert_f32_equal

pytestmark = pytest.mark.gpu

lc = pytest.importorskip("paper_2411_16462_b200")
from paper_2411_16462_b200 import _lib  # noqa: E402
from paper_2411_16462_b200.transport import host_wait  # noqa: E402
from paper_2411_16462_b200.collectives import owner_elems, owner_valid  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _lib.load()


LR, WD = 1e-3, 0.1


def _hyper():
    return _lib.Hyper(0.9, 1.0 - 0.9, 0.99, 1.0 - 0.99, LR, WD)


class _Ranks:
    """P simulated ranks' device state and peer-memory buffers on one GPU."""

    def __init__(self, P: int, n: int, seed: int, kind: str = "laplace"):
        self.P, self.n = P, n
        self.inputs = O.synth_rank_inputs(seed, P, {"w": (n,)}, kind)
        dev = "cuda"
        f = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)  # noqa
        self.theta = [f(r["theta"]["w"]) for r in self.inputs]
        self.m = [f(r["m"]["w"]) for r in self.inputs]
        self.g = [f(r["g"]["w"]) for r in self.inputs]
        self.L = owner_elems(n, P)
        self.cw = self.L // 32
        z = lambda k, dt=torch.int32: torch.zeros(k, dtype=dt, device=dev)  # noqa
        self.recv = [z(P * self.cw) for _ in range(P)]      # owner j: P slots
        self.full = [z(P * self.cw) for _ in range(P)]      # every rank: gather buffer
        self.nz = [z(P * self.cw) for _ in range(P)]
        self.flags = [torch.full((P,), 100, dtype=torch.int64, device=dev) for _ in range(P)]
        self.counter = [z(32) for _ in range(P)]
        self.err = [z(2) for _ in range(P)]
        self.kflags = [z(1) for _ in range(P)]
        # pinned step-verdict words (lc_sync.verdict)
        self.verdict = [torch.zeros(1, dtype=torch.int64, pin_memory=True) for _ in range(P)]

    def sync(self, r, wait, arrive, timeout=5.0, counter=0):
        sy = _lib.Sync()
        for j in range(self.P):
            sy.peer_flags[j] = self.flags[j].data_ptr()
        sy.my_flags = self.flags[r].data_ptr()
        sy.counter = self.counter[r].data_ptr() + 32 * counter
        sy.err = self.err[r].data_ptr()
        sy.wait_epoch, sy.arrive_epoch = wait, arrive
        sy.P, sy.rank, sy.timeout_s = self.P, r, timeout
        sy.verdict = self.verdict[r].data_ptr()
        return sy

    def oracle(self, algo, spec, it, zm):
        ins = self.inputs
        nt, nm, sign, ties, _, _ = O.distributed_step(
            [x["theta"] for x in ins], [x["m"] for x in ins], [x["g"] for x in ins],
            O.Hyper(0.9, 0.99, LR, WD), spec, algo, it, zero_mode=zm)
        return nt[0]["w"], [x["w"] for x in nm], sign["w"]


def _fill(zm, it):
    return 0 if zm == "exact-ternary" else O.zero_fill(it + 1)


CASES = [
    # (P, n, algo, bits, zero_mode, kind): owner-block tails, empty owners
    (2, 3 * 1024 + 517, "compressed1bit", None, "alternating", "laplace"),
    (4, 64 * 1024 + 33, "compressed1bit", None, "alternating", "ties"),
    (8, 5000, "compressed1bit", None, "alternating", "ties"),
    (8, 40 * 1024 + 999, "direct", 1, "alternating", "laplace"),
    (4, 9 * 1024 + 7, "direct", 1, "exact-ternary", "laplace"),
    (3, 20_000, "compressed1bit", None, "alternating", "cancel"),
]


@pytest.mark.parametrize("P,n,algo,bits,zm,kind", CASES)
def test_vote_apply_abi_matches_oracle(P, n, algo, bits, zm, kind):
    """K1 of every rank publishes e1; then the P ranks' k_vote_apply run
    CONCURRENTLY on P streams (grids sized for 1/P of the SMs so all are
    co-resident), each waiting in-kernel for e1 and, per owner block, for
    that owner's e2 -- the real barrier protocol, on one GPU."""
    it = 3
    R = _Ranks(P, n, seed=P * 131 + n % 97, kind=kind)
    for f in R.flags:
        f.zero_()
    fill = _fill(zm, it)
    sum_mode = 0 if algo == "compressed1bit" else 1
    nzmode = fill == 0 and sum_mode == 1
    hyp = _hyper()
    main = torch.cuda.current_stream()
    st = main.cuda_stream
    # K1: every rank's block j -> owner j's slot r (the all-to-all in the kernel)
    for r in range(P):
        dst = _lib.table([R.recv[j].data_ptr() + r * R.cw * 4 for j in range(P)])
        _lib.call("lc_encode", R.g[r].data_ptr(), R.m[r].data_ptr(), None, n, C.byref(hyp),
                  fill, _lib.LC_ENC_SIGN1, 1, None, dst, P, R.L, 0, R.kflags[r].data_ptr(),
                  C.byref(R.sync(r, 0, 7, counter=0)), st)
    th_ref, m_ref, sign_ref = R.oracle(algo, None if bits is None else O.Spec(bits), it, zm)
    streams = [torch.cuda.Stream() for _ in range(P)]
    lib = _lib.load()
    _lib.check(lib.lc_set_grid_divisor(P))
    try:
        for r in range(P):
            streams[r].wait_stream(main)
            vout = _lib.table([R.full[k].data_ptr() + r * R.cw * 4 for k in range(P)])
            nzout = _lib.table([R.nz[k].data_ptr() + r * R.cw * 4 for k in range(P)]) \
                if nzmode else None
            sy = R.sync(r, 7, 8, counter=1)
            _lib.call("lc_vote_apply", R.recv[r].data_ptr(), P, R.cw, owner_valid(n, P, r),
                      fill, sum_mode, vout, nzout, P, R.kflags[r].data_ptr(), C.byref(sy),
                      R.theta[r].data_ptr(), n, R.full[r].data_ptr(),
                      R.nz[r].data_ptr() if nzmode else None, LR, WD, streams[r].cuda_stream)
    finally:
        _lib.check(lib.lc_set_grid_divisor(1))
    torch.cuda.synchronize()
    # sign bit = voted +1 (a zero aggregate has bit 0 and nz 0 in ternary)
    words = O.pack_words((sign_ref > 0).astype(np.int64), 1)
    nzw = O.pack_words((sign_ref != 0).astype(np.int64), 1)
    # bits past n in the last word are wire padding (voted +1): compare valid bits
    valid = np.full(words.size, 0xFFFFFFFF, np.uint32)
    if n % 32:
        valid[-1] = (1 << (n % 32)) - 1
    for k in range(P):
        assert R.err[k].tolist() == [0, 0], f"rank {k} barrier error {R.err[k].tolist()}"
        got = R.full[k].cpu().numpy().view(np.uint32)[:words.size]
        assert np.array_equal(got & valid, words & valid), f"gather buffer of rank {k}"
        if nzmode:
            gz = R.nz[k].cpu().numpy().view(np.uint32)[:nzw.size]
            assert np.array_equal(gz & valid, nzw & valid)
        assert_f32_equal(R.theta[k].cpu().numpy(), th_ref, f"theta r{k}")
        assert_f32_equal(R.m[k].cpu().numpy(), m_ref[k], f"m r{k}")
        assert int(R.kflags[k][0]) == 0
        assert R.flags[k].tolist() == [8] * P     # every owner published e2
        assert int(R.verdict[k][0]) == 8 << 8     # the step verdict: e2, no flags


@pytest.mark.parametrize("P,n,algo,bits,zm,kind", CASES)
def test_replicate_encode_and_vote_update_abi_match_oracle(P, n, algo, bits, zm, kind):
    it = 4
    R = _Ranks(P, n, seed=P * 17 + n % 89, kind=kind)
    fill = _fill(zm, it)
    sum_mode = 0 if algo == "compressed1bit" else 1
    hyp = _hyper()
    st = torch.cuda.current_stream().cuda_stream
    row = max(32, -(-n // 1024) * 32)                    # words per replicated row
    rows = [torch.zeros(P * row, dtype=torch.int32, device="cuda") for _ in range(P)]
    for r in range(P):   # K1 replicate: rank r's words into row r of EVERY rank
        dst = _lib.table([rows[k].data_ptr() + r * row * 4 for k in range(P)])
        _lib.call("lc_encode", R.g[r].data_ptr(), R.m[r].data_ptr(), None, n, C.byref(hyp),
                  fill, _lib.LC_ENC_SIGN1 | _lib.LC_ENC_REPLICATE, 1, None, dst, P, row * 32,
                  0, R.kflags[r].data_ptr(), C.byref(R.sync(r, 0, 9)), st)
    torch.cuda.synchronize()
    cs = [0.9 * x["m"]["w"].astype(np.float64) + (1.0 - 0.9) * x["g"]["w"].astype(np.float64)
          for x in R.inputs]
    for k in range(P):
        got = rows[k].cpu().numpy().view(np.uint32).reshape(P, row)
        for r in range(P):
            s = O.apply_sign(cs[r], "alternating" if fill else "exact-ternary", it + 1)
            ref = O.pack_signs(np.where(s == 0, 1, s))
            valid = np.full(ref.size, 0xFFFFFFFF, np.uint32)
            if n % 32:
                valid[-1] = (1 << (n % 32)) - 1
            assert np.array_equal(got[r, :ref.size] & valid, ref & valid), f"row {r} on rank {k}"
    th_ref, m_ref, _ = R.oracle(algo, None if bits is None else O.Spec(bits), it, zm)
    for r in range(P):
        _lib.call("lc_vote_update", rows[r].data_ptr(), row, P, R.theta[r].data_ptr(), n, fill,
                  sum_mode, LR, WD, R.kflags[r].data_ptr(), C.byref(R.sync(r, 9, 0)), st)
    torch.cuda.synchronize()
    for r in range(P):
        assert_f32_equal(R.theta[r].cpu().numpy(), th_ref, f"theta r{r}")
        assert_f32_equal(R.m[r].cpu().numpy(), m_ref[r], f"m r{r}")
        assert int(R.err[r][0]) == 0
        assert int(R.verdict[r][0]) == 9 << 8     # verdict at the wait epoch e1


def test_vote_apply_large_offsets_and_double_buffered_slots():
    """Two consecutive steps through the production Python path on the
    fused simulated transport at P = 4: the second step's K1 writes the
    other half of the owners' receive slots (the write-after-read hazard of
    the in-warp own-block vote), and the result equals two oracle steps."""
    P, sizes = 4, {"emb": (70_001,), "w": (131_072,)}
    ranks = O.synth_rank_inputs(5, P, sizes, "laplace")
    h = O.Hyper(0.9, 0.99, 1e-3, 0.0)
    f32 = lambda d: {k: np.asarray(v, np.float32).astype(np.float64) for k, v in d.items()}  # noqa
    th = [f32(ranks[0]["theta"])] * P
    ms = [f32(r["m"]) for r in ranks]
    for i in range(2):
        nt, nm, *_ = O.distributed_step(th, ms, [r["g"] for r in ranks], h, None,
                                        "compressed1bit", i)
        th, ms = [f32(t) for t in nt], [f32(m) for m in nm]

    def fn(topo):
        r = ranks[topo.rank]
        st = lc.WorkerState.initial({k: torch.from_numpy(v).cuda() for k, v in r["theta"].items()})
        for k, v in r["m"].items():
            st.momentum[k].copy_(torch.from_numpy(v))
        g = st.new_grad_buffer()
        for k, v in r["g"].items():
            g[k].copy_(torch.from_numpy(v))
        for _ in range(2):
            st = lc.distributed_lion_step(st, g, lc.LionHyper(lr=1e-3), None, topo,
                                          "compressed1bit")
        host_wait()
        return {k: v.cpu().numpy() for k, v in st.params.items()}

    res = lc.run_ranks(P, fn, transport=lc.LocalTransport(P, fused=True))
    for r in range(P):
        for k in sizes:
            assert_f32_equal(res[r][k], th[r][k], f"theta {k} r{r}")


# ---- failure contract ------------------------------------------------------

def test_kernels_time_out_on_a_missing_rank_and_write_nothing():
    """Rank 1 never publishes: rank 0's vote_apply / vote_update /
    apply_update / barrier give up after the timeout, leave theta and the
    gather buffers untouched, and report rank 1 in the error words."""
    P, n = 2, 4096
    R = _Ranks(P, n, seed=3)
    R.flags[0].zero_()                       # nobody has arrived anywhere
    st = torch.cuda.current_stream().cuda_stream
    th0 = R.theta[0].clone()
    full0 = R.full[0].clone()
    flags_pub = lambda: R.flags[0][0].fill_(50)  # rank 0 itself "arrived"  # noqa
    flags_pub()
    vout = _lib.table([R.full[k].data_ptr() for k in range(P)])
    sy = R.sync(0, 50, 51, timeout=0.2, counter=1)
    _lib.call("lc_vote_apply", R.recv[0].data_ptr(), P, R.cw, owner_valid(n, P, 0), 1, 0, vout,
              None, P, R.kflags[0].data_ptr(), C.byref(sy), R.theta[0].data_ptr(), n,
              R.full[0].data_ptr(), None, LR, WD, st)
    torch.cuda.synchronize()
    assert R.err[0].tolist() == [_lib.LC_FLAG_BARRIER_TIMEOUT, 1 << 1]
    assert int(R.verdict[0][0]) == (51 << 8) | _lib.LC_FLAG_BARRIER_TIMEOUT
    assert torch.equal(R.theta[0], th0) and torch.equal(R.full[0], full0)
    assert int(R.flags[1][0]) == 100         # no epoch published to the peer
    row = 32 * -(-n // 1024)
    rows = torch.zeros(P * row, dtype=torch.int32, device="cuda")
    R.err[0].zero_()
    _lib.call("lc_vote_update", rows.data_ptr(), row, P, R.theta[0].data_ptr(), n, 1, 0, LR, WD,
              R.kflags[0].data_ptr(), C.byref(R.sync(0, 50, 0, timeout=0.2)), st)
    tbl = _lib.table([R.full[0].data_ptr()])
    _lib.call("lc_apply_update", R.theta[0].data_ptr(), n, tbl, None, 1, P * R.cw, 0, LR, WD,
              C.byref(R.sync(0, 50, 0, timeout=0.2)), st)
    torch.cuda.synchronize()
    assert R.err[0].tolist() == [_lib.LC_FLAG_BARRIER_TIMEOUT, 1 << 1]
    assert int(R.verdict[0][0]) == (50 << 8) | _lib.LC_FLAG_BARRIER_TIMEOUT
    assert torch.equal(R.theta[0], th0)
    R.err[0].zero_()
    _lib.call("lc_barrier", _lib.table([f.data_ptr() for f in R.flags]), P, 0,
              R.flags[0].data_ptr(), 60, 0.2, R.err[0].data_ptr(), st)
    torch.cuda.synchronize()
    assert R.err[0].tolist() == [_lib.LC_FLAG_BARRIER_TIMEOUT, 1 << 1]


@pytest.mark.parametrize("algo", ["compressed1bit", "direct"])
def test_step_raises_collective_error_naming_missing_rank(algo):
    """Public API, production fused path: rank 1 stops calling the step.
    Rank 0's step raises CollectiveError(rank=1) in the SAME call, leaves
    theta (and the iteration) as they were, and the transport refuses
    further use."""
    P = 4 if algo == "direct" else 2
    sizes = {"w": (50_000,)}
    ranks = O.synth_rank_inputs(9, P, sizes, "laplace")
    tp = lc.LocalTransport(P, fused=True, timeout=1.0)
    spec = lc.QuantSpec(bits=1) if algo == "direct" else None
    out = {}

    def fn(topo):
        r = ranks[topo.rank]
        st = lc.WorkerState.initial({"w": torch.from_numpy(r["theta"]["w"]).cuda()})
        g = st.new_grad_buffer()
        g["w"].copy_(torch.from_numpy(r["g"]["w"]))
        st = lc.distributed_lion_step(st, g, lc.LionHyper(lr=1e-3), spec, topo, algo)
        host_wait()
        if topo.rank == 1:
            return None                      # rank 1 dies after step 1
        before = st.params["w"].clone()
        with pytest.raises(lc.CollectiveError) as ei:
            lc.distributed_lion_step(st, g, lc.LionHyper(lr=1e-3), spec, topo, algo)
        host_wait()
        out[topo.rank] = (ei.value.rank, torch.equal(st.params["w"], before), st.iteration)
        with pytest.raises(lc.CollectiveError, match="unusable"):
            lc.distributed_lion_step(st, g, lc.LionHyper(lr=1e-3), spec, topo, algo)
        return None

    lc.run_ranks(P, fn, transport=tp)
    for r, (who, same, it) in out.items():
        assert who == 1, (r, who)
        assert same, f"theta changed on rank {r}"
        assert it == 1
