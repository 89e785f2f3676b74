"""Multi-GPU NCCL parity (needs >= 2 B200s; skipped otherwise)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


MODES = {
    # default policy (allgather at P = 2, owner vote above)
    "nvlink-default": {"LIONCUB_P2P": "1"},
    # allgather exchange forced: K1 -> every rank, K5v votes + updates
    "nvlink-allgather": {"LIONCUB_P2P": "1", "LIONCUB_AG_MAX_P": "64"},
    # owner vote forced: K1 -> owner, fused vote + voted-word push + update
    "nvlink-owner-vote": {"LIONCUB_P2P": "1", "LIONCUB_AG_MAX_P": "1"},
    "nccl": {"LIONCUB_P2P": "0"},
}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_process_per_gpu_parity(nproc, mode):
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={29600 + 8 * nproc + list(MODES).index(mode)}",
           os.path.join(ROOT, "tests", "mgpu_parity.py")]
    env = dict(os.environ, **MODES[mode])
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    assert '"failures_all_ranks": 0' in res.stdout


@pytest.mark.parametrize("p2p", [True, False], ids=["nvlink-peer-memory", "nccl"])
def test_thread_per_gpu_run_ranks(p2p):
    """One process, one thread per GPU (ncclCommInitAll + peer access),
    reference-style run_ranks: the vote collective and a full 1-bit step
    with momentum sync equal the oracle on every rank."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    import paper_2411_16462_b200 as lc
    from oracle import lioncub_oracle as O
    from tests.gpu_helpers import assert_f32_equal, run_step_case
    tp = lc.NcclTransport.init_all(list(range(n)))
    tp.p2p = p2p
    rng = np.random.default_rng(0)
    cs = [rng.normal(size=100_003) for _ in range(n)]
    expect = O.vote_1bit(cs, "alternating", 1)

    def fn(topo):
        x = torch.from_numpy(cs[topo.rank]).to(topo.device)
        v = lc.compressed_allreduce_1bit(x, topo, lc.SignPolicy("alternating", 1))
        return v.values.cpu().numpy(), v.ties

    try:
        for vals, ties in lc.run_ranks(n, fn, transport=tp):
            assert np.array_equal(vals, expect.values)
            assert ties == expect.ties
        sizes = {"a": (70_001,), "b": (4_099,)}
        ranks = O.synth_rank_inputs(5, n, sizes, "laplace")
        h = O.Hyper(0.9, 0.99, 1e-3, 0.1)
        nt, nm, sign, ties, _, _ = O.distributed_step(
            [r["theta"] for r in ranks], [r["m"] for r in ranks], [r["g"] for r in ranks],
            h, None, "compressed1bit", 9)
        nm = O.sync_momentum(nm, 10, "all", 10)
        case = dict(world=n, lr=1e-3, wd=0.1, bits=None, algo="compressed1bit",
                    iteration=9, zero_mode="alternating", sync=(10, "all"))
        res = run_step_case(case, ranks[0]["theta"], [r["m"] for r in ranks],
                            [r["g"] for r in ranks], transport=tp)
        for r, (th, m, met, _) in enumerate(res):
            for k in sizes:
                assert_f32_equal(th[k], nt[0][k], f"theta {k}")
                assert_f32_equal(m[k], nm[r][k], f"m {k}")
                assert met["ties"][k] == ties[k]
        # production path (no metrics): the allgather exchange on peer memory
        nt, nm, *_ = O.distributed_step(
            [r["theta"] for r in ranks], [r["m"] for r in ranks], [r["g"] for r in ranks],
            h, O.Spec(1), "direct", 9)
        case = dict(world=n, lr=1e-3, wd=0.1, bits=1, algo="direct", iteration=9,
                    zero_mode="alternating")
        res = run_step_case(case, ranks[0]["theta"], [r["m"] for r in ranks],
                            [r["g"] for r in ranks], transport=tp, metrics=False)
        for r, (th, m, _, _) in enumerate(res):
            for k in sizes:
                assert_f32_equal(th[k], nt[0][k], f"theta {k}")
                assert_f32_equal(m[k], nm[r][k], f"m {k}")
    finally:
        tp.close()


def _lioncomm():
    """The unmodified reference, pip-installed in baseline/_ref (travels with
    the repo snapshot; /root/reference does not exist on the GPU box)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "lioncomm")):
        pytest.skip("baseline/_ref has no lioncomm install")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import lioncomm.collectives as RC
    import lioncomm.quant as RQ
    import lioncomm.transport as RT
    return RC, RQ, RT


def test_reference_collectives_over_nccl_frame_transport():
    """The reference's own Python collectives (compressed_allreduce_1bit,
    direct_allreduce, allreduce_mean_f32, ps_gather_broadcast) run unchanged
    over NcclFrameTransport -- the Transport interface of transport.py:32-45
    with frames crossing NVLink -- and give the results they give over the
    reference's InprocTransport."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    import paper_2411_16462_b200 as lc
    RC, RQ, RT = _lioncomm()
    P = min(n, 4)
    rng = np.random.default_rng(5)
    cs = [rng.normal(size=10_007).astype(np.float32).astype(np.float64) for _ in range(P)]
    qs = [rng.integers(-7, 8, size=10_007) for _ in range(P)]

    def fn(topo):
        r = topo.rank
        a = RC.compressed_allreduce_1bit(cs[r], topo, RQ.SignPolicy("alternating", 3))
        b = RC.direct_allreduce(qs[r], topo, q_max=7)
        c = RC.allreduce_mean_f32(cs[r], topo)
        d = RC.ps_gather_broadcast(cs[r], topo, efficient=True)
        return a.values, a.ties, b.values, b.ties, c, d.values

    eps = lc.NcclFrameTransport.init_all(list(range(P)))
    got = RC.run_ranks(P, fn, transport_factory=lambda r: eps[r])
    ref = RC.run_ranks(P, fn, transport=RT.InprocTransport(P))
    for g, e in zip(got, ref):
        for x, y in zip(g, e):
            assert np.array_equal(np.asarray(x), np.asarray(y))


@pytest.mark.parametrize("p2p", [True, False], ids=["nvlink-in-kernel-barriers", "nccl"])
def test_dead_rank_raises_collective_error_naming_it(p2p):
    """Thread-per-GPU, real NVLink: rank 1 stops after step 1.  Rank 0's
    step 2 raises CollectiveError(rank=1) in the same call -- from the
    kernels' barrier timeout (peer memory) or from the host deadline that
    polls ncclCommGetAsyncError and aborts the communicator (NCCL) -- and
    theta is unchanged."""
    n = _ngpu()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    import paper_2411_16462_b200 as lc
    import torch
    tp = lc.NcclTransport.init_all([0, 1])
    tp.p2p = p2p
    tp.timeout = 3.0
    out = {}

    def fn(topo):
        dev = topo.device
        st = lc.WorkerState.initial({"w": torch.randn(300_000, device=dev,
                                                      generator=torch.Generator(dev).manual_seed(0))})
        g = st.new_grad_buffer()
        g["w"].copy_(torch.randn(300_000, device=dev))
        st = lc.distributed_lion_step(st, g, lc.LionHyper(lr=1e-3), None, topo, "compressed1bit")
        torch.cuda.synchronize(dev)
        if topo.rank == 1:
            return
        before = st.params["w"].clone()
        with pytest.raises(lc.CollectiveError) as ei:
            lc.distributed_lion_step(st, g, lc.LionHyper(lr=1e-3), None, topo, "compressed1bit")
        torch.cuda.synchronize(dev)
        out["who"] = ei.value.rank
        out["same"] = bool(torch.equal(st.params["w"], before))

    lc.run_ranks(2, fn, transport=tp)
    assert out == {"who": 1, "same": True}
