"""signSGD majority step and the divergence metrics on the GPU against the
reference's own outputs (tests/golden/golden_metrics.npz) and the
reference test-suite's known answers (test_optimizer.py:199-292,
test_collectives.py:226-235).  theta' equals float32 of the reference's
float64 result exactly; divergences are bit-identical float64."""

import numpy as np
import pytest
import torch

from tests import golden_io as G
from tests.gpu_helpers import EXCHANGES, assert_f32_equal, grads_like, make_state, make_transport

pytestmark = pytest.mark.gpu

lc = pytest.importorskip("paper_2411_16462_b200")
from paper_2411_16462_b200 import _lib  # noqa: E402
from paper_2411_16462_b200.transport import host_wait  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _lib.load()


@pytest.mark.parametrize("xchg", EXCHANGES)
@pytest.mark.parametrize("i", range(len(G.metrics_golden()[1]["signsgd"])))
def test_signsgd_and_divergence_match_reference(i, xchg):
    sizes = G.step_sizes()
    c = G.signsgd_case(i, sizes)
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=1e-3, weight_decay=0.1)

    def fn(topo):
        r = topo.rank
        st = make_state(c["theta"], c["m"][r], c["iteration"])
        g = grads_like(st, c["g"][r])
        g0 = g.flat.clone()
        st2 = lc.signsgd_majority_step(st, g, h, topo, algo=c["algo"],
                                       zero_mode=c["zero_mode"])
        div = lc.momentum_divergence(st2, topo)
        host_wait()
        assert torch.equal(g.flat.view(torch.int32), g0.view(torch.int32))  # grads untouched
        return ({k: v.cpu().numpy() for k, v in st2.params.items()},
                {k: v.cpu().numpy() for k, v in st2.momentum.items()}, div, st2.iteration)

    res = lc.run_ranks(c["world"], fn, transport=make_transport(c["world"], xchg))
    for r, (th, m, div, it) in enumerate(res):
        assert it == c["iteration"] + 1
        for k in sizes:
            assert_f32_equal(th[k], c["theta_out"][k], f"theta {k} r{r}")
            assert np.array_equal(m[k], c["m"][r][k])        # momentum untouched
            assert div[k] == c["div"][k], (k, div[k], c["div"][k])
    moms = [{k: torch.from_numpy(v).cuda() for k, v in c["m"][r].items()}
            for r in range(c["world"])]
    dm = lc.divergence_from_momenta(moms)
    assert all(dm[k] == c["divm"][k] for k in sizes)


def test_signsgd_reference_known_answers():
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=0.1, weight_decay=0.0)
    grads = [[1.0, 1.0], [2.0, -1.0], [-3.0, -1.0]]

    def fn(topo):
        st = lc.WorkerState.initial({"w": torch.zeros(2, device="cuda")})
        g = st.new_grad_buffer()
        g["w"].copy_(torch.tensor(grads[topo.rank]))
        st = lc.signsgd_majority_step(st, g, h, topo)
        return st.params["w"].cpu().tolist(), st.momentum["w"].cpu().tolist()

    for th, m in lc.run_ranks(3, fn):                # test_optimizer.py:200-211
        assert th == pytest.approx([-0.1, 0.1]) and m == [0.0, 0.0]

    def fn1(topo):
        st = lc.WorkerState.initial({"w": torch.zeros(2, device="cuda")})
        g = st.new_grad_buffer()
        g["w"].copy_(torch.tensor([5.0, -0.2]))
        st = lc.signsgd_majority_step(st, g, h, topo, zero_mode="exact-ternary")
        return st.params["w"].cpu().tolist()

    assert lc.run_ranks(1, fn1)[0] == pytest.approx([-0.1, 0.1])  # :213-223

    rng = np.random.default_rng(5)                   # :225-238
    world, n = 5, 64
    gs = [rng.normal(size=n).astype(np.float32) for _ in range(world)]
    agg = np.sum([np.where(g >= 0, 1, -1) for g in gs], axis=0)
    oracle = np.where(agg > 0, 1, np.where(agg < 0, -1, 1))
    h1 = lc.LionHyper(beta1=0.9, beta2=0.99, lr=1.0, weight_decay=0.0)

    def fn2(topo):
        st = lc.WorkerState.initial({"w": torch.zeros(n, device="cuda")})
        g = st.new_grad_buffer()
        g["w"].copy_(torch.from_numpy(gs[topo.rank]))
        return lc.signsgd_majority_step(st, g, h1, topo, algo="direct").params["w"].cpu().numpy()

    for th in lc.run_ranks(world, fn2):
        assert np.array_equal(th, -oracle.astype(np.float32))


def test_divergence_and_allgather_known_answers():
    cuda = lambda v: torch.tensor(v, dtype=torch.float32, device="cuda")  # noqa: E731
    assert lc.divergence_from_momenta([{"w": cuda([1.0] * 4)}, {"w": cuda([1.0] * 4)}]) \
        == {"w": 0.0}
    assert lc.divergence_from_momenta([{"w": cuda([1.0])}, {"w": cuda([3.0])}])["w"] == 1.0
    assert lc.divergence_from_momenta([{"w": cuda([0.0, 10.0])},
                                       {"w": cuda([0.0, 0.0])}])["w"] == 5.0
    vecs = [np.array([float(i), -float(i)]) for i in range(3)]

    def fn(topo):
        return [v.cpu().numpy() for v in
                lc.allgather_f64(torch.from_numpy(vecs[topo.rank]).cuda(), topo)]

    for out in lc.run_ranks(3, fn):                  # test_collectives.py:226-235
        assert len(out) == 3 and all(np.array_equal(out[i], vecs[i]) for i in range(3))
        assert out[0].dtype == np.float64


@pytest.mark.parametrize("xchg", ["peer-memory", "collectives"])
@pytest.mark.parametrize("name", [c["name"] for c in G.step_cases()])
def test_vote_agreement_and_phase_timing_match_reference(name, xchg):
    """The runner's per-step vote metrics (runner.py:171-182) through
    vote_agreement -- the vote sign against sign(allreduce_mean_f32(c_local))
    -- equal the reference's counts exactly; metrics_out carries the
    reference's phase-timing keys (t_quant only off the 1-bit path,
    optimizer.py:141-168) as positive device times."""
    gc = G.step_case(name)
    case = gc["case"]
    world = case["world"]
    from tests.golden.cases import quant_kwargs
    kw = quant_kwargs(case)
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=case["lr"], weight_decay=case["wd"])
    cmask = None
    if gc["mask"] is not None:
        cmask = {k: torch.from_numpy(np.asarray(v)).cuda() for k, v in gc["mask"].items()}

    def fn(topo):
        r = topo.rank
        st = make_state(gc["theta"], gc["m"][r], case["iteration"])
        g = grads_like(st, gc["g"][r])
        met = {}
        lc.distributed_lion_step(st, g, h, None if kw is None else lc.QuantSpec(**kw), topo,
                                 case["algo"], mask=cmask, zero_mode=case["zero_mode"],
                                 metrics_out=met)
        agree = lc.vote_agreement(met, topo)
        return agree, {k: met[k] for k in ("t_quant", "t_comm") if k in met}

    res = lc.run_ranks(world, fn, transport=make_transport(world, xchg))
    match, flip, counted = (int(x) for x in gc["agree"])
    has_q, has_c = (bool(x) for x in gc["timing_keys"])
    for agree, times in res:
        assert round(agree["sign_match"] * counted) == match, (agree, match)
        assert round(agree["flip_rate"] * counted) == flip, (agree, flip)
        assert round(agree["tie_rate"] * counted) == sum(gc["ties"].values())
        assert ("t_quant" in times) == has_q and ("t_comm" in times) == has_c
        assert all(v > 0 for v in times.values())
