"""Parity of the CUDA path with the reference (golden vectors produced by the
real reference) and with the CPU oracle at larger sizes.  Needs a B200.

Tolerances: packed words, votes, ties, p-bit sums, quantized ints and c
(float64) are compared bit-for-bit.  theta' and m' are fp32 state: they must
equal float32 of the reference's float64 result exactly (0 ulp), because the
kernels compute the same float64 expression and round once.
"""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import lioncub_oracle as O
from tests import golden_io as G
from tests.golden.cases import quant_kwargs
from tests.gpu_helpers import (EXCHANGES, assert_f32_equal, make_transport, run_step_case,
                               step_seeds)

pytestmark = pytest.mark.gpu

lc = pytest.importorskip("paper_2411_16462_b200")
from paper_2411_16462_b200 import _lib  # noqa: E402
from paper_2411_16462_b200.transport import host_wait  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _lib.load()  # fail loudly if the extension is missing


STEP_NAMES = [c["name"] for c in G.step_cases()]


@pytest.mark.parametrize("xchg", EXCHANGES)
@pytest.mark.parametrize("name", STEP_NAMES)
def test_step_matches_reference_golden(name, xchg):
    """Both exchange modes: kernels storing into peers' buffers (NVLink
    path) and the collective path (NCCL path), simulated ranks on one GPU."""
    gc = G.step_case(name)
    case = gc["case"]
    res = run_step_case(case, gc["theta"], gc["m"], gc["g"], mask=gc["mask"],
                        transport=make_transport(case["world"], xchg),
                        metrics=xchg != "fused")
    for r, (th, m, met, it) in enumerate(res):
        assert it == case["iteration"] + 1
        for k in gc["sizes"]:
            assert_f32_equal(th[k], gc["theta_out"][k], f"{name} theta {k} r{r}")
            assert_f32_equal(m[k], gc["m_out"][r][k], f"{name} m {k} r{r}")
            if met is None:   # fused exchange: the production kernels, no metrics
                continue
            assert np.array_equal(met["vote_sign"][k], gc["sign"][k]), (name, k)
            assert met["ties"][k] == gc["ties"][k], (name, k, met["ties"][k])
            if gc["c"][r][k] is not None:
                assert np.array_equal(met["c_local"][k].view(np.int64),
                                      gc["c"][r][k].view(np.int64)), (name, k)


def _hyper(lr=1e-3, wd=0.0):
    return _lib.Hyper(0.9, 1.0 - 0.9, 0.99, 1.0 - 0.99, lr, wd)


@pytest.mark.parametrize("name", [c["name"] for c in G.step_cases()
                                  if c["algo"] == "compressed1bit"])
def test_packed_sign_words_bit_exact(name):
    """K1's 1-bit words == pack(apply_sign(c), 1, 1).payload (quant.py:255-281)."""
    gc = G.step_case(name)
    case = gc["case"]
    fill = 0 if case["zero_mode"] == "exact-ternary" else O.zero_fill(case["iteration"] + 1)
    for r in range(case["world"]):
        for k in gc["sizes"]:
            ref = gc["words"][r][k]
            if ref is None:
                continue
            g = torch.from_numpy(gc["g"][r][k]).cuda()
            m = torch.from_numpy(gc["m"][r][k].copy()).cuda()
            mask = None
            if gc["mask"] is not None and k in gc["mask"]:
                mask = torch.from_numpy(gc["mask"][k].astype(np.uint8)).cuda()
            n = g.numel()
            out = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
            flags = torch.zeros(1, dtype=torch.int32, device="cuda")
            hyp = _hyper()
            L = -(-n // 1024) * 1024
            _lib.call("lc_encode", g.data_ptr(), m.data_ptr(), _lib.ptr(mask), n,
                      C.byref(hyp), fill, _lib.LC_ENC_SIGN1, 1, None,
                      _lib.table([out.data_ptr()]), 1, L, 0, flags.data_ptr(), None, 0)
            got = out.cpu().numpy().view(np.uint32)
            nb = (n + 7) // 8  # reference payload bytes; compare the valid bits
            gb = got.view(np.uint8)[:nb].copy()
            rb = ref.view(np.uint8)[:nb].copy()
            if n % 8:
                keep = (1 << (n % 8)) - 1
                gb[-1] &= keep
                rb[-1] &= keep
            assert np.array_equal(gb, rb), (name, k, r)


@pytest.mark.parametrize("name", [c["name"] for c in G.step_cases()
                                  if c["bits"] is not None and c["bits"] > 1])
def test_l1_norm_and_quantized_ints_bit_exact(name):
    """numpy-order mean p-norm (quant.py:81-104) and q ints (quant.py:127-173)
    of every quantizer variant.  Norms: bit-exact for p in {1, 2, 0.5, inf}
    (numpy's own fast paths: copy, square, sqrt, max); for other p and p = 0
    numpy's SIMD pow/log differ from CUDA's by ulps, so those norms are
    within 1e-13 relative.  Quantized ints: bit-exact."""
    gc = G.step_case(name)
    case = gc["case"]
    sizes = gc["sizes"]
    names = sorted(sizes)
    spec = lc.QuantSpec(**quant_kwargs(case))
    qmax = spec.qmax
    exact_norm = spec.norm_p in (1.0, 2.0, 0.5, float("inf"))
    starts = [0]
    for k in names:
        starts.append(starts[-1] + int(np.prod(sizes[k])))
    n = starts[-1]
    arr = (C.c_int64 * len(starts))(*starts)
    plan = C.c_void_p()
    _lib.check(_lib.load().lc_l1_plan_create(C.byref(plan), arr, len(names)))
    try:
        for r in range(case["world"]):
            g = torch.from_numpy(np.concatenate([gc["g"][r][k] for k in names])).cuda()
            m = torch.from_numpy(np.concatenate([gc["m"][r][k] for k in names])).cuda()
            mask = None
            if gc["mask"] is not None:
                mk = np.concatenate([gc["mask"].get(k, np.ones(sizes[k], bool))
                                     for k in names]).astype(np.uint8)
                mask = torch.from_numpy(mk).cuda()
            norms = torch.zeros(len(names), dtype=torch.float64, device="cuda")
            scales = torch.zeros_like(norms)
            logs = None
            hyp = _hyper()
            args = (plan.value, g.data_ptr(), m.data_ptr(), _lib.ptr(mask), C.byref(hyp))
            if spec.log_transform:
                logs = torch.zeros_like(norms)
                _lib.call("lc_l1_scales", *args, qmax, logs.data_ptr(),
                          torch.zeros_like(norms).data_ptr(), 0)
            if spec.norm_p == 1.0 and logs is None:
                _lib.call("lc_l1_scales", *args, qmax, norms.data_ptr(), scales.data_ptr(), 0)
            else:
                ns = _lib.NormSpec(spec.norm_p, qmax, 0, _lib.ptr(logs))
                _lib.call("lc_norm_scales", *args, C.byref(ns), norms.data_ptr(),
                          scales.data_ptr(), 0)
            # the golden norm is lp_mean_norm(c, p): the quantizer's own norm
            # unless the log map is on (then the log scale M1(c) for p = 1)
            got_norms = (logs if logs is not None else norms).cpu().numpy()
            if logs is None or spec.norm_p == 1.0:
                for i, k in enumerate(names):
                    ref_n = float(gc["norm"][r][k])
                    if exact_norm or logs is not None:
                        assert got_norms[i] == ref_n, (name, k, r)
                    else:
                        assert abs(got_norms[i] - ref_n) <= 1e-13 * abs(ref_n), (name, k, r)
            # quantize into 32-bit fields and compare ints
            seg_start = torch.tensor(starts, dtype=torch.int64, device="cuda")
            segs = _lib.Segments(seg_start.data_ptr(), scales.data_ptr(), len(names), qmax,
                                 _lib.ptr(logs), spec.kernel_flags(), 0, 0)
            out = torch.zeros(n, dtype=torch.int32, device="cuda")
            flags = torch.zeros(1, dtype=torch.int32, device="cuda")
            _lib.call("lc_encode", g.data_ptr(), m.clone().data_ptr(), _lib.ptr(mask), n,
                      C.byref(hyp), 1, _lib.LC_ENC_QUANT_FIELDS, 32, C.byref(segs),
                      _lib.table([out.data_ptr()]), 1, -(-n // 1024) * 1024, 0,
                      flags.data_ptr(), None, 0)
            q = out.cpu().numpy().astype(np.int64) - qmax
            ref = np.concatenate([gc["q"][r][k].astype(np.int64) for k in names])
            assert np.array_equal(q, ref), (name, r)
    finally:
        _lib.load().lc_l1_plan_destroy(plan.value)


@pytest.mark.parametrize("name", [c["name"] for c in G.collective_cases()])
def test_collective_matches_reference_golden(name):
    gc = G.collective_case(name)
    case = gc["case"]
    world = case["world"]

    def fn(topo):
        x = torch.from_numpy(np.asarray(gc["inputs"][topo.rank])).cuda()
        if case["kind"] == "direct":
            v = lc.direct_allreduce(x, topo, q_max=case["q_max"],
                                    binary_signs=case.get("binary", False))
            return v.values.cpu().numpy(), v.ties
        if case["kind"] == "compressed":
            v = lc.compressed_allreduce_1bit(x, topo, lc.SignPolicy("alternating", case["t"]))
            return v.values.cpu().numpy(), v.ties
        return lc.allreduce_mean_f32(x, topo).cpu().numpy(), None

    for vals, ties in lc.run_ranks(world, fn):
        if case["kind"] == "mean":
            assert np.array_equal(vals.view(np.int32), gc["values"].view(np.int32))
        else:
            assert np.array_equal(vals, gc["values"])
            assert ties == gc["ties"]


# ---- larger sizes against the oracle ---------------------------------------

BIG = {"emb": (40_000,), "h0.w": (300_017,), "h1.w": (262_144,), "norm": (1_000,)}


@pytest.mark.parametrize("xchg", EXCHANGES)
@pytest.mark.parametrize("algo,bits,world,kind,zm", [
    ("compressed1bit", None, 4, "laplace", "alternating"),
    ("compressed1bit", None, 8, "ties", "alternating"),
    ("direct", 1, 8, "laplace", "alternating"),
    ("direct", 1, 3, "ties", "exact-ternary"),
    ("direct", 5, 8, "outliers", "alternating"),
    ("direct", 8, 4, "laplace", "exact-ternary"),
    ("ps", None, 4, "cancel", "exact-ternary"),
    ("ps_efficient", None, 8, "laplace", "alternating"),
    ("compressed1bit", None, 1, "laplace", "alternating"),
    ("direct", 5, 1, "outliers", "alternating"),
])
def test_step_matches_oracle_large(algo, bits, world, kind, zm, xchg):
    ranks = O.synth_rank_inputs(7, world, BIG, kind)
    h = O.Hyper(0.9, 0.99, 1e-4, 0.1)
    spec = None if bits is None else O.Spec(bits)
    it = 2
    nt, nm, sign, ties, _, _ = O.distributed_step(
        [rk["theta"] for rk in ranks], [rk["m"] for rk in ranks], [rk["g"] for rk in ranks],
        h, spec, algo, it, zero_mode=zm)
    case = dict(world=world, lr=1e-4, wd=0.1, bits=bits, algo=algo, iteration=it,
                zero_mode=zm)
    res = run_step_case(case, ranks[0]["theta"], [rk["m"] for rk in ranks],
                        [rk["g"] for rk in ranks],
                        transport=make_transport(world, xchg),
                        metrics=xchg != "fused")
    for r, (th, m, met, _) in enumerate(res):
        for k in BIG:
            assert_f32_equal(th[k], nt[0][k], f"theta {k}")
            assert_f32_equal(m[k], nm[r][k], f"m {k}")
            if met is not None:
                assert np.array_equal(met["vote_sign"][k], sign[k])
                assert met["ties"][k] == ties[k]


QVARIANTS = [
    dict(bits=5, norm_p=float("inf")),
    dict(bits=5, rounding="stochastic"),
    dict(bits=4, norm_p=float("inf"), rounding="stochastic", no_zero=True),
    dict(bits=8, norm_p=2.0, no_zero=True),
    dict(bits=5, log_transform=True),
    dict(bits=6, norm_p=0.5, log_transform=True, rounding="stochastic"),
]


@pytest.mark.parametrize("xchg", EXCHANGES)
@pytest.mark.parametrize("world", [1, 4])
@pytest.mark.parametrize("qi", range(len(QVARIANTS)))
def test_quant_variants_match_oracle_large(qi, world, xchg):
    """Every exactly-reproducible quantizer variant at 600K params: max norm,
    p = 2 / 0.5, log map, no_zero, and stochastic rounding -- the latter
    bit-exact against the oracle fed the same counter-based stream (its
    agreement with the reference's PCG64 draws is statistical, see
    test_stochastic_rounding_is_unbiased)."""
    kw = QVARIANTS[qi]
    ranks = O.synth_rank_inputs(11, world, BIG, "outliers")
    h = O.Hyper(0.9, 0.99, 1e-4, 0.1)
    seeds = step_seeds(500, world)
    it = 4
    nt, nm, sign, ties, _, _ = O.distributed_step(
        [rk["theta"] for rk in ranks], [rk["m"] for rk in ranks], [rk["g"] for rk in ranks],
        h, O.Spec(**kw), "direct", it, seeds=seeds)
    case = dict(world=world, lr=1e-4, wd=0.1, bits=kw["bits"], algo="direct", iteration=it,
                zero_mode="alternating", quant={k: v for k, v in kw.items() if k != "bits"},
                rng_seed=500)
    res = run_step_case(case, ranks[0]["theta"], [rk["m"] for rk in ranks],
                        [rk["g"] for rk in ranks],
                        transport=make_transport(world, xchg),
                        metrics=xchg != "fused")
    for r, (th, m, met, _) in enumerate(res):
        for k in BIG:
            if met is not None:
                assert np.array_equal(met["vote_sign"][k], sign[k]), (k, r)
                assert met["ties"][k] == ties[k]
            assert_f32_equal(th[k], nt[0][k], f"theta {k}")
            assert_f32_equal(m[k], nm[r][k], f"m {k}")


def test_stochastic_rounding_is_unbiased():
    """Statistical parity with the reference's sround (quant.py:107-116):
    every q is floor or ceil of the scaled value and E[q] = scaled.  One
    rank, one layer of 2^20 elements: the vote sign of each element is
    sign(q), so fix c and compare the fraction of +1 votes where the scaled
    value lies in (0, 1) with the mean fractional part."""
    n = 1 << 20
    rng = np.random.default_rng(3)
    g = (rng.random(n) * 0.5).astype(np.float32)          # c = 0.1 g in (0, 0.05)
    theta = np.zeros(n, np.float32)
    spec = lc.QuantSpec(bits=2, norm_p=float("inf"), rounding="stochastic")  # qmax 1

    def fn(topo):
        st = lc.WorkerState.initial({"w": torch.from_numpy(theta).cuda()})
        gb = st.new_grad_buffer()
        gb["w"].copy_(torch.from_numpy(g))
        met = {}
        lc.distributed_lion_step(st, gb, lc.LionHyper(lr=1.0), spec, topo, "direct",
                                 zero_mode="exact-ternary", rng=np.random.default_rng(9),
                                 metrics_out=met)
        with pytest.raises(lc.ConfigError, match="rng"):
            lc.distributed_lion_step(st, gb, lc.LionHyper(), spec, topo, "direct")
        return met

    met = lc.run_ranks(1, fn)[0]
    c = 0.1 * g.astype(np.float64)
    scaled = c / c.max()                     # in (0, 1]: q in {0, 1}
    up = met["vote_sign"]["w"].cpu().numpy() == 1
    assert abs(up.mean() - scaled.mean()) < 3e-3
    lo = scaled < 0.25
    assert abs(up[lo].mean() - scaled[lo].mean()) < 5e-3


@pytest.mark.parametrize("xchg", EXCHANGES)
@pytest.mark.parametrize("world,layers,algo,bits", [
    (8, ("emb", "h1.w"), "compressed1bit", None),
    (8, "all", "compressed1bit", None),        # fused into the step (fused exchange)
    (4, "all", "direct", 1),                   # sum-of-signs + fused sync
    (3, "all", "compressed1bit", None),
])
def test_momentum_sync_matches_oracle_large(xchg, world, layers, algo, bits):
    ranks = O.synth_rank_inputs(3, world, BIG, "laplace")
    h = O.Hyper(0.9, 0.99, 1e-4, 0.0)
    nt, nm, *_ = O.distributed_step([rk["theta"] for rk in ranks], [rk["m"] for rk in ranks],
                                    [rk["g"] for rk in ranks], h,
                                    None if bits is None else O.Spec(bits), algo, 9)
    sel = "all" if layers == "all" else frozenset(layers)
    synced = O.sync_momentum(nm, 10, sel, 10)
    case = dict(world=world, lr=1e-4, wd=0.0, bits=bits, algo=algo,
                iteration=9, zero_mode="alternating",
                sync=(10, "all" if layers == "all" else list(layers)))
    res = run_step_case(case, ranks[0]["theta"], [rk["m"] for rk in ranks],
                        [rk["g"] for rk in ranks], metrics=False,
                        transport=make_transport(world, xchg))
    for r, (th, m, _, _) in enumerate(res):
        for k in BIG:
            assert_f32_equal(m[k], synced[r][k], f"m {k} r{r}")
            assert_f32_equal(th[k], nt[0][k], f"theta {k} r{r}")


# ---- edge sizes and multi-step trajectories --------------------------------

EDGE_SIZES = [
    {"x": (1,)},
    {"x": (33,)},
    {"a": (1,), "b": (1025,), "c": (4097,)},
    {"a": (31,), "b": (32,), "c": (1023,), "d": (1024,), "e": (3, 7)},
]


@pytest.mark.parametrize("xchg", EXCHANGES)
@pytest.mark.parametrize("si", range(len(EDGE_SIZES)))
@pytest.mark.parametrize("algo,bits,world,zm", [
    ("compressed1bit", None, 3, "alternating"),
    ("direct", 1, 4, "alternating"),
    ("direct", 6, 5, "exact-ternary"),
    ("ps", None, 2, "exact-ternary"),
    ("ps_efficient", None, 4, "alternating"),
    ("direct", 5, 1, "alternating"),
])
def test_edge_sizes_match_oracle(algo, bits, world, zm, si, xchg):
    """Vectors smaller than one owner block / one warp tile / one word, and
    layer boundaries off the 32- and 1024-element grids: most ranks own
    nothing and every tail path runs."""
    sizes = EDGE_SIZES[si]
    ranks = O.synth_rank_inputs(11 + si, world, sizes, "ties")
    h = O.Hyper(0.9, 0.99, 1e-3, 0.1)
    spec = None if bits is None else O.Spec(bits)
    nt, nm, sign, ties, _, _ = O.distributed_step(
        [rk["theta"] for rk in ranks], [rk["m"] for rk in ranks], [rk["g"] for rk in ranks],
        h, spec, algo, 4, zero_mode=zm)
    case = dict(world=world, lr=1e-3, wd=0.1, bits=bits, algo=algo, iteration=4, zero_mode=zm)
    res = run_step_case(case, ranks[0]["theta"], [rk["m"] for rk in ranks],
                        [rk["g"] for rk in ranks], transport=make_transport(world, xchg),
                        metrics=xchg != "fused")
    for r, (th, m, met, _) in enumerate(res):
        for k in sizes:
            assert_f32_equal(th[k], nt[0][k], f"theta {k}")
            assert_f32_equal(m[k], nm[r][k], f"m {k}")
            if met is not None:
                assert np.array_equal(met["vote_sign"][k].reshape(-1), sign[k].reshape(-1))
                assert met["ties"][k] == ties[k]


@pytest.mark.parametrize("xchg", EXCHANGES)
@pytest.mark.parametrize("algo,bits,world,zm,sync", [
    ("compressed1bit", None, 4, "alternating", (2, ["emb"])),
    ("compressed1bit", None, 4, "alternating", (2, "all")),   # fused sync every other step
    ("direct", 1, 3, "alternating", (1, "all")),              # fused sync every step
    ("direct", 1, 3, "alternating", None),
    ("direct", 5, 4, "exact-ternary", (3, "all")),
    ("ps", None, 2, "exact-ternary", None),
])
def test_multi_step_trajectory_matches_oracle(algo, bits, world, zm, sync, xchg):
    """Six consecutive steps on the device-resident state (workspaces,
    epochs and symmetric buffers reused) against the oracle fed the fp32-
    rounded state each step -- the fp32-state contract of DESIGN.md."""
    sizes = {"emb": (5_003,), "w": (70_000,), "b": (96,)}
    ranks = O.synth_rank_inputs(23, world, sizes, "laplace")
    h = O.Hyper(0.9, 0.99, 1e-3, 0.1)
    spec = None if bits is None else O.Spec(bits)
    f32 = lambda d: {k: np.asarray(v, np.float32).astype(np.float64) for k, v in d.items()}  # noqa: E731
    thetas = [f32(ranks[0]["theta"])] * world
    moms = [f32(rk["m"]) for rk in ranks]
    steps, it0 = 6, 0
    for i in range(steps):
        nt, nm, sign, ties, _, _ = O.distributed_step(
            thetas, moms, [rk["g"] for rk in ranks], h, spec, algo, it0 + i, zero_mode=zm)
        nm = [f32(m) for m in nm]
        if sync is not None:
            layers = "all" if sync[1] == "all" else frozenset(sync[1])
            nm = O.sync_momentum(nm, sync[0], layers, it0 + i + 1)
        thetas = [f32(t) for t in nt]
        moms = [f32(m) for m in nm]
    case = dict(world=world, lr=1e-3, wd=0.1, bits=bits, algo=algo, iteration=it0,
                zero_mode=zm, sync=sync)
    res = run_step_case(case, ranks[0]["theta"], [rk["m"] for rk in ranks],
                        [rk["g"] for rk in ranks], transport=make_transport(world, xchg),
                        metrics=xchg != "fused",
                        steps=steps)
    for r, (th, m, met, it) in enumerate(res):
        assert it == it0 + steps
        for k in sizes:
            assert_f32_equal(th[k], thetas[r][k], f"theta {k} r{r}")
            assert_f32_equal(m[k], moms[r][k], f"m {k} r{r}")
            if met is not None:
                assert np.array_equal(met["vote_sign"][k], sign[k])
                assert met["ties"][k] == ties[k]


# ---- reference error behaviour ---------------------------------------------

def test_capacity_guard_before_any_communication():
    tp = lc.LocalTransport(125)
    topo = lc.Topology(world_size=125, rank=0, transport=tp)
    with pytest.raises(lc.CapacityError):
        lc.direct_allreduce(torch.zeros(4, dtype=torch.int64, device="cuda"), topo,
                            q_max=15, lane_bits=8)
    assert all(p is None for p in tp._posts)


def test_step_capacity_error_propagates():
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=0.01)
    topo = lc.Topology(world_size=10 ** 8, rank=0, transport=lc.LocalTransport(1))
    st = lc.WorkerState.initial({"w": torch.zeros(2, device="cuda")})
    with pytest.raises(lc.CapacityError):
        lc.distributed_lion_step(st, {"w": torch.ones(2, device="cuda")}, h,
                                 lc.QuantSpec(bits=8), topo, "direct")


def test_direct_requires_spec_and_zero_rejection():
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=0.01)

    def fn(topo):
        st = lc.WorkerState.initial({"w": torch.zeros(2, device="cuda")})
        return lc.distributed_lion_step(st, {"w": torch.ones(2, device="cuda")}, h,
                                        None, topo, "direct")

    with pytest.raises(lc.ConfigError):
        lc.run_ranks(2, fn)

    def zeros(topo):
        return lc.compressed_allreduce_1bit(torch.zeros(3, device="cuda"), topo,
                                            lc.SignPolicy("exact-ternary"))

    with pytest.raises(lc.ConfigError):
        lc.run_ranks(2, zeros)


def test_timeout_names_missing_rank():
    def fn(topo):
        if topo.rank == 1:
            return None
        return lc.compressed_allreduce_1bit(torch.ones(8, device="cuda"), topo,
                                            lc.SignPolicy("alternating", 1))

    with pytest.raises(lc.CollectiveError) as e:
        lc.run_ranks(2, fn, timeout=0.3)
    assert "1" in str(e.value)


def test_tie_parity_two_steps():
    """test_optimizer.py:137-153: t=1 tie -> theta -= lr; t=2 -> cancels."""
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=0.5)
    grads = [torch.tensor([1.0]), torch.tensor([-1.0])]

    def fn(topo):
        st = lc.WorkerState.initial({"w": torch.zeros(1, device="cuda")})
        g = {"w": grads[topo.rank].cuda()}
        st = lc.distributed_lion_step(st, g, h, lc.QuantSpec(bits=1), topo, "compressed1bit")
        first = st.params["w"].cpu().tolist()
        st = lc.distributed_lion_step(st, g, h, lc.QuantSpec(bits=1), topo, "compressed1bit")
        return first, st.params["w"].cpu().tolist()

    for first, second in lc.run_ranks(2, fn):
        assert first == [-0.5]
        assert second == [0.0]


def test_tie_rates():
    """test_collectives.py:174-186: C(P,P/2)/2^P."""
    n = 100_000
    for world, expect in ((4, 0.375), (8, 0.2734375)):
        rng = np.random.default_rng(world)
        cs = [torch.from_numpy(rng.choice([-1.0, 1.0], size=n)).cuda() for _ in range(world)]

        def fn(topo):
            return lc.compressed_allreduce_1bit(cs[topo.rank], topo,
                                                lc.SignPolicy("alternating", 1)).ties

        assert abs(lc.run_ranks(world, fn)[0] / n - expect) < 0.01


def test_lion_step_single_worker():
    """test_optimizer.py:25-43."""
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=0.1)
    st = lc.WorkerState.initial({"w": torch.zeros(1, device="cuda")})
    st = lc.lion_step(st, {"w": torch.tensor([2.0], device="cuda")}, h)
    assert st.params["w"].cpu().tolist() == [np.float32(-0.1)]
    assert st.iteration == 1
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=0.1, weight_decay=0.1)
    st = lc.WorkerState.initial({"w": torch.ones(1, device="cuda")})
    st = lc.lion_step(st, {"w": torch.zeros(1, device="cuda")}, h)
    assert st.params["w"].cpu().tolist() == [np.float32(0.99)]


def test_cpu_tensors_fail_loudly():
    h = lc.LionHyper()
    with pytest.raises(lc.ConfigError):
        lc.WorkerState.initial({"w": torch.zeros(3)})
    st = lc.WorkerState.initial({"w": torch.zeros(3, device="cuda")})
    topo = lc.Topology(1, 0, lc.LocalTransport(1))
    with pytest.raises(lc.ConfigError):
        lc.distributed_lion_step(st, {"w": torch.zeros(3)}, h, None, topo, "compressed1bit")


def test_reciprocal_division_is_correctly_rounded():
    """The norm kernel divides |c| by the layer max with a precomputed
    reciprocal + one FMA correction; it must equal IEEE division bitwise."""
    rng = np.random.default_rng(11)
    n = 20_000_000
    b = np.exp(rng.uniform(-700, 700, size=n)) * rng.choice([1.0, 3.0, 7.0], size=n)
    a = b * rng.uniform(0.0, 1.0, size=n)
    a[::7] = b[::7] * (1.0 - 2.0 ** -52)          # adversarial: just below b
    a[::11] = np.nextafter(b[::11], 0.0)
    a[::13] = b[::13]
    a[::17] = 0.0
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.call("lc_debug_div_check", da.data_ptr(), db.data_ptr(), n, bad.data_ptr(), 0)
    assert int(bad.item()) == 0


@pytest.mark.parametrize("sizes", [
    {"a": (1_000_003,), "b": (7,), "c": (3_000_000,), "d": (8191,), "e": (8193,), "f": (129,)},
    {"w": (4_194_305,)},
])
def test_l1_norms_bit_exact_large(sizes):
    """Per-layer numpy L1 norms (np.mean pairwise order) on multi-million
    element layers with outliers, and the quantized ints."""
    ranks = O.synth_rank_inputs(9, 1, sizes, "outliers")
    names = sorted(sizes)
    starts = [0]
    for k in names:
        starts.append(starts[-1] + int(np.prod(sizes[k])))
    g = np.concatenate([ranks[0]["g"][k] for k in names])
    m = np.concatenate([ranks[0]["m"][k] for k in names])
    c = 0.9 * m.astype(np.float64) + (1.0 - 0.9) * g.astype(np.float64)
    ref = [O.lp_mean_norm_l1(c[starts[i]:starts[i + 1]]) for i in range(len(names))]
    arr = (C.c_int64 * len(starts))(*starts)
    plan = C.c_void_p()
    _lib.check(_lib.load().lc_l1_plan_create(C.byref(plan), arr, len(names)))
    try:
        gt, mt = torch.from_numpy(g).cuda(), torch.from_numpy(m).cuda()
        norms = torch.zeros(len(names), dtype=torch.float64, device="cuda")
        scales = torch.zeros_like(norms)
        hyp = _hyper()
        _lib.call("lc_l1_scales", plan.value, gt.data_ptr(), mt.data_ptr(), None, C.byref(hyp),
                  127, norms.data_ptr(), scales.data_ptr(), 0)
        assert norms.cpu().numpy().tolist() == ref
    finally:
        _lib.load().lc_l1_plan_destroy(plan.value)


@pytest.mark.parametrize("xchg", EXCHANGES)
@pytest.mark.parametrize("algo,bits,world,chunk", [
    ("compressed1bit", None, 1, 65536), ("direct", 1, 1, 1 << 20), ("direct", 5, 1, 4096),
    ("compressed1bit", None, 3, 65536), ("direct", 1, 4, 3 * 1024), ("direct", 5, 2, 65536),
    ("ps", None, 2, 100_000),
])
def test_host_buffer_step_matches_device_step(algo, bits, world, chunk, xchg):
    """distributed_lion_step_host (pipelined pinned-host grads in, theta out)
    == distributed_lion_step on device buffers, bit for bit."""
    sizes = {"a": (150_001,), "b": (7,), "c": (65_536,)}
    ranks = O.synth_rank_inputs(21, world, sizes, "laplace")
    case = dict(world=world, lr=1e-3, wd=0.1, bits=bits, algo=algo, iteration=4,
                zero_mode="alternating")
    ref = run_step_case(case, ranks[0]["theta"], [r["m"] for r in ranks],
                        [r["g"] for r in ranks], metrics=False,
                        transport=make_transport(world, xchg))
    h = lc.LionHyper(0.9, 0.99, 1e-3, 0.1)
    spec = None if bits is None else lc.QuantSpec(bits=bits)
    names = sorted(sizes)

    def fn(topo):
        from tests.gpu_helpers import make_state
        r = ranks[topo.rank]
        st = make_state(r["theta"], r["m"], 4)
        host_g = torch.from_numpy(np.concatenate([r["g"][k] for k in names])).pin_memory()
        out = torch.empty(host_g.numel(), dtype=torch.float32).pin_memory()
        st = lc.distributed_lion_step_host(st, host_g, h, spec, topo, algo,
                                           params_out=out, chunk=chunk)
        host_wait()
        return out.numpy().copy(), {k: v.cpu().numpy() for k, v in st.momentum.items()}

    got = lc.run_ranks(world, fn, transport=make_transport(world, xchg))
    for r in range(world):
        th_flat, mom = got[r]
        exp_th = np.concatenate([ref[r][0][k] for k in names])
        assert np.array_equal(th_flat.view(np.int32), exp_th.view(np.int32))
        for k in names:
            assert np.array_equal(mom[k].view(np.int32), ref[r][1][k].view(np.int32))


def test_torch_optim_lioncub_trains_and_matches_step():
    """LionCub (torch.optim front end) on a small MLP: the model's params
    are the flat state; one step equals distributed_lion_step on the same
    gradient; replicas stay bit-identical across simulated ranks."""
    torch.manual_seed(0)

    def make():
        return torch.nn.Sequential(torch.nn.Linear(16, 32), torch.nn.Tanh(),
                                   torch.nn.Linear(32, 1)).cuda()

    init = {k: v.clone() for k, v in make().state_dict().items()}  # same replica everywhere
    world = 3
    xs = [torch.randn(64, 16, device="cuda") for _ in range(world)]
    ys = [x.sum(dim=1, keepdim=True).sin() for x in xs]

    def fn(topo):
        model = make()
        model.load_state_dict(init)
        opt = lc.LionCub(model.named_parameters(), topo, lr=1e-2,
                         spec=lc.QuantSpec(bits=1), algo="direct")
        losses = []
        for _ in range(30):
            opt.zero_grad()
            loss = torch.nn.functional.mse_loss(model(xs[topo.rank]), ys[topo.rank])
            loss.backward()
            opt.step()
            losses.append(float(loss.detach()))
        torch.cuda.synchronize()
        flat = opt.lion_state.params.flat.cpu().numpy()
        return losses, flat

    res = lc.run_ranks(world, fn)
    for _, flat in res[1:]:
        assert np.array_equal(flat.view(np.int32), res[0][1].view(np.int32))
    for losses, _ in res:
        assert losses[-1] < 0.7 * losses[0]


def test_torch_optim_step_equals_functional_step():
    model = torch.nn.Linear(8, 4).cuda()
    topo = lc.Topology(1, 0, lc.LocalTransport(1))
    opt = lc.LionCub(model.named_parameters(), topo, lr=1e-3, weight_decay=0.1,
                     spec=None, algo="compressed1bit")
    x = torch.randn(5, 8, device="cuda")
    opt.zero_grad()
    model(x).square().sum().backward()
    g = {k: v.clone() for k, v in opt.grads.items()}
    theta0 = {k: v.clone() for k, v in opt.lion_state.params.items()}
    opt.step()
    st = lc.WorkerState.initial(theta0)
    st = lc.distributed_lion_step(st, g, lc.LionHyper(0.9, 0.99, 1e-3, 0.1), None, topo,
                                  "compressed1bit")
    for k in g:
        assert torch.equal(st.params[k], opt.lion_state.params[k])
    assert torch.equal(model.weight.detach(), opt.lion_state.params["weight"])


@pytest.mark.parametrize("algo,bits", [("compressed1bit", None), ("direct", 1), ("ps", None)])
def test_step_graph_replay_equals_eager(algo, bits):
    """StepGraph (CUDA-graph replay of the P=1 step, odd/even fill graphs)
    == distributed_lion_step, bit for bit, over several steps."""
    sizes = {"a": (70_001,), "b": (129,)}
    ranks = O.synth_rank_inputs(4, 1, sizes, "zeros")
    h = lc.LionHyper(0.9, 0.99, 1e-3, 0.1)
    spec = None if bits is None else lc.QuantSpec(bits=bits)
    topo = lc.Topology(1, 0, lc.LocalTransport(1))
    from tests.gpu_helpers import grads_like, make_state
    zm = "exact-ternary" if algo == "ps" else "alternating"
    a = make_state(ranks[0]["theta"], ranks[0]["m"], 0)
    b = make_state(ranks[0]["theta"], ranks[0]["m"], 0)
    ga, gb = grads_like(a, ranks[0]["g"]), grads_like(b, ranks[0]["g"])
    graph = lc.StepGraph(b, gb, h, spec, topo, algo, zero_mode=zm)
    for _ in range(5):
        a = lc.distributed_lion_step(a, ga, h, spec, topo, algo, zero_mode=zm)
        b = graph.step()
    torch.cuda.synchronize()
    assert a.iteration == b.iteration == 5
    assert torch.equal(a.params.flat, b.params.flat)
    assert torch.equal(a.momentum.flat, b.momentum.flat)


@pytest.mark.gpu
def test_checkpoint_resume_equals_continuous(tmp_path):
    """save_checkpoint / load_checkpoint (reference format) mid-run: resuming
    from the checkpoint continues bit-identically to the uninterrupted run."""
    sizes = {"a": (3, 1001), "b": (17,)}
    ranks = O.synth_rank_inputs(5, 1, sizes, "laplace")
    h = lc.LionHyper(0.9, 0.99, 1e-3, 0.1)
    topo = lc.Topology(1, 0, lc.LocalTransport(1))
    from tests.gpu_helpers import grads_like, make_state
    a = make_state(ranks[0]["theta"], ranks[0]["m"], 0)
    ga = grads_like(a, ranks[0]["g"])
    for _ in range(3):
        a = lc.distributed_lion_step(a, ga, h, None, topo, "compressed1bit")
    path = str(tmp_path / "ck.bin")
    lc.save_checkpoint(path, a, h)
    b, side = lc.load_checkpoint(path)
    assert side["iteration"] == 3 and b.params.flat.is_cuda
    gb = grads_like(b, ranks[0]["g"])
    for _ in range(3):
        a = lc.distributed_lion_step(a, ga, h, None, topo, "compressed1bit")
        b = lc.distributed_lion_step(b, gb, h, None, topo, "compressed1bit")
    torch.cuda.synchronize()
    assert a.iteration == b.iteration == 6
    assert torch.equal(a.params.flat[:a.params.layout.n], b.params.flat[:b.params.layout.n])
    assert torch.equal(a.momentum.flat[:a.params.layout.n], b.momentum.flat[:b.params.layout.n])


@pytest.mark.parametrize("world,algo,bits,xchg", [
    (1, "compressed1bit", None, "peer-memory"),
    (1, "direct", 1, "peer-memory"),
    (1, "ps", None, "peer-memory"),
    (2, "compressed1bit", None, "fused"),      # allgather exchange
    (3, "direct", 1, "fused"),                # owner vote, sum-of-signs
    (4, "compressed1bit", None, "fused"),
])
def test_lioncub_overlap_backward_equals_plain(world, algo, bits, xchg, monkeypatch):
    """LionCub(overlap_backward=True) encodes 1024-aligned chunks of the flat
    buffer from post-accumulate-grad hooks while backward runs; six training
    steps give the bit-identical state of the ordinary step."""
    from paper_2411_16462_b200 import overlap
    monkeypatch.setattr(overlap, "CHUNK", 1 << 14)
    torch.manual_seed(1)

    def make():
        return torch.nn.Sequential(torch.nn.Linear(64, 512), torch.nn.Tanh(),
                                   torch.nn.Linear(512, 256), torch.nn.Tanh(),
                                   torch.nn.Linear(256, 1)).cuda()

    init = {k: v.clone() for k, v in make().state_dict().items()}
    xs = [torch.randn(128, 64, device="cuda") for _ in range(world)]
    ys = [x.sum(dim=1, keepdim=True).sin() for x in xs]

    def run(overlap_on):
        def fn(topo):
            model = make()
            model.load_state_dict(init)
            opt = lc.LionCub(model.named_parameters(), topo, lr=1e-3,
                             spec=None if bits is None else lc.QuantSpec(bits=bits), algo=algo,
                             overlap_backward=overlap_on)
            if overlap_on:
                assert opt._early is not None, "configuration should overlap"
            for _ in range(6):
                opt.zero_grad()
                torch.nn.functional.mse_loss(model(xs[topo.rank]), ys[topo.rank]).backward()
                opt.step()
            host_wait()
            return opt.lion_state.params.flat.cpu().numpy(), opt.lion_state.momentum.flat.cpu().numpy()
        return lc.run_ranks(world, fn, transport=make_transport(world, xchg))

    plain, over = run(False), run(True)
    for (tp_, mp_), (to_, mo_) in zip(plain, over):
        assert np.array_equal(tp_.view(np.int32), to_.view(np.int32))
        assert np.array_equal(mp_.view(np.int32), mo_.view(np.int32))


@pytest.mark.parametrize("world,algo,bits", [(4, "compressed1bit", None), (3, "direct", 1),
                                             (8, "compressed1bit", None)])
def test_selective_sync_fused_into_step_matches_oracle(world, algo, bits, monkeypatch):
    """sync=SyncPolicy(period, {layers}) passed to the step on the production
    exchange with LIONCUB_SYNC_FUSE=1: each owner's pull of the selected
    layers runs beside the theta update inside the step (mode "pull"); three
    steps (the sync firing on the second) equal the oracle's step +
    maybe_sync_momentum."""
    import paper_2411_16462_b200.optimizer as opt
    monkeypatch.setattr(opt, "SYNC_FUSE", "1")
    sizes = {"emb": (40_000,), "h0.w": (300_017,), "h1.w": (262_144,), "norm": (1_000,)}
    sel = ["emb", "h1.w"]
    ranks = O.synth_rank_inputs(13, world, sizes, "laplace")
    h = O.Hyper(0.9, 0.99, 1e-4, 0.1)
    spec = None if bits is None else O.Spec(bits)
    f32 = lambda d: {k: np.asarray(v, np.float32).astype(np.float64) for k, v in d.items()}  # noqa
    thetas = [f32(ranks[0]["theta"])] * world
    moms = [f32(rk["m"]) for rk in ranks]
    it0 = 0
    for i in range(3):
        nt, nm, *_ = O.distributed_step(thetas, moms, [rk["g"] for rk in ranks], h, spec, algo,
                                        it0 + i)
        nm = O.sync_momentum([f32(x) for x in nm], 2, frozenset(sel), it0 + i + 1)
        thetas, moms = [f32(x) for x in nt], [f32(x) for x in nm]
    case = dict(world=world, lr=1e-4, wd=0.1, bits=bits, algo=algo, iteration=it0,
                zero_mode="alternating", sync=(2, sel))
    res = run_step_case(case, ranks[0]["theta"], [rk["m"] for rk in ranks],
                        [rk["g"] for rk in ranks], metrics=False,
                        transport=make_transport(world, "fused"), steps=3)
    for r, (th, m, _, it) in enumerate(res):
        assert it == it0 + 3
        for k in sizes:
            assert_f32_equal(th[k], thetas[r][k], f"theta {k} r{r}")
            assert_f32_equal(m[k], moms[r][k], f"m {k} r{r}")
