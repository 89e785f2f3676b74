"""Pin the CPU oracle against the reference's own golden vectors (CPU only).

The fixtures were produced by the real reference (tests/golden/make_golden.py);
the hand-written known answers below are the reference tests' own
(pkg/tests/test_quant.py, test_collectives.py, test_optimizer.py).
"""

import numpy as np
import pytest

from oracle import lioncub_oracle as O
from tests import golden_io as G
from tests.golden.cases import quant_kwargs


# ---- known-answer tests of the reference test-suite ------------------------

def test_pack_golden_bytes():
    # test_quant.py:164-173
    assert O.pack_words(np.array([3, 12]), 4)[0] == 0xC3
    assert O.pack_words(np.array([1, 0, 1, 1, 0, 0, 0, 0]), 1)[0] == 0x0D
    assert O.pack_signs(np.array([-1, 1]))[0] == 0x02
    v = np.arange(16)
    assert O.unpack_words(O.pack_words(v, 4), 4, 16).tolist() == v.tolist()


def test_quantize_known_answers():
    # test_quant.py:38-44
    assert O.quantize_l1(np.array([1.0, -1, 1, -1]), 4).tolist() == [4, -4, 4, -4]
    assert O.quantize_l1(np.array([7.0, 1, 1, 1]), 4).tolist() == [7, 1, 1, 1]
    assert not O.quantize_l1(np.zeros(5), 8).any()
    rng = np.random.default_rng(1)
    x = rng.laplace(size=257)
    for c in (1e-6, 0.5, 3.0, 1e7):  # test_quant.py:60-65
        assert np.array_equal(O.quantize_l1(c * x, 8), O.quantize_l1(x, 8))


def test_norm_known_answers():
    assert O.lp_mean_norm_l1(np.array([1, -1, 1, -1])) == 1.0
    with pytest.raises(O.OracleConfigError):
        O.lp_mean_norm_l1(np.array([]))


def test_sign_policy():
    # test_quant.py:143-160
    assert O.apply_sign(np.array([2.5, -0.1, 0.0]), "exact-ternary", 0).tolist() == [1, -1, 0]
    assert O.apply_sign(np.array([0.0]), "alternating", 3).tolist() == [1]
    assert O.apply_sign(np.array([0.0]), "alternating", 4).tolist() == [-1]
    assert O.apply_sign(np.array([-0.0, 0.0]), "alternating", 1).tolist() == [1, 1]


def test_lane_bits():
    # test_collectives.py:118-124
    assert O.choose_lane_bits(8, 15) == 8
    assert O.choose_lane_bits(125, 15) == 16
    assert O.choose_lane_bits(2, 7) == 8
    assert O.choose_lane_bits(125, 1, binary_signs=True) == 8
    with pytest.raises(O.OracleCapacityError):
        O.choose_lane_bits(10 ** 9, 127)


def test_hand_lion_step():
    # test_optimizer.py:25-31, :39-43
    h = O.Hyper(0.9, 0.99, 0.1, 0.0)
    nt, nm = O.lion_step({"w": np.array([0.0])}, {"w": np.array([0.0])},
                         {"w": np.array([2.0])}, h)
    assert nt["w"].tolist() == [-0.1]
    assert nm["w"][0] == pytest.approx(0.02)
    h = O.Hyper(0.9, 0.99, 0.1, 0.1)
    nt, _ = O.lion_step({"w": np.array([1.0])}, {"w": np.array([0.0])},
                        {"w": np.array([0.0])}, h)
    assert nt["w"][0] == pytest.approx(0.99)


def test_tie_parity_two_steps():
    # test_optimizer.py:137-153: t=1 tie -> +1, t=2 tie -> -1
    h = O.Hyper(0.9, 0.99, 0.5, 0.0)
    th = [{"w": np.zeros(1)}, {"w": np.zeros(1)}]
    m = [{"w": np.zeros(1)}, {"w": np.zeros(1)}]
    g = [{"w": np.array([1.0])}, {"w": np.array([-1.0])}]
    th, m, *_ = O.distributed_step(th, m, g, h, O.Spec(1), "compressed1bit", 0)
    assert th[0]["w"].tolist() == [-0.5]
    th, m, *_ = O.distributed_step(th, m, g, h, O.Spec(1), "compressed1bit", 1)
    assert th[0]["w"].tolist() == [0.0]


def test_pairwise_sum_is_numpy_order():
    rng = np.random.default_rng(0)
    for n in (1, 7, 8, 9, 127, 128, 129, 1000, 4099, 20000):
        x = np.abs(rng.standard_cauchy(size=n)) * 10.0 ** rng.integers(-6, 6, size=n)
        assert O.pairwise_sum(x) == float(np.sum(x))


def test_mean_within_two_ulp_of_fsum():
    # test_collectives.py:210-224
    rng = np.random.default_rng(1)
    vecs = [rng.normal(size=200) for _ in range(3)]
    got = O.mean_f32(vecs).astype(np.float64)
    oracle = O.fsum_mean(vecs)
    ulp = np.spacing(np.abs(oracle).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(got - oracle) <= 2 * ulp)


# ---- golden vectors produced by running the reference ----------------------

@pytest.mark.parametrize("name", [c["name"] for c in G.step_cases()])
def test_oracle_matches_reference_step(name):
    gc = G.step_case(name)
    case = gc["case"]
    world = case["world"]
    h = O.Hyper(0.9, 0.99, case["lr"], case["wd"])
    kw = quant_kwargs(case)
    spec = None if kw is None else O.Spec(**kw)
    thetas = [dict(gc["theta"]) for _ in range(world)]
    nt, nm, sign, ties, cs, _ = O.distributed_step(
        thetas, gc["m"], gc["g"], h, spec, case["algo"], case["iteration"],
        zero_mode=case["zero_mode"], masks=gc["mask"])
    if case.get("sync"):
        period, layers = case["sync"]
        nm = O.sync_momentum(nm, period, layers, case["iteration"] + 1)
    t = case["iteration"] + 1
    for k in gc["sizes"]:
        assert np.array_equal(nt[0][k], gc["theta_out"][k]), k
        assert np.array_equal(sign[k], gc["sign"][k]), k
        assert ties[k] == gc["ties"][k], k
        for r in range(world):
            assert np.array_equal(nm[r][k], gc["m_out"][r][k]), (k, r)
            if gc["c"][r][k] is not None:
                assert np.array_equal(cs[r][k], gc["c"][r][k])
            if gc["words"][r][k] is not None:
                s = O.apply_sign(cs[r][k], case["zero_mode"], t)
                assert np.array_equal(O.pack_signs(s), gc["words"][r][k])
            if gc["q"][r][k] is not None:
                assert np.array_equal(O.quantize(cs[r][k], spec),
                                      gc["q"][r][k].astype(np.int64))
                assert O.lp_mean_norm(cs[r][k], spec.norm_p) == float(gc["norm"][r][k])
                if spec.norm_p == 1.0 and not spec.log_transform and not spec.no_zero:
                    assert np.array_equal(O.quantize_l1(cs[r][k], case["bits"]),
                                          gc["q"][r][k].astype(np.int64))
                    assert O.lp_mean_norm_l1(cs[r][k]) == float(gc["norm"][r][k])


@pytest.mark.parametrize("name", [c["name"] for c in G.collective_cases()])
def test_oracle_matches_reference_collective(name):
    gc = G.collective_case(name)
    case = gc["case"]
    if case["kind"] == "direct":
        v = O.direct_sum(gc["inputs"], case["q_max"], case.get("binary", False))
        assert np.array_equal(v.values, gc["values"])
        assert v.ties == gc["ties"]
    elif case["kind"] == "compressed":
        v = O.vote_1bit(gc["inputs"], "alternating", case["t"])
        assert np.array_equal(v.values, gc["values"])
        assert v.ties == gc["ties"]
    else:
        assert np.array_equal(O.mean_f32(gc["inputs"]), gc["values"])


# ---- standalone quant.py functions (golden_quant.npz) ----------------------

def _quant_keys():
    _, meta = G.quant_golden()
    for kind in meta["inputs"]:
        for p in meta["ps"]:
            for bits in meta["bits"]:
                for lt in (0, 1):
                    for nz in (0, 1):
                        yield kind, p, bits, lt, nz


def test_oracle_lp_mean_norm_matches_reference():
    data, meta = G.quant_golden()
    for kind in meta["inputs"]:
        for p in meta["ps"]:
            assert O.lp_mean_norm(data[f"x/{kind}"], p) == float(data[f"norm/{kind}/{p}"]), \
                (kind, p)


def test_oracle_quantize_dequantize_match_reference():
    data, _ = G.quant_golden()
    for kind, p, bits, lt, nz in _quant_keys():
        x = data[f"x/{kind}"]
        spec = O.Spec(bits=bits, norm_p=p, log_transform=bool(lt), no_zero=bool(nz))
        key = f"{kind}/{p}/{bits}/{lt}/{nz}"
        q = O.quantize(x, spec)
        assert np.array_equal(q, data[f"q/{key}"].astype(np.int64)), key
        _, s, norm = O.quant_scale(x, spec)
        assert np.array_equal(O.dequantize(q, spec, norm, s), data[f"deq/{key}"]), key


def test_oracle_apply_sign_and_pack_match_reference():
    data, meta = G.quant_golden()
    for kind in meta["inputs"]:
        x = data[f"x/{kind}"]
        for mode, it in (("alternating", 1), ("alternating", 2), ("exact-ternary", 1)):
            assert np.array_equal(O.apply_sign(x, mode, it),
                                  data[f"sign/{kind}/{mode}/{it}"].astype(np.int64))
    for i, (w, off, *_rest) in enumerate(meta["pack"]):
        v = data[f"pack/{i}/values"]
        wire = data[f"pack/{i}/wire"].tobytes()
        stored = (v + 1) >> 1 if (w == 1 and off == 1) else v + off
        words = O.pack_words(stored, w)
        nbytes = (v.size * w + 7) // 8
        assert words.astype("<u4").tobytes()[:nbytes] == wire[9:], i
        assert wire[:9] == np.array([v.size], "<u4").tobytes() + bytes([w]) + \
            np.array([off], "<i4").tobytes()


def test_counter_stream_is_uniform_and_sround_unbiased():
    u = O.stream_uniforms(12345, np.arange(1 << 20))
    assert u.min() >= 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 2e-3 and abs(u.var() - 1 / 12) < 2e-3
    # different seeds / offsets give different streams
    assert not np.array_equal(u[:100], O.stream_uniforms(12346, np.arange(100)))
    assert np.array_equal(u[50:60], O.stream_uniforms(12345, np.arange(50, 60)))
    v = np.full(u.size, 2.3)
    q = O.sround(v, u)
    assert set(np.unique(q)) == {2, 3}
    assert abs(q.mean() - 2.3) < 2e-3          # E[sround(v)] = v (quant.py:107-116)


# ---- signSGD majority and divergence metrics (golden_metrics.npz) ----------

@pytest.mark.parametrize("i", range(len(G.metrics_golden()[1]["signsgd"])))
def test_oracle_signsgd_and_divergence_match_reference(i):
    sizes = G.step_sizes()
    c = G.signsgd_case(i, sizes)
    out = O.signsgd_step([c["theta"]] * c["world"], c["g"], 1e-3, c["algo"], c["iteration"],
                         c["zero_mode"])
    for k in sizes:
        assert np.array_equal(out[k], c["theta_out"][k]), k
    div = O.divergence(c["m"])
    for k in sizes:
        assert div[k] == c["div"][k] == c["divm"][k], k


# ---- the C restatement (oracle/lioncub_oracle.c) used for large checks -----

def _c_oracle_case_ok(case) -> bool:
    kw = quant_kwargs(case)
    if kw is None:
        return True
    extra = {k: v for k, v in kw.items() if k not in ("bits", "norm_p")}
    return kw.get("norm_p", 1.0) == 1.0 and not extra


@pytest.mark.parametrize("name", [c["name"] for c in G.step_cases() if _c_oracle_case_ok(c)])
def test_c_oracle_matches_reference_step(name):
    """The C oracle against the reference's golden step outputs: theta' and
    m' are float32 of the reference float64 values, votes and ties exact."""
    from oracle import c_oracle as CO
    gc = G.step_case(name)
    case = gc["case"]
    names = sorted(gc["sizes"])
    flat = lambda d: np.concatenate([np.asarray(d[k], np.float32).ravel() for k in names])  # noqa
    seg = np.cumsum([0] + [int(np.prod(gc["sizes"][k])) for k in names])
    mask = None
    if gc["mask"] is not None:
        mask = np.concatenate([np.asarray(gc["mask"][k]).ravel() if k in gc["mask"]
                               else np.ones(int(np.prod(gc["sizes"][k])), bool)
                               for k in names]).astype(np.uint8)
    t = case["iteration"] + 1
    fill = 0 if case["zero_mode"] == "exact-ternary" else O.zero_fill(t)
    th, ms, sign, ties = CO.step(flat(gc["theta"]), [flat(x) for x in gc["m"]],
                                 [flat(x) for x in gc["g"]], seg,
                                 CO.hyper(0.9, 0.99, case["lr"], case["wd"]),
                                 CO.algo_name(case["algo"], case["bits"]), fill,
                                 bits=case["bits"] or 0, mask=mask)
    if case.get("sync"):
        return  # the sync is not part of the C oracle
    ref_t = np.concatenate([np.asarray(gc["theta_out"][k]).ravel() for k in names])
    assert np.array_equal(th, ref_t.astype(np.float32))
    for r in range(case["world"]):
        ref_m = np.concatenate([np.asarray(gc["m_out"][r][k]).ravel() for k in names])
        assert np.array_equal(ms[r], ref_m.astype(np.float32)), r
    ref_s = np.concatenate([gc["sign"][k].ravel() for k in names])
    assert np.array_equal(sign.astype(np.int64), ref_s)
    assert [int(x) for x in ties] == [gc["ties"][k] for k in names]


@pytest.mark.parametrize("n", [1, 7, 8, 127, 128, 129, 1000, 65_537, 1_000_003, 38_597_376])
def test_c_oracle_pairwise_sum_is_numpy_order(n):
    """numpy's pairwise order, up to the GPT-2 embedding's 38.6M elements
    (the np.mean inside lp_mean_norm, quant.py:104)."""
    from oracle import c_oracle as CO
    x = np.random.default_rng(n).random(n) * 1e-3
    assert CO.pairwise_sum(x) == float(np.add.reduce(x))


@pytest.mark.parametrize("algo,bits,world,kind,zm", [
    ("compressed1bit", None, 8, "ties", "alternating"),
    ("direct", 1, 8, "laplace", "alternating"),
    ("direct", 5, 8, "outliers", "alternating"),
    ("direct", 8, 3, "laplace", "exact-ternary"),
    ("ps_efficient", None, 5, "cancel", "exact-ternary"),
])
def test_c_oracle_matches_numpy_oracle_600k(algo, bits, world, kind, zm):
    from oracle import c_oracle as CO
    sizes = {"emb": (40_000,), "h0.w": (300_017,), "h1.w": (262_144,), "norm": (1_000,)}
    names = sorted(sizes)
    ranks = O.synth_rank_inputs(7, world, sizes, kind)
    h = O.Hyper(0.9, 0.99, 1e-4, 0.1)
    spec = None if bits is None else O.Spec(bits)
    nt, nm, sign, ties, _, _ = O.distributed_step(
        [rk["theta"] for rk in ranks], [rk["m"] for rk in ranks], [rk["g"] for rk in ranks],
        h, spec, algo, 2, zero_mode=zm)
    flat = lambda d: np.concatenate([np.asarray(d[k]).ravel() for k in names])  # noqa
    seg = np.cumsum([0] + [sizes[k][0] for k in names])
    fill = 0 if zm == "exact-ternary" else O.zero_fill(3)
    th, ms, sg, tc = CO.step(flat(ranks[0]["theta"]), [flat(rk["m"]) for rk in ranks],
                             [flat(rk["g"]) for rk in ranks], seg, CO.hyper(lr=1e-4, wd=0.1),
                             CO.algo_name(algo, bits), fill, bits=bits or 0)
    assert np.array_equal(th, flat(nt[0]).astype(np.float32))
    for r in range(world):
        assert np.array_equal(ms[r], flat(nm[r]).astype(np.float32))
    assert np.array_equal(sg.astype(np.int64), flat(sign))
    assert [int(x) for x in tc] == [ties[k] for k in names]
