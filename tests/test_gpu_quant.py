"""Standalone quant operators on the GPU (quant.py:81-300) against the
reference's own outputs (tests/golden/golden_quant.npz) and the oracle.

Tolerances: quantized ints, signs, packed bytes and unpacked values are
bit-exact.  lp_mean_norm is bit-exact for p in {1, 2, 0.5, inf} (numpy's
fast paths: copy, square, sqrt, max); for other p and p = 0 numpy's SIMD
pow/log and CUDA's differ by ulps -> 1e-13 relative.  dequantize is exact
without the log map; with it, CUDA expm1 vs libm expm1 -> 4e-16 relative.
"""

import numpy as np
import pytest
import torch

from oracle import lioncub_oracle as O
from tests import golden_io as G

pytestmark = pytest.mark.gpu

lc = pytest.importorskip("paper_2411_16462_b200")
from paper_2411_16462_b200 import _lib  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _lib.load()


def _x(data, kind):
    return torch.from_numpy(data[f"x/{kind}"]).cuda()   # float64, fp32-representable


def test_lp_mean_norm_matches_reference():
    data, meta = G.quant_golden()
    for kind in meta["inputs"]:
        x = _x(data, kind)
        for p in meta["ps"]:
            ref = float(data[f"norm/{kind}/{p}"])
            got = lc.lp_mean_norm(x, p)
            if p in (1.0, 2.0, 0.5, float("inf")):
                assert got == ref, (kind, p, got, ref)
            else:
                assert abs(got - ref) <= 1e-13 * abs(ref), (kind, p, got, ref)


def test_quantize_and_dequantize_match_reference():
    data, meta = G.quant_golden()
    for kind in meta["inputs"]:
        x = _x(data, kind)
        xf = x.float()
        for p in meta["ps"]:
            for bits in meta["bits"]:
                for lt in (0, 1):
                    for nz in (0, 1):
                        key = f"{kind}/{p}/{bits}/{lt}/{nz}"
                        spec = lc.QuantSpec(bits=bits, norm_p=p, log_transform=bool(lt),
                                            no_zero=bool(nz))
                        ref_q = data[f"q/{key}"].astype(np.int64)
                        q = lc.quantize(x, spec)
                        assert q.dtype == torch.int64 and q.shape == x.shape
                        assert np.array_equal(q.cpu().numpy(), ref_q), key
                        assert torch.equal(lc.quantize(xf, spec), q), key
                        ospec = O.Spec(bits=bits, norm_p=p, log_transform=bool(lt),
                                       no_zero=bool(nz))
                        _, s, norm = O.quant_scale(data[f"x/{kind}"], ospec)
                        d = lc.dequantize(q, spec, norm, s).cpu().numpy()
                        ref_d = data[f"deq/{key}"]
                        if lt:
                            assert np.allclose(d, ref_d, rtol=4e-16, atol=0), key
                        else:
                            assert np.array_equal(d, ref_d), key


def test_apply_sign_matches_reference():
    data, meta = G.quant_golden()
    for kind in meta["inputs"]:
        x = _x(data, kind)
        for mode, it in (("alternating", 1), ("alternating", 2), ("exact-ternary", 1)):
            ref = data[f"sign/{kind}/{mode}/{it}"]
            pol = lc.SignPolicy(mode=mode, iteration=it)
            assert np.array_equal(lc.apply_sign(x, pol).cpu().numpy(), ref), (kind, mode, it)
            assert np.array_equal(lc.apply_sign(x.float(), pol).cpu().numpy(), ref)


def test_pack_unpack_wire_bytes_match_reference():
    data, meta = G.quant_golden()
    for i, (w, off, *_r) in enumerate(meta["pack"]):
        v = torch.from_numpy(data[f"pack/{i}/values"]).cuda()
        wire = data[f"pack/{i}/wire"].tobytes()
        pk = lc.pack(v, w, off)
        assert pk.to_bytes() == wire, i
        assert torch.equal(lc.unpack(pk), v), i
        back = lc.PackedBits.from_bytes(wire)
        assert back == pk
        assert torch.equal(lc.unpack(back), v)


def test_pack_errors_match_reference():
    v = torch.tensor([1, -1, 1, 1, 1, 0, 1, 3], device="cuda")
    with pytest.raises(lc.PackRangeError) as ei:
        lc.pack(v, 1, 1)                      # sign map: 0 at index 5
    assert (ei.value.index, ei.value.value, ei.value.width) == (5, 0, 1)
    with pytest.raises(lc.PackRangeError) as ei:
        lc.pack(torch.tensor([0, 3, 4, -1], device="cuda"), 2)
    assert (ei.value.index, ei.value.value) == (2, 4)
    with pytest.raises(lc.ConfigError):
        lc.pack(v, 3)
    pk = lc.pack(torch.tensor([3, 12], device="cuda"), 4)
    assert pk.payload.cpu().numpy().tolist() == [0xC3]        # test_quant.py:164-166
    with pytest.raises(lc.PackFormatError):
        lc.PackedBits.from_bytes(pk.to_bytes()[:-1])
    with pytest.raises(lc.PackFormatError):
        lc.PackedBits.from_bytes(b"\x01\x00")


def test_operators_reject_cpu_and_inexact_inputs():
    with pytest.raises(lc.ConfigError):
        lc.quantize(torch.ones(4), lc.QuantSpec())
    with pytest.raises(lc.ConfigError, match="float32"):
        lc.lp_mean_norm(torch.tensor([0.1, 0.2], dtype=torch.float64, device="cuda"), 1.0)
    with pytest.raises(lc.ConfigError, match="empty"):
        lc.quantize(torch.zeros(0, device="cuda"), lc.QuantSpec())
    with pytest.raises(lc.ConfigError, match="norm order"):
        lc.lp_mean_norm(torch.ones(3, device="cuda"), -1.0)


@pytest.mark.parametrize("p", [1.0, float("inf"), 2.0])
def test_stochastic_quantize_matches_oracle_stream(p):
    rng = np.random.default_rng(5)
    x = rng.laplace(size=200_003).astype(np.float32)
    spec = lc.QuantSpec(bits=4, norm_p=p, rounding="stochastic")
    seed = lc.QuantSpec(rounding="stochastic").draw_seed(np.random.default_rng(17))
    q = lc.quantize(torch.from_numpy(x).cuda(), spec, rng=np.random.default_rng(17))
    u = O.stream_uniforms(seed, np.arange(x.size))
    ref = O.quantize(x.astype(np.float64), O.Spec(bits=4, norm_p=p, rounding="stochastic"), u)
    assert np.array_equal(q.cpu().numpy(), ref)
    with pytest.raises(lc.ConfigError, match="rng"):
        lc.quantize(torch.from_numpy(x).cuda(), spec)
    # the reference returns zeros without an rng when the norm is 0
    assert not lc.quantize(torch.zeros(5, device="cuda"), spec).any()


def test_quantize_large_matches_oracle():
    rng = np.random.default_rng(8)
    x = (rng.standard_normal(3_000_017) * 0.01).astype(np.float32)
    x[::1001] = 0.0
    for kw in (dict(bits=5), dict(bits=8, norm_p=float("inf"), no_zero=True),
               dict(bits=5, norm_p=2.0, log_transform=True)):
        q = lc.quantize(torch.from_numpy(x).cuda(), lc.QuantSpec(**kw)).cpu().numpy()
        assert np.array_equal(q, O.quantize(x.astype(np.float64), O.Spec(**kw))), kw


@pytest.mark.parametrize("p", [1.0, 2.0, 0.5])
def test_norm_extreme_magnitudes_bit_exact(p):
    """fp32 denormals next to values near FLT_MAX in one layer: the
    reciprocal division's no-guard argument (csrc/l1norm.cu term_div) must
    hold -- every quotient normal, every term correctly rounded."""
    rng = np.random.default_rng(11)
    n = 70_001
    x = rng.standard_normal(n).astype(np.float32)
    x[::7] = np.float32(1.4e-45) * rng.integers(1, 100, size=x[::7].size).astype(np.float32)
    x[::11] *= np.float32(1e30)
    x[5] = np.float32(3.0e38)
    x[9] = np.float32(-1.4e-45)
    x64 = x.astype(np.float64)
    xt = torch.from_numpy(x).cuda()
    assert lc.lp_mean_norm(xt, p) == O.lp_mean_norm(x64, p)
    spec = lc.QuantSpec(bits=8, norm_p=p)
    assert np.array_equal(lc.quantize(xt, spec).cpu().numpy(),
                          O.quantize(x64, O.Spec(bits=8, norm_p=p)))
