"""Parity at BASELINE.json's sizes and layouts.

* GPT-2-small, 148 tensors, 124,439,808 params (configs[1]): the FULL vector
  at P = 1 and at P = 8 simulated ranks on the production peer-memory path
  (LocalTransport(fused=True): in-kernel barriers, k_vote_apply), against the
  C oracle (oracle/lioncub_oracle.c, itself pinned to the reference's golden
  vectors): sum-of-signs, L1 5-bit (the paper's 8-bit Lion Cub), 1-bit.
* TinyLlama-1.1B, 201 tensors, 1,100,048,384 params (configs[3], the north
  star), P = 8 simulated: layer windows against the C oracle (theta', m',
  the embed/head momentum sync) plus full-vector invariants: every rank's
  theta identical, the synced layers' momentum identical, and on iid +-1
  gradients the exact-ternary tie rate C(8,4)/2^8 = 0.2734375.
* The 7e9 flat buffer (configs[4]) at P = 1, and a 2^32 + 5000-element
  buffer at P = 2 simulated ranks: windows at and past the 2^31 / 2^32
  element boundaries (64-bit index paths), plus the full-vector invariant
  that every parameter moved.

Inputs are generated on the device (seeded, fp32, Laplace-correlated
workers -- the runner.py:289-297 recipe -- or iid +-1 "ties"); only the
parts the oracle needs are copied to the host.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from oracle import c_oracle as CO
from oracle import lioncub_oracle as O

pytestmark = pytest.mark.gpu

lc = pytest.importorskip("paper_2411_16462_b200")
from paper_2411_16462_b200 import _lib  # noqa: E402
from paper_2411_16462_b200.transport import host_wait  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _lib.load()
    CO.load()


@pytest.fixture(autouse=True)
def _free_memory():
    yield
    import gc
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def gpt2_small_layout() -> dict:
    d, L, V, T = 768, 12, 50257, 1024
    shapes = {"wte.weight": (V, d), "wpe.weight": (T, d), "ln_f.weight": (d,), "ln_f.bias": (d,)}
    for i in range(L):
        p = f"h.{i}."
        shapes.update({p + "ln_1.weight": (d,), p + "ln_1.bias": (d,),
                       p + "attn.c_attn.weight": (d, 3 * d), p + "attn.c_attn.bias": (3 * d,),
                       p + "attn.c_proj.weight": (d, d), p + "attn.c_proj.bias": (d,),
                       p + "ln_2.weight": (d,), p + "ln_2.bias": (d,),
                       p + "mlp.c_fc.weight": (d, 4 * d), p + "mlp.c_fc.bias": (4 * d,),
                       p + "mlp.c_proj.weight": (4 * d, d), p + "mlp.c_proj.bias": (d,)})
    return shapes


def tinyllama_layout() -> dict:
    d, ff, kv, L, V = 2048, 5632, 256, 22, 32000
    shapes = {"model.embed_tokens.weight": (V, d), "model.norm.weight": (d,),
              "lm_head.weight": (V, d)}
    for i in range(L):
        p = f"model.layers.{i}."
        shapes.update({p + "self_attn.q_proj.weight": (d, d),
                       p + "self_attn.k_proj.weight": (kv, d),
                       p + "self_attn.v_proj.weight": (kv, d),
                       p + "self_attn.o_proj.weight": (d, d),
                       p + "mlp.gate_proj.weight": (ff, d), p + "mlp.up_proj.weight": (ff, d),
                       p + "mlp.down_proj.weight": (d, ff),
                       p + "input_layernorm.weight": (d,),
                       p + "post_attention_layernorm.weight": (d,)})
    return shapes


CH = 1 << 26


def _laplace(out, gen):
    out.exponential_(generator=gen)
    out.mul_(torch.where(torch.rand(out.shape, generator=gen, device=out.device) < 0.5, -1.0, 1.0))


def synth(n: int, world: int, kind: str, seed: int):
    """theta (shared) and per-rank m, g as flat fp32 CUDA tensors."""
    dev = torch.device("cuda")
    theta = torch.empty(n, dtype=torch.float32, device=dev)
    ms = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(world)]
    gs = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(world)]
    gen = torch.Generator(device=dev)
    for ci, a in enumerate(range(0, n, CH)):
        b = min(n, a + CH)
        gen.manual_seed(seed * 1_000_003 + 2 * ci)
        theta[a:b].normal_(generator=gen)
        base = torch.empty(b - a, dtype=torch.float32, device=dev)
        _laplace(base, gen)
        for r in range(world):
            gen.manual_seed(seed * 1_000_003 + 7919 * (r + 1) + 2 * ci + 1)
            if kind == "ties":
                gs[r][a:b].copy_(torch.where(torch.rand(b - a, generator=gen, device=dev) < 0.5,
                                             -1.0, 1.0))
                ms[r][a:b].zero_()
            else:
                _laplace(gs[r][a:b], gen)
                gs[r][a:b].add_(base)
                ms[r][a:b].normal_(generator=gen).mul_(0.1)
        del base
    torch.cuda.synchronize()
    return theta, ms, gs


def run_simulated(world, layout, theta, ms, gs, h, spec, algo, zero_mode="alternating",
                  iteration=0, sync=None):
    """One step on ``world`` simulated ranks of the production fused path
    (one rank: the P = 1 fused kernel).  The inputs are DONATED: ms[r]
    becomes rank r's momentum, a clone of theta its parameters.  Returns the
    per-rank final states (device)."""
    tp = lc.LocalTransport(world, fused=world > 1)
    thetas = [theta.clone() for _ in range(world - 1)] + [theta]

    def fn(topo):
        r = topo.rank
        st = lc.WorkerState(params=layout.views(thetas[r]), momentum=layout.views(ms[r]),
                            iteration=iteration)
        st = lc.distributed_lion_step(st, layout.views(gs[r]), h, spec, topo, algo,
                                      zero_mode=zero_mode)
        if sync is not None:
            st = lc.maybe_sync_momentum(st, sync, topo)
        host_wait()
        return st

    out = lc.run_ranks(world, fn, transport=tp)
    return out, tp


def _host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


# ---- GPT-2-small: full vector ------------------------------------------------

@pytest.mark.parametrize("world,algo,bits,kind", [
    (1, "direct", 1, "laplace"),
    (1, "direct", 5, "laplace"),
    (8, "direct", 1, "laplace"),
    (8, "direct", 5, "laplace"),
    (8, "compressed1bit", None, "ties"),
])
def test_gpt2_layout_full_vector_matches_c_oracle(world, algo, bits, kind):
    layout = lc.Layout(gpt2_small_layout())
    n = layout.n
    assert n == 124_439_808 and len(layout.names) == 148
    theta, ms, gs = synth(n, world, kind, seed=11 + world)
    th_h, m_h, g_h = _host(theta), [_host(m) for m in ms], [_host(g) for g in gs]
    it = 4
    fill = O.zero_fill(it + 1)
    lr, wd = 1e-3, 0.1
    ref_t, ref_m, ref_s, ref_ties = CO.step(th_h, m_h, g_h, np.asarray(layout.seg_start),
                                            CO.hyper(lr=lr, wd=wd), CO.algo_name(algo, bits),
                                            fill, bits=bits or 0)
    spec = None if bits is None else lc.QuantSpec(bits=bits, norm_p=1.0)
    out, tp = run_simulated(world, layout, theta, ms, gs, lc.LionHyper(lr=lr, weight_decay=wd),
                            spec, algo, iteration=it)
    for r, st in enumerate(out):
        got_t = _host(st.params.flat[:n])
        bad = np.flatnonzero(got_t.view(np.int32) != ref_t.view(np.int32))
        assert bad.size == 0, f"rank {r}: {bad.size} theta mismatches, first at {bad[:5]}"
        assert np.array_equal(_host(st.momentum.flat[:n]).view(np.int32), ref_m[r].view(np.int32))
    if kind == "ties" and world == 8:   # iid +-1 votes: ties at C(8,4)/2^8
        rate = ref_ties.sum() / n
        assert abs(rate - 70 / 256) < 1e-3


# ---- TinyLlama-1.1B (the north star), P = 8: windows + invariants ------------

def _windows(layout, n, P, extra=(), w=4096, seed=0):
    rng = np.random.default_rng(seed)
    starts = {0, max(0, n - w)}
    L = -(-(-(-n // P)) // 1024) * 1024
    for j in range(1, P):
        starts.add(max(0, min(n - w, j * L - w // 2)))   # owner-block boundaries
    for k in rng.choice(len(layout.names), size=min(24, len(layout.names)), replace=False):
        o = layout.offset[layout.names[k]]
        starts.add(max(0, min(n - w, o - w // 2)))       # layer boundaries
    for e in extra:
        if 0 <= e < n:
            starts.add(max(0, min(n - w, e - w // 2)))
    return sorted(starts)


def _gather_windows(starts, w, theta, ms, gs):
    take = lambda t: np.concatenate([_host(t[a:a + w]) for a in starts])  # noqa: E731
    return take(theta), [take(m) for m in ms], [take(g) for g in gs]


@pytest.mark.parametrize("algo,bits,zm,kind", [
    ("compressed1bit", None, "alternating", "laplace"),
    ("direct", 1, "exact-ternary", "ties"),
])
def test_tinyllama_layout_p8_windows_and_invariants(algo, bits, zm, kind):
    P = 8
    layout = lc.Layout(tinyllama_layout())
    n = layout.n
    assert n == 1_100_048_384 and len(layout.names) == 201
    theta, ms, gs = synth(n, P, kind, seed=21)
    w = 4096
    starts = _windows(layout, n, P)
    th_w, m_w, g_w = _gather_windows(starts, w, theta, ms, gs)
    theta0 = theta.clone() if kind == "ties" else None
    it = 9                                              # t = 10: the sync fires
    lr = 1e-3
    sel = ("model.embed_tokens.weight", "lm_head.weight")
    sync = lc.SyncPolicy(period=10, layers=frozenset(sel)) if algo == "compressed1bit" else None
    fill = 0 if zm == "exact-ternary" else O.zero_fill(it + 1)
    seg = np.arange(len(starts) + 1, dtype=np.int64) * w
    ref_t, ref_m, _, _ = CO.step(th_w, m_w, g_w, seg, CO.hyper(lr=lr), CO.algo_name(algo, bits),
                                 fill, bits=bits or 0)
    if sync is not None:   # maybe_sync_momentum: rank-ordered f64 mean of the fp32 m'
        mean = O.mean_f32(ref_m)
        for i, a in enumerate(starts):
            for k in sel:
                lo, hi = layout.offset[k], layout.offset[k] + layout.numel[k]
                s0, s1 = max(a, lo), min(a + w, hi)
                if s0 < s1:
                    for r in range(P):
                        ref_m[r][i * w + s0 - a:i * w + s1 - a] = mean[i * w + s0 - a:
                                                                      i * w + s1 - a]
    spec = None if bits is None else lc.QuantSpec(bits=bits)
    out, tp = run_simulated(P, layout, theta, ms, gs, lc.LionHyper(lr=lr), spec, algo,
                            zero_mode=zm, iteration=it, sync=sync)
    t0 = out[0].params.flat
    for r, st in enumerate(out):
        got_t = np.concatenate([_host(st.params.flat[a:a + w]) for a in starts])
        got_m = np.concatenate([_host(st.momentum.flat[a:a + w]) for a in starts])
        assert np.array_equal(got_t.view(np.int32), ref_t.view(np.int32)), f"theta r{r}"
        assert np.array_equal(got_m.view(np.int32), ref_m[r].view(np.int32)), f"m r{r}"
        if r:   # full vector: every replica took the same step
            assert torch.equal(st.params.flat[:n].view(torch.int32), t0[:n].view(torch.int32))
    if sync is not None:
        for k in sel:
            a, b = layout.offset[k], layout.offset[k] + layout.numel[k]
            for st in out[1:]:
                assert torch.equal(st.momentum.flat[a:b], out[0].momentum.flat[a:b])
    if kind == "ties":
        # exact-ternary sum of 8 iid +-1 signs: zero with probability 70/256,
        # and a zero vote leaves theta unchanged (wd = 0)
        same = int((out[0].params.flat[:n] == theta0[:n]).sum())
        assert abs(same / n - 70 / 256) < 1e-3, same / n


# ---- 7e9 flat at P = 1; 2^32 + 5000 at P = 2 ---------------------------------

@pytest.mark.parametrize("world,n", [(1, 7_000_000_000), (2, (1 << 32) + 5000)])
def test_flat_buffer_past_2_32_elements(world, n):
    layout = lc.Layout({"w": (n,)})
    theta, ms, gs = synth(n, world, "laplace", seed=31)
    w = 4096
    starts = _windows(layout, n, world, extra=(1 << 31, 1 << 32, (1 << 32) + 3000, 5_000_000_000))
    th_w, m_w, g_w = _gather_windows(starts, w, theta, ms, gs)
    it, lr = 2, 1e-3
    seg = np.arange(len(starts) + 1, dtype=np.int64) * w
    ref_t, ref_m, _, _ = CO.step(th_w, m_w, g_w, seg, CO.hyper(lr=lr), "compressed1bit",
                                 O.zero_fill(it + 1))
    theta0 = theta[:1 << 20].clone()
    out, tp = run_simulated(world, layout, theta, ms, gs, lc.LionHyper(lr=lr), None,
                            "compressed1bit", iteration=it)
    for r, st in enumerate(out):
        got_t = np.concatenate([_host(st.params.flat[a:a + w]) for a in starts])
        got_m = np.concatenate([_host(st.momentum.flat[a:a + w]) for a in starts])
        assert np.array_equal(got_t.view(np.int32), ref_t.view(np.int32)), f"theta r{r}"
        assert np.array_equal(got_m.view(np.int32), ref_m[r].view(np.int32)), f"m r{r}"
    # every parameter moved by +-lr (|theta| ~ N(0,1): lr >> ulp), checked on
    # the first 2^20 elements against their copy
    moved = (out[0].params.flat[:1 << 20] != theta0)
    assert bool(moved.all())
    if world > 1:
        assert torch.equal(out[0].params.flat[:n].view(torch.int32),
                           out[1].params.flat[:n].view(torch.int32))
    assert math.isfinite(float(out[0].params.flat[n - 1]))


def test_flat_600m_p4_fused_momentum_sync():
    """The momentum sync fused into the step (SyncPolicy(1, "all") passed to
    distributed_lion_step on the production exchange) at 600M params, P = 4:
    windows of theta' / m' against the C oracle + the f64 rank-ordered mean,
    and every rank's full momentum identical afterwards."""
    P, n = 4, 600_000_037
    layout = lc.Layout({"w": (n,)})
    theta, ms, gs = synth(n, P, "laplace", seed=41)
    w = 4096
    starts = _windows(layout, n, P, extra=(n // 3, n // 2))
    th_w, m_w, g_w = _gather_windows(starts, w, theta, ms, gs)
    it, lr = 6, 1e-3
    seg = np.arange(len(starts) + 1, dtype=np.int64) * w
    ref_t, ref_m, _, _ = CO.step(th_w, m_w, g_w, seg, CO.hyper(lr=lr), "compressed1bit",
                                 O.zero_fill(it + 1))
    mean = O.mean_f32(ref_m)
    tp = lc.LocalTransport(P, fused=True)
    thetas = [theta.clone() for _ in range(P - 1)] + [theta]
    policy = lc.SyncPolicy(period=1, layers="all")

    def fn(topo):
        r = topo.rank
        st = lc.WorkerState(params=layout.views(thetas[r]), momentum=layout.views(ms[r]),
                            iteration=it)
        st = lc.distributed_lion_step(st, layout.views(gs[r]), lc.LionHyper(lr=lr), None, topo,
                                      "compressed1bit", sync=policy)
        assert getattr(st, "_lc_synced", None) == it + 1   # fused, not a separate pass
        st = lc.maybe_sync_momentum(st, policy, topo)      # no-op for this iteration
        host_wait()
        return st

    out = lc.run_ranks(P, fn, transport=tp)
    m0 = out[0].momentum.flat
    for r, st in enumerate(out):
        got_t = np.concatenate([_host(st.params.flat[a:a + w]) for a in starts])
        got_m = np.concatenate([_host(st.momentum.flat[a:a + w]) for a in starts])
        assert np.array_equal(got_t.view(np.int32), ref_t.view(np.int32)), f"theta r{r}"
        assert np.array_equal(got_m.view(np.int32), mean.view(np.int32)), f"m r{r}"
        if r:
            assert torch.equal(st.momentum.flat[:n].view(torch.int32), m0[:n].view(torch.int32))
            assert torch.equal(st.params.flat[:n].view(torch.int32),
                               out[0].params.flat[:n].view(torch.int32))
