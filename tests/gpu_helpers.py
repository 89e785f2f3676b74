"""Shared helpers for the GPU parity tests (CUDA path vs golden / oracle)."""

from __future__ import annotations

import numpy as np
import torch
from paper_2411_16462_b200.transport import host_wait

import paper_2411_16462_b200 as lc
from paper_2411_16462_b200.optimizer import FlatParamSet
from tests.golden.cases import quant_kwargs


def cuda_params(d: dict) -> dict:
    return {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda()
            for k, v in d.items()}


def make_state(theta: dict, m: dict, iteration: int) -> lc.WorkerState:
    st = lc.WorkerState.initial(cuda_params(theta))
    for k, v in m.items():
        st.momentum[k].copy_(torch.from_numpy(np.asarray(v, dtype=np.float32)))
    st.iteration = iteration
    return st


def grads_like(st: lc.WorkerState, g: dict) -> FlatParamSet:
    buf = st.new_grad_buffer()
    for k, v in g.items():
        buf[k].copy_(torch.from_numpy(np.asarray(v, dtype=np.float32)))
    return buf


def run_step_case(case: dict, theta, ms, gs, mask=None, transport=None,
                  metrics=True, sizes=None, steps=1):
    """Run one distributed step (+ optional sync) on ``case['world']`` ranks
    through the public API; returns per-rank (theta', m', metrics) numpy.
    ``steps`` > 1 repeats the step on the device-resident state (same
    gradients), exercising workspace/epoch reuse across steps."""
    world = case["world"]
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=case["lr"], weight_decay=case["wd"])
    kw = quant_kwargs(case)
    spec = None if kw is None else lc.QuantSpec(**kw)
    rng_seed = case.get("rng_seed")
    sync = None
    if case.get("sync"):
        period, layers = case["sync"]
        sync = lc.SyncPolicy(period=period,
                             layers=layers if isinstance(layers, str) else frozenset(layers))
    fused_sync = bool(getattr(transport, "fused", False))
    cmask = None
    if mask is not None:
        cmask = {k: torch.from_numpy(np.asarray(v)).cuda() for k, v in mask.items()}

    def fn(topo):
        r = topo.rank
        st = make_state(theta, ms[r], case["iteration"])
        g = grads_like(st, gs[r])
        st2 = st
        for _ in range(steps):
            met = {} if metrics else None
            rng = None if rng_seed is None else np.random.default_rng(rng_seed + r)
            if fused_sync:
                # the production path: the sync rides inside the step when it
                # can (layers="all" on the owner-vote exchange)
                st2 = lc.distributed_lion_step(st2, g, h, spec, topo, case["algo"], mask=cmask,
                                               zero_mode=case["zero_mode"], metrics_out=met,
                                               rng=rng, sync=sync)
            else:
                st2 = lc.distributed_lion_step(st2, g, h, spec, topo, case["algo"], mask=cmask,
                                               zero_mode=case["zero_mode"], metrics_out=met,
                                               rng=rng)
            if sync is not None:
                st2 = lc.maybe_sync_momentum(st2, sync, topo)
        host_wait()
        out_t = {k: v.detach().cpu().numpy().copy() for k, v in st2.params.items()}
        out_m = {k: v.detach().cpu().numpy().copy() for k, v in st2.momentum.items()}
        out_met = None
        if met is not None:
            out_met = {
                "ties": dict(met["ties"]),
                "vote_sign": {k: v.cpu().numpy() for k, v in met["vote_sign"].items()},
                "c_local": {k: v.cpu().numpy() for k, v in met["c_local"].items()},
            }
        return out_t, out_m, out_met, st2.iteration

    return lc.run_ranks(world, fn, transport=transport)


# Exchange modes of the simulated multi-rank tests (P ranks on one GPU):
#   peer-memory -- kernels store into the peers' buffers, host rendezvous
#                  between phases (one shared stream);
#   collectives -- the NCCL-path structure (all-to-all / reduce-scatter /
#                  allgather) as device copies;
#   fused       -- the production NVLink path: per-rank streams, in-kernel
#                  epoch barriers, k_vote_apply / k_vote_update / replicated
#                  K1 (run without metrics_out, which selects the plain vote).
EXCHANGES = ["peer-memory", "collectives", "fused"]


def make_transport(world: int, mode: str):
    return lc.LocalTransport(world, p2p=mode != "collectives", fused=mode == "fused")


def assert_f32_equal(got, ref64, what=""):
    """The CUDA state is fp32; the reference keeps float64.  The step computes
    in float64 and rounds once, so it must equal float32(reference) exactly
    (tolerance: 0 fp32 ulp)."""
    ref = np.asarray(ref64, dtype=np.float64).astype(np.float32)
    got = np.asarray(got, dtype=np.float32)
    if not np.array_equal(got.view(np.int32), ref.view(np.int32)):
        bad = np.flatnonzero(got.view(np.int32).ravel() != ref.view(np.int32).ravel())
        i = int(bad[0])
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {i}: "
                             f"got {got.ravel()[i]!r} ref {ref.ravel()[i]!r}")


def step_seeds(rng_seed: int, world: int) -> list:
    """The per-rank stochastic-rounding seeds run_step_case's steps draw."""
    from paper_2411_16462_b200.quant import draw_seed
    return [draw_seed(np.random.default_rng(rng_seed + r)) for r in range(world)]
