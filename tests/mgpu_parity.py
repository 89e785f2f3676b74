"""Multi-GPU parity over NCCL (one process per GPU), checked against the CPU
oracle.  Launched by tests/test_multigpu.py:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/mgpu_parity.py

Every rank builds the same seeded inputs for all P ranks, runs ITS step
through the public API over an NcclTransport, and compares its outputs with
the oracle's P-rank result (theta'/m' bit-exact to float32 of the reference,
votes/ties exact).  Rank 0 prints a JSON summary; the exit code is non-zero
on any mismatch.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2411_16462_b200 as lc  # noqa: E402
from oracle import lioncub_oracle as O  # noqa: E402
from tests import golden_io as G  # noqa: E402

SIZES = {"emb": (50_000,), "h0.w": (300_017,), "h1.w": (262_144,), "norm": (7,)}

INF = float("inf")
CONFIGS = [  # (algo, QuantSpec kwargs or None, input kind, zero mode, sync)
    ("compressed1bit", None, "laplace", "alternating", None),
    ("compressed1bit", None, "ties", "alternating", None),
    ("direct", dict(bits=1), "laplace", "alternating", None),
    ("direct", dict(bits=1), "ties", "exact-ternary", None),
    ("direct", dict(bits=5), "outliers", "alternating", None),
    ("direct", dict(bits=8), "laplace", "exact-ternary", None),
    ("ps", None, "cancel", "exact-ternary", None),
    ("ps_efficient", None, "laplace", "alternating", None),
    ("compressed1bit", None, "laplace", "alternating", (10, frozenset({"emb", "h1.w"}))),
    ("direct", dict(bits=1), "zeros", "alternating", (10, "all")),
    # sync of every layer every other step: fused into the step on NVLink
    ("compressed1bit", None, "laplace", "alternating", (2, "all")),
    ("direct", dict(bits=1), "laplace", "alternating", (1, "all")),
    # quantizer variants (stochastic: the oracle is fed the same stream)
    ("direct", dict(bits=5, norm_p=INF), "outliers", "alternating", None),
    ("direct", dict(bits=4, rounding="stochastic"), "laplace", "alternating", None),
    ("direct", dict(bits=6, norm_p=2.0, log_transform=True, no_zero=True), "zeros",
     "alternating", None),
]
SEED_BASE = 1000


def step_seeds(qkw, world):
    if not qkw or qkw.get("rounding") != "stochastic":
        return None
    from paper_2411_16462_b200.quant import draw_seed
    return [draw_seed(np.random.default_rng(SEED_BASE + r)) for r in range(world)]


def rng_for(qkw, rank):
    if not qkw or qkw.get("rounding") != "stochastic":
        return None
    return np.random.default_rng(SEED_BASE + rank)


def f32_eq(a, b):
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float64).astype(np.float32)
    return np.array_equal(a.view(np.int32), b.view(np.int32))


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    tp = lc.NcclTransport.init_process(rank, world, dev)
    topo = lc.Topology(world_size=world, rank=rank, transport=tp)
    fails = []
    checked = 0
    for ci, (algo, qkw, kind, zm, sync) in enumerate(CONFIGS):
        bits = None if qkw is None else qkw["bits"]
        ranks = O.synth_rank_inputs(100 + ci, world, SIZES, kind)
        h = O.Hyper(0.9, 0.99, 1e-4, 0.1)
        it = 9
        nt, nm, sign, ties, _, _ = O.distributed_step(
            [r["theta"] for r in ranks], [r["m"] for r in ranks], [r["g"] for r in ranks],
            h, None if qkw is None else O.Spec(**qkw), algo, it, zero_mode=zm,
            seeds=step_seeds(qkw, world))
        if sync is not None:
            nm = O.sync_momentum(nm, sync[0], sync[1], it + 1)
        mine = ranks[rank]
        st = lc.WorkerState.initial({k: torch.from_numpy(v).to(dev)
                                     for k, v in mine["theta"].items()})
        for k, v in mine["m"].items():
            st.momentum[k].copy_(torch.from_numpy(v))
        st.iteration = it
        g = st.new_grad_buffer()
        for k, v in mine["g"].items():
            g[k].copy_(torch.from_numpy(v))
        met = {}
        st = lc.distributed_lion_step(st, g, lc.LionHyper(0.9, 0.99, 1e-4, 0.1),
                                      None if qkw is None else lc.QuantSpec(**qkw),
                                      topo, algo, zero_mode=zm, metrics_out=met,
                                      rng=rng_for(qkw, rank))
        if sync is not None:
            st = lc.maybe_sync_momentum(st, lc.SyncPolicy(period=sync[0], layers=sync[1]), topo)
        torch.cuda.synchronize()
        for k in SIZES:
            checked += 1
            if not f32_eq(st.params[k].cpu().numpy(), nt[rank][k]):
                fails.append(f"{algo}/{bits}/{kind}/{zm}: theta {k}")
            if not f32_eq(st.momentum[k].cpu().numpy(), nm[rank][k]):
                fails.append(f"{algo}/{bits}/{kind}/{zm}: m {k}")
            if not np.array_equal(met["vote_sign"][k].cpu().numpy(), sign[k]):
                fails.append(f"{algo}/{bits}/{kind}/{zm}: sign {k}")
            if met["ties"][k] != ties[k]:
                fails.append(f"{algo}/{bits}/{kind}/{zm}: ties {k} {met['ties'][k]} != {ties[k]}")
    # the production path (no metrics): fused in-kernel barriers / the
    # streamed step, three consecutive steps against the oracle fed the
    # fp32-rounded state each step
    f32 = lambda d: {k: np.asarray(v, np.float32).astype(np.float64) for k, v in d.items()}  # noqa
    for ci, (algo, qkw, kind, zm, sync) in enumerate(CONFIGS):
        if qkw is not None and qkw.get("rounding") == "stochastic":
            continue   # one stream per step: covered by the metrics pass above
        bits = None if qkw is None else qkw["bits"]
        ranks = O.synth_rank_inputs(300 + ci, world, SIZES, kind)
        h = O.Hyper(0.9, 0.99, 1e-4, 0.1)
        it0 = 4
        thetas = [f32(ranks[0]["theta"])] * world
        moms = [f32(r["m"]) for r in ranks]
        for i in range(3):
            nt, nm, *_ = O.distributed_step(thetas, moms, [r["g"] for r in ranks], h,
                                            None if qkw is None else O.Spec(**qkw), algo,
                                            it0 + i, zero_mode=zm)
            nm = [f32(x) for x in nm]
            if sync is not None:
                nm = O.sync_momentum(nm, sync[0], sync[1], it0 + i + 1)
            thetas, moms = [f32(x) for x in nt], [f32(x) for x in nm]
        mine = ranks[rank]
        st = lc.WorkerState.initial({k: torch.from_numpy(v).to(dev)
                                     for k, v in ranks[0]["theta"].items()})
        for k, v in mine["m"].items():
            st.momentum[k].copy_(torch.from_numpy(v))
        st.iteration = it0
        g = st.new_grad_buffer()
        for k, v in mine["g"].items():
            g[k].copy_(torch.from_numpy(v))
        policy = None if sync is None else lc.SyncPolicy(period=sync[0], layers=sync[1])
        for i in range(3):
            # sync=policy: the sync rides inside the step when it can
            st = lc.distributed_lion_step(st, g, lc.LionHyper(0.9, 0.99, 1e-4, 0.1),
                                          None if qkw is None else lc.QuantSpec(**qkw),
                                          topo, algo, zero_mode=zm, sync=policy)
        torch.cuda.synchronize()
        for k in SIZES:
            checked += 1
            if not f32_eq(st.params[k].cpu().numpy(), thetas[rank][k]):
                fails.append(f"prod {algo}/{bits}/{kind}/{zm}: theta {k}")
            if not f32_eq(st.momentum[k].cpu().numpy(), moms[rank][k]):
                fails.append(f"prod {algo}/{bits}/{kind}/{zm}: m {k}")
    # reference golden collectives at this world size
    for c in G.collective_cases():
        if c["world"] != world:
            continue
        gc = G.collective_case(c["name"])
        x = torch.from_numpy(np.asarray(gc["inputs"][rank])).to(dev)
        checked += 1
        if c["kind"] == "direct":
            v = lc.direct_allreduce(x, topo, q_max=c["q_max"], binary_signs=c.get("binary", False))
            ok = np.array_equal(v.values.cpu().numpy(), gc["values"]) and v.ties == gc["ties"]
        elif c["kind"] == "compressed":
            v = lc.compressed_allreduce_1bit(x, topo, lc.SignPolicy("alternating", c["t"]))
            ok = np.array_equal(v.values.cpu().numpy(), gc["values"]) and v.ties == gc["ties"]
        else:
            v = lc.allreduce_mean_f32(x, topo)
            ok = np.array_equal(v.cpu().numpy().view(np.int32), gc["values"].view(np.int32))
        if not ok:
            fails.append(f"golden {c['name']}")
    # signSGD majority and the divergence metric (golden_metrics.npz) at this world size
    gsizes = G.step_sizes()
    for i, case in enumerate(G.metrics_golden()[1]["signsgd"]):
        if case[1] != world:
            continue
        c = G.signsgd_case(i, gsizes)
        st = lc.WorkerState.initial({k: torch.from_numpy(v).to(dev)
                                     for k, v in c["theta"].items()})
        for k, v in c["m"][rank].items():
            st.momentum[k].copy_(torch.from_numpy(v))
        st.iteration = c["iteration"]
        g = st.new_grad_buffer()
        for k, v in c["g"][rank].items():
            g[k].copy_(torch.from_numpy(v))
        st = lc.signsgd_majority_step(st, g, lc.LionHyper(0.9, 0.99, 1e-3, 0.1), topo,
                                      algo=c["algo"], zero_mode=c["zero_mode"])
        div = lc.momentum_divergence(st, topo)
        for k in gsizes:
            checked += 1
            if not f32_eq(st.params[k].cpu().numpy(), c["theta_out"][k]):
                fails.append(f"signsgd {i}: theta {k}")
            if div[k] != c["div"][k]:
                fails.append(f"signsgd {i}: divergence {k}")
    nfail = torch.tensor([len(fails)], device=dev)
    dist.all_reduce(nfail)
    if fails:
        print(f"rank {rank} FAIL: {fails[:10]}", file=sys.stderr)
    if rank == 0:
        print(json.dumps({"world": world, "checked_per_rank": checked,
                          "failures_all_ranks": int(nfail.item())}))
    tp.close()
    dist.destroy_process_group()
    return 0 if int(nfail.item()) == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
