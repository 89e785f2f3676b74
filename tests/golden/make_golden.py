"""Generate golden vectors by running the REAL reference (``lioncomm`` at
/root/reference/pkg/src) on seeded inputs.  Run in the build container only:

    python tests/golden/make_golden.py

Writes tests/golden/golden_steps.npz and tests/golden/golden_collectives.npz.
The reference is imported read-only (no bytecode written); nothing here runs
on the GPU box.  Inputs are fp32-representable (generated as float32, then
upcast to float64 for the reference), so the CUDA path, which keeps fp32
state and computes in fp64, can be compared bit-for-bit with float32 of the
reference's float64 outputs.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from lioncomm.collectives import (allreduce_mean_f32,  # noqa: E402
                                  compressed_allreduce_1bit, direct_allreduce,
                                  run_ranks)
from lioncomm.optimizer import (LionHyper, SyncPolicy, WorkerState,  # noqa: E402
                                distributed_lion_step, divergence_from_momenta,
                                maybe_sync_momentum, momentum_divergence,
                                save_checkpoint, signsgd_majority_step)
from lioncomm.quant import (PackedBits, QuantSpec, SignPolicy,  # noqa: E402
                            apply_sign, dequantize, lp_mean_norm, pack,
                            quantize, unpack)
from lioncomm.transport import InprocTransport  # noqa: E402

from tests.golden.cases import (COLLECTIVE_CASES, SIZES, STEP_CASES,  # noqa: E402
                                quant_kwargs)
from oracle.lioncub_oracle import synth_rank_inputs  # noqa: E402


def sign_words(s: np.ndarray) -> np.ndarray:
    """pack(s,1,1).payload as little-endian uint32 (zero-padded to 4 B)."""
    payload = pack(s.ravel(), 1, 1).payload
    buf = payload + b"\x00" * ((-len(payload)) % 4)
    return np.frombuffer(buf, dtype="<u4").copy()


def run_step_case(case: dict, out: dict):
    name = case["name"]
    world = case["world"]
    ranks = synth_rank_inputs(case["seed"], world, SIZES, case["kind"])
    h = LionHyper(beta1=0.9, beta2=0.99, lr=case["lr"],
                  weight_decay=case["wd"])
    kw = quant_kwargs(case)
    spec = None if kw is None else QuantSpec(**kw)
    mask = None
    if case.get("mask"):
        mrng = np.random.default_rng(case["seed"] + 77)
        mask = {case["mask"]: mrng.random(size=SIZES[case["mask"]]) < 0.8}
    sync = None
    if case.get("sync"):
        period, layers = case["sync"]
        sync = SyncPolicy(period=period,
                          layers=layers if isinstance(layers, str) else frozenset(layers))
    t = case["iteration"] + 1
    policy = SignPolicy(mode=case["zero_mode"], iteration=t)

    def fn(topo):
        r = topo.rank
        st = WorkerState(
            params={k: v.astype(np.float64) for k, v in ranks[r]["theta"].items()},
            momentum={k: v.astype(np.float64) for k, v in ranks[r]["m"].items()},
            iteration=case["iteration"])
        grads = {k: v.astype(np.float64) for k, v in ranks[r]["g"].items()}
        metrics = {}
        st2 = distributed_lion_step(st, grads, h, spec, topo, case["algo"],
                                    mask=mask, zero_mode=case["zero_mode"],
                                    metrics_out=metrics)
        # the runner's vote metrics of this step (runner.py:171-182), before
        # the sync (the runner computes them from the step's metrics_out)
        match = flip = counted = 0
        for layer in sorted(SIZES):
            ref = np.sign(allreduce_mean_f32(metrics["c_local"][layer], topo))
            vs = metrics["vote_sign"][layer]
            match += int(np.count_nonzero((vs == ref) & (vs != 0)))
            flip += int(np.count_nonzero((vs == -ref) & (vs != 0) & (ref != 0)))
            counted += vs.size
        metrics["agree"] = (match, flip, counted)
        if sync is not None:
            st2 = maybe_sync_momentum(st2, sync, topo)
        return st2, metrics

    res = run_ranks(world, fn, transport=InprocTransport(world))
    out[f"{name}/out/agree"] = np.asarray(res[0][1]["agree"], dtype=np.int64)
    out[f"{name}/out/timing_keys"] = np.asarray(
        [int("t_quant" in res[0][1]), int("t_comm" in res[0][1])], dtype=np.int64)
    p = f"{name}/"
    for layer in SIZES:
        out[p + f"in/theta/{layer}"] = ranks[0]["theta"][layer]
        for r in range(world):
            out[p + f"in/m/{r}/{layer}"] = ranks[r]["m"][layer]
            out[p + f"in/g/{r}/{layer}"] = ranks[r]["g"][layer]
        th0 = res[0][0].params[layer]
        for r in range(world):
            assert np.array_equal(res[r][0].params[layer], th0), "theta diverged"
            out[p + f"out/m/{r}/{layer}"] = res[r][0].momentum[layer]
        out[p + f"out/theta/{layer}"] = th0
        out[p + f"out/sign/{layer}"] = np.asarray(
            res[0][1]["vote_sign"][layer]).astype(np.int8)
        out[p + f"out/ties/{layer}"] = np.int64(res[0][1]["ties"][layer])
        for r in range(world):
            c = res[r][1]["c_local"][layer]
            if world <= 2:
                out[p + f"out/c/{r}/{layer}"] = c
            s = apply_sign(c, policy)
            if np.all(np.abs(s) == 1):
                out[p + f"out/words/{r}/{layer}"] = sign_words(s)
            if spec is not None and spec.bits > 1:
                out[p + f"out/q/{r}/{layer}"] = quantize(c.ravel(), spec).astype(np.int16)
                out[p + f"out/norm/{r}/{layer}"] = np.float64(
                    lp_mean_norm(c.ravel(), spec.norm_p))
    if mask is not None:
        for k, v in mask.items():
            out[p + f"in/mask/{k}"] = v


def run_collective_case(case: dict, out: dict):
    name = case["name"]
    world, n, kind = case["world"], case["n"], case["kind"]
    rng = np.random.default_rng(case["seed"])
    p = f"{name}/"
    if kind == "direct":
        q_max = case["q_max"]
        binary = case.get("binary", False)
        if binary:
            vecs = [rng.choice([-1, 1], size=n).astype(np.int64) for _ in range(world)]
        else:
            vecs = [rng.integers(-q_max, q_max + 1, size=n).astype(np.int64)
                    for _ in range(world)]

        def fn(topo):
            return direct_allreduce(vecs[topo.rank], topo, q_max=q_max,
                                    binary_signs=binary)
    elif kind == "compressed":
        vecs = [rng.normal(size=n).astype(np.float32).astype(np.float64)
                for _ in range(world)]
        policy = SignPolicy("alternating", iteration=case["t"])

        def fn(topo):
            return compressed_allreduce_1bit(vecs[topo.rank], topo, policy)
    elif kind == "mean":
        vecs = [rng.normal(size=n).astype(np.float32).astype(np.float64)
                for _ in range(world)]

        def fn(topo):
            return allreduce_mean_f32(vecs[topo.rank], topo)
    else:
        raise ValueError(kind)
    res = run_ranks(world, fn, transport=InprocTransport(world))
    for r in range(world):
        out[p + f"in/{r}"] = vecs[r]
    if kind == "mean":
        for r in range(1, world):
            assert np.array_equal(res[r], res[0])
        out[p + "out/values"] = res[0]
    else:
        for r in range(1, world):
            assert np.array_equal(res[r].values, res[0].values)
        out[p + "out/values"] = np.asarray(res[0].values)
        out[p + "out/ties"] = np.int64(res[0].ties)


def make_checkpoint():
    """A checkpoint written by the reference's save_checkpoint
    (optimizer.py:279) for the byte-level format test."""
    rng = np.random.default_rng(7)
    shapes = {"w.weight": (3, 5), "a.bias": (4,), "z": (1, 2, 3)}
    f32 = lambda s: rng.standard_normal(s).astype(np.float32).astype(np.float64)  # noqa: E731
    state = WorkerState(params={k: f32(v) for k, v in shapes.items()},
                        momentum={k: f32(v) for k, v in shapes.items()}, iteration=17)
    save_checkpoint(os.path.join(HERE, "ref_ckpt.bin"), state,
                    LionHyper(lr=3e-4, beta1=0.9, beta2=0.99, weight_decay=0.1))


QUANT_INPUTS = ("lap", "halves", "zeros", "one", "spiky")
QUANT_PS = (1.0, 2.0, 0.5, 3.0, float("inf"), 0.0)
QUANT_BITS = (2, 5, 8)
PACK_CASES = [  # (width, offset, low, high, count)
    (1, 1, None, None, 1001), (1, 0, 0, 1, 77), (2, 1, -1, 2, 1000), (2, 0, 0, 3, 5),
    (4, 7, -7, 8, 999), (4, 0, 0, 15, 1), (8, 128, -128, 127, 1003), (8, 0, 0, 255, 0),
]


def quant_input(kind: str) -> np.ndarray:
    rng = np.random.default_rng(len(kind) * 7919)
    if kind == "lap":
        x = rng.laplace(size=3001)
        x[rng.random(3001) < 0.05] = 0.0
        x[3] = -0.0
        x[17] = 250.0
    elif kind == "halves":   # exact half-way points of the scaled grid
        x = np.array([0.5, -0.5, 1.5, -1.5, 2.5, -2.5, 3.5, 0.0, -0.0, 1.0, 7.0, -7.0])
    elif kind == "zeros":
        x = np.zeros(10)
    elif kind == "one":
        x = np.array([-3.25])
    else:
        x = rng.standard_normal(2048) * 1e-3
        x[::97] = rng.choice([-1.0, 1.0], size=x[::97].size) * 40.0
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def make_quant_golden():
    """Standalone quant.py functions of the reference on fixed inputs:
    lp_mean_norm (every p), quantize/dequantize (every variant, nearest),
    apply_sign (both policies), pack/unpack/PackedBits wire bytes."""
    out: dict = {}
    for kind in QUANT_INPUTS:
        x = quant_input(kind)
        out[f"x/{kind}"] = x
        for p in QUANT_PS:
            out[f"norm/{kind}/{p}"] = np.float64(lp_mean_norm(x, p))
            for bits in QUANT_BITS:
                for lt in (False, True):
                    for nz in (False, True):
                        spec = QuantSpec(bits=bits, norm_p=p, log_transform=lt, no_zero=nz)
                        key = f"{kind}/{p}/{bits}/{int(lt)}/{int(nz)}"
                        q = quantize(x, spec)
                        out[f"q/{key}"] = q.astype(np.int16)
                        y, s = x, None
                        if lt:
                            s = lp_mean_norm(x, 1.0)
                            if s > 0:
                                y = np.sign(x) * np.log1p(np.abs(x) / s)
                        norm = lp_mean_norm(y, p)
                        out[f"deq/{key}"] = dequantize(q, spec, norm, s)
        for mode, it in (("alternating", 1), ("alternating", 2), ("exact-ternary", 1)):
            out[f"sign/{kind}/{mode}/{it}"] = apply_sign(
                x, SignPolicy(mode=mode, iteration=it)).astype(np.int8)
    rng = np.random.default_rng(99)
    for i, (w, off, lo, hi, count) in enumerate(PACK_CASES):
        if lo is None:
            v = rng.choice([-1, 1], size=count).astype(np.int64)
        else:
            v = rng.integers(lo, hi + 1, size=count).astype(np.int64)
        pk = pack(v, w, off)
        assert np.array_equal(unpack(pk), v)
        assert PackedBits.from_bytes(pk.to_bytes()) == pk
        out[f"pack/{i}/values"] = v
        out[f"pack/{i}/wire"] = np.frombuffer(pk.to_bytes(), dtype=np.uint8).copy()
    meta = {"inputs": list(QUANT_INPUTS), "ps": list(QUANT_PS), "bits": list(QUANT_BITS),
            "pack": PACK_CASES}
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden_quant.npz"), **out)
    return len(out)


SIGNSGD_CASES = [  # (algo, world, kind, zero_mode, iteration)
    ("ps", 3, "laplace", "alternating", 0), ("ps", 4, "zeros", "exact-ternary", 1),
    ("ps_efficient", 5, "ties", "alternating", 1), ("direct", 2, "laplace", "alternating", 0),
    ("direct", 8, "ties", "alternating", 3), ("compressed1bit", 4, "zeros", "alternating", 0),
    ("compressed1bit", 1, "laplace", "alternating", 1), ("ps", 1, "zeros", "exact-ternary", 0),
]


def make_metrics_golden():
    """signsgd_majority_step and the momentum-divergence metrics of the
    reference on seeded inputs."""
    out: dict = {}
    for i, (algo, world, kind, zm, it) in enumerate(SIGNSGD_CASES):
        ranks = synth_rank_inputs(300 + i, world, SIZES, kind)
        h = LionHyper(beta1=0.9, beta2=0.99, lr=1e-3, weight_decay=0.1)

        def fn(topo, ranks=ranks):
            r = topo.rank
            st = WorkerState(
                params={k: v.astype(np.float64) for k, v in ranks[r]["theta"].items()},
                momentum={k: v.astype(np.float64) for k, v in ranks[r]["m"].items()},
                iteration=it)
            grads = {k: v.astype(np.float64) for k, v in ranks[r]["g"].items()}
            st2 = signsgd_majority_step(st, grads, h, topo, algo=algo, zero_mode=zm)
            return st2, momentum_divergence(st2, topo)

        res = run_ranks(world, fn, transport=InprocTransport(world))
        p = f"sgd{i}/"
        for k in SIZES:
            out[p + f"in/theta/{k}"] = ranks[0]["theta"][k]
            for r in range(world):
                out[p + f"in/m/{r}/{k}"] = ranks[r]["m"][k]
                out[p + f"in/g/{r}/{k}"] = ranks[r]["g"][k]
                assert np.array_equal(res[r][0].params[k], res[0][0].params[k])
            out[p + f"out/theta/{k}"] = res[0][0].params[k]
            out[p + f"out/div/{k}"] = np.float64(res[0][1][k])
        moms = [{k: v.astype(np.float64) for k, v in rk["m"].items()} for rk in ranks]
        div = divergence_from_momenta(moms)
        for k in SIZES:
            out[p + f"out/divm/{k}"] = np.float64(div[k])
    meta = {"signsgd": SIGNSGD_CASES}
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden_metrics.npz"), **out)


def main():
    steps: dict = {}
    for case in STEP_CASES:
        run_step_case(case, steps)
    steps["meta"] = np.frombuffer(json.dumps(
        {"cases": STEP_CASES, "sizes": {k: list(v) for k, v in SIZES.items()}}
    ).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden_steps.npz"), **steps)
    colls: dict = {}
    for case in COLLECTIVE_CASES:
        run_collective_case(case, colls)
    colls["meta"] = np.frombuffer(json.dumps({"cases": COLLECTIVE_CASES}).encode(),
                                  dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden_collectives.npz"), **colls)
    make_checkpoint()
    make_metrics_golden()
    nq = make_quant_golden()
    print(f"{nq} standalone quant arrays")
    print(f"{len(STEP_CASES)} step cases, {len(COLLECTIVE_CASES)} collective cases")


if __name__ == "__main__":
    main()
