"""Benchmark of the B200 Lion Cub distributed optimizer step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload NAME]

N > 1 runs under torchrun (one process per GPU, NCCL over NVLink).  A "step"
is one ``distributed_lion_step`` (+ ``maybe_sync_momentum`` where the
workload syncs) over the workload's full synthetic parameter buffer, inputs
resident in HBM.  Rank 0 prints ONE JSON line.

Default workload = BASELINE.json configs[4], the largest configuration that
fits one B200: a 7e9-parameter flat buffer, Lion Cub full step (1-bit
majority vote + all-layer momentum sync every step; the sync is a no-op at
one rank).  theta/m/g are 28 GB each (84 GB resident).  ``--workload
tinyllama_1bit_sync`` is the north-star line (configs[3]), ``gpt2s_sumsigns``
configs[1].  Every array of those workloads is larger than the 126 MB L2, so
no L2 flush is needed between steps; workloads whose 12 B/param working set
is under 2x L2 (c1_1bit_1m) flush L2 before every step and time each step
alone with its own event pair.

Reference arm (``--impl reference``): the UNMODIFIED reference ``lioncomm``
(installed once into baseline/_ref with pip) through its own
``run_ranks(P, fn, transport=InprocTransport(P))`` on the host cores, on a
bounded per-rank sample of the workload, extrapolated linearly in params.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


# ---------------------------------------------------------------------------
# Workloads (BASELINE.json configs)
# ---------------------------------------------------------------------------

def gpt2_small_layout() -> dict:
    d, L, V, T = 768, 12, 50257, 1024
    shapes = {"wte.weight": (V, d), "wpe.weight": (T, d),
              "ln_f.weight": (d,), "ln_f.bias": (d,)}
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


WORKLOADS = {
    # name: (layout fn, algo, bits, sync (period, layers) or None, description)
    "gpt2s_sumsigns": (gpt2_small_layout, "direct", 1, None,
                       "GPT-2-small-sized buffer, p-bit sum-of-signs vote (configs[1])"),
    "c1_1bit_1m": (lambda: {"w": (1 << 20,)}, "compressed1bit", None, None,
                   "1M-param flat buffer, 1-bit compressed vote (configs[0] at GPU scale)"),
    "tinyllama_1bit_sync": (tinyllama_layout, "compressed1bit", None,
                            (10, ("model.embed_tokens.weight", "lm_head.weight")),
                            "TinyLlama-1.1B layout, 1-bit vote, embed/head momentum sync "
                            "every 10 steps (configs[3])"),
    "tinyllama_1bit": (tinyllama_layout, "compressed1bit", None, None,
                       "TinyLlama-1.1B layout, 1-bit vote, no sync"),
    "gpt2s_l1_5bit": (gpt2_small_layout, "direct", 5, None,
                      "GPT-2-small-sized buffer, L1 5-bit p-bit vote (paper's 8-bit Lion Cub)"),
    "gpt2s_qinf_stoch_5bit": (gpt2_small_layout, "direct",
                              dict(bits=5, norm_p=float("inf"), rounding="stochastic"), None,
                              "GPT-2-small-sized buffer, 5-bit max-norm quantizer with "
                              "stochastic rounding (QuantSpec variant)"),
    "gpt2s_ps": (gpt2_small_layout, "ps", None, None,
                 "GPT-2-small-sized buffer, full-precision (ps) vote"),
    "gpt2s_1bit_syncall": (gpt2_small_layout, "compressed1bit", None, (1, "all"),
                           "GPT-2-small-sized buffer, 1-bit vote + all-layer momentum sync "
                           "every step"),
    "flat7b_1bit_sync": (lambda: {"w": (7_000_000_000,)}, "compressed1bit", None,
                         (1, "all"), "7e9 flat buffer, 1-bit vote + all-layer sync (configs[4])"),
    "flat7b_1bit": (lambda: {"w": (7_000_000_000,)}, "compressed1bit", None, None,
                    "7e9 flat buffer, 1-bit vote, no momentum sync (the non-firing C5 step)"),
}


def quant_kwargs(bits) -> dict | None:
    """QuantSpec kwargs of a workload's ``bits`` entry (int: L1, nearest)."""
    if bits is None:
        return None
    return dict(bits) if isinstance(bits, dict) else dict(bits=bits, norm_p=1.0)


def norm_bytes(bits) -> float:
    """HBM bytes/param of the per-layer norm pass(es) of a quantizer."""
    kw = quant_kwargs(bits)
    if kw is None or kw["bits"] == 1:
        return 0.0
    b = 8.0 if kw.get("norm_p") == float("inf") else 16.0  # max pass (+ pairwise sum)
    return b + (16.0 if kw.get("log_transform") else 0.0)


def numel(shapes: dict) -> int:
    return sum(math.prod(s) for s in shapes.values())


# ---------------------------------------------------------------------------
# Algorithmic bytes
# ---------------------------------------------------------------------------

def kernel_bytes(name: str, n: int, P: int, F: int, kind: str, nb: float = 16.0) -> float:
    """Algorithmic HBM bytes of ONE launch of our kernel on an n-param step."""
    L = -(-max(-(-n // P), 1) // 1024) * 1024
    if name == "lc_fused_local_step":
        return 20.0 * n
    if name == "lc_encode":
        if kind == "f64":
            return 12.0 * n + 8.0 * n
        return 12.0 * n + n * F / 8.0
    if name == "lc_encode_sync":   # g, m in; signs + m' out (m' to the owners' staging)
        return 12.0 * n + n / 8.0
    if name == "lc_vote_apply_sync":  # theta r/w, staging rows in, words; means land in m
        return 8.0 * n + 4.0 * n + n / 8.0
    if name == "lc_apply_update":
        return 8.0 * n + n / 8.0
    if name == "lc_vote_apply":   # theta r/w, voted words, the owner's P slots
        return 8.0 * n + n / 8.0 + P * L / 8.0
    if name == "lc_vote_update":  # theta r/w, P replicated rows
        return 8.0 * n + P * n / 8.0
    if name == "lc_vote_bits":
        return (P + 1) * L / 8.0
    if name == "lc_fields_vote":
        return L * F / 8.0 + L / 8.0
    if name == "lc_f64_sum_vote":
        return P * L * 8.0 + L / 8.0
    if name == "lc_l1_scales":
        return 16.0 * n  # g, m read twice: max pass, then the pairwise sum
    if name == "lc_norm_scales":
        return nb * n
    return 0.0


def step_roofline(n: int, P: int, F: int, kind: str, sync_frac: float,
                  hbm_gbs: float, nvl_gbs: float = 770.0, nb: float = 0.0) -> dict:
    """Whole-step lower bound: max(HBM bytes / HBM BW, NVLink bytes / link BW)."""
    if P == 1:
        hbm = 20.0 * n + nb * n
        nvl = 0.0
    elif kind == "1bit":
        hbm = 20.0 * n + 2 * n / 8.0
        nvl = 2 * (P - 1) / P * n / 8.0
    elif kind == "fields":
        hbm = 20.0 * n + 2 * n * F / 8.0 + 2 * n / 8.0 + nb * n
        nvl = (P - 1) / P * n * (F + 1) / 8.0
    else:
        hbm = 36.0 * n
        nvl = (P - 1) / P * n * 8.0 + (P - 1) / P * n / 8.0
    if sync_frac and P > 1:   # one rank: the mean of one row is the row (no-op)
        hbm += 16.0 * sync_frac * n
        nvl += sync_frac * 2 * (P - 1) / P * 4.0 * n
    t_h = hbm / (hbm_gbs * 1e9)
    t_n = nvl / (nvl_gbs * 1e9)
    return {"hbm_bytes": hbm, "nvlink_bytes": nvl, "t_hbm_ms": t_h * 1e3,
            "t_nvlink_ms": t_n * 1e3, "t_nvlink_ms_at_900": nvl / 900e9 * 1e3,
            "bound": "hbm" if t_h >= t_n else "nvlink"}


NVL_GBS = 770.0   # NVLink 5 per direction, measured peak in B200_PROFILING.md
NVL_NOMINAL_GBS = 900.0  # north_star: 900 GB/s per direction


def measured_peaks() -> tuple[dict, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0}, "fallback"


def traffic_table() -> dict:
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------------------
# Clock sampling (NVML, every ~5 ms in a thread)
# ---------------------------------------------------------------------------

class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting"}

    def __init__(self, device_index: int):
        self.samples = []
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), sm, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self, t0: float, t1: float) -> dict:
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        if not win:  # region shorter than the sampling period: nearest samples
            win = sorted(self.samples, key=lambda s: abs(s[0] - (t0 + t1) / 2))[:3]
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        mask = 0
        for s in win:
            mask |= s[2]
        reasons = sorted({v for k, v in self.REASONS.items() if mask & k})
        return {"sm_mhz": statistics.median(s[1] for s in win),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(win)}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the oracle port on the host cores
# ---------------------------------------------------------------------------

class CpuReference:
    """The reference algorithm (the oracle's restatement of
    optimizer.distributed_lion_step, ranks simulated in one process) on a
    bounded sample, timed on the host cores.  Element chunks run on a thread
    pool (numpy releases the GIL), so ``cores`` threads work at once."""

    def __init__(self, world: int, algo: str, bits, sample: int, threads: int | None = None):
        from concurrent.futures import ThreadPoolExecutor

        from oracle import lioncub_oracle as O

        self.O = O
        self.world, self.algo, self.bits, self.sample = world, algo, bits, sample
        self.cores = threads or len(os.sched_getaffinity(0))
        ranks = O.synth_rank_inputs(0, world, {"w": (sample,)}, "laplace")
        self.h = O.Hyper(0.9, 0.99, 1e-4, 0.0)
        kw = quant_kwargs(bits)
        self.spec = None if kw is None else O.Spec(**kw)
        self.seeds = list(range(1, world + 1)) \
            if kw and kw.get("rounding") == "stochastic" else None
        chunk = -(-sample // self.cores)
        self.pieces = []
        for a in range(0, sample, chunk):
            b = min(sample, a + chunk)
            self.pieces.append(([{"w": rk["theta"]["w"][a:b]} for rk in ranks],
                                [{"w": rk["m"]["w"][a:b]} for rk in ranks],
                                [{"w": rk["g"]["w"][a:b]} for rk in ranks]))
        self.pool = ThreadPoolExecutor(max_workers=self.cores)

    def _one(self, piece):
        th, m, g = piece
        self.O.distributed_step(th, m, g, self.h, self.spec, self.algo, 0, seeds=self.seeds)

    def step(self) -> float:
        t0 = time.perf_counter()
        list(self.pool.map(self._one, self.pieces))
        return time.perf_counter() - t0

    def describe(self) -> str:
        b = "" if self.bits is None else f", bits={self.bits}"
        return (f"{self.sample}-param slice per rank x {self.world} simulated ranks "
                f"({self.algo}{b}), float64 numpy port of optimizer.distributed_lion_step "
                f"(oracle/lioncub_oracle.py) on {self.cores} host threads")

    def timed(self, budget_s: float) -> dict:
        self.step()
        times = []
        t_end = time.perf_counter() + budget_s
        while not times or time.perf_counter() < t_end or len(times) < 2:
            times.append(self.step())
        t = statistics.median(times)
        return {"value": self.world * self.sample / t, "unit": "params/s",
                "cores": self.cores, "kind": "port", "sample": self.describe()}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_lioncomm():
    """The unmodified reference package, pip-installed into baseline/_ref
    (`pip install --no-index --target baseline/_ref`), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "lioncomm")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import lioncomm
    return lioncomm


class LioncommReference:
    """The reference's own CPU path, unmodified: ``lioncomm``'s
    ``distributed_lion_step`` (+ ``maybe_sync_momentum`` where the workload
    syncs) on P rank threads sharing one ``InprocTransport`` through
    ``run_ranks`` (collectives.py:363-403), on a ``sample``-param flat buffer
    per rank.  Inputs follow BASELINE.md §2: fp32-generated, upcast to f64,
    correlated workers (shared Laplace base + Laplace noise, runner.py:289-297),
    seeds SeedSequence([0, rank]).  A workload that syncs a subset of its
    layers keeps that fraction as a second layer of the sample.  Step time =
    max over ranks of each rank's wall time for that step."""

    def __init__(self, world: int, algo: str, bits, sync, frac_synced: float, sample: int):
        import numpy as np
        lcm = load_lioncomm()
        if lcm is None:
            raise RuntimeError("baseline/_ref has no lioncomm install")
        from lioncomm import collectives as CC
        from lioncomm import optimizer as O
        from lioncomm import quant as Q
        from lioncomm import transport as T
        self.O, self.CC, self.T = O, CC, T
        self.world, self.algo, self.bits, self.sample = world, algo, bits, sample
        self.cores = world  # one numpy rank thread each (elementwise numpy is single-threaded)
        kw = quant_kwargs(bits)
        self.spec = None if kw is None else Q.QuantSpec(**kw)
        self.policy = None
        names = {"w": sample}
        if sync is not None:
            period, layers = sync
            if layers == "all":
                self.policy = O.SyncPolicy(period=period, layers="all")
            else:
                ns = max(1, int(round(frac_synced * sample)))
                names = {"a_synced": ns, "w": sample - ns}
                self.policy = O.SyncPolicy(period=period, layers=frozenset({"a_synced"}))
        g0 = np.random.default_rng(np.random.SeedSequence([0]))
        theta = {k: g0.standard_normal(c, dtype=np.float32).astype(np.float64)
                 for k, c in names.items()}
        base = {k: g0.laplace(0.0, 1.0, c).astype(np.float32) for k, c in names.items()}
        self.states, self.grads = [], []
        for r in range(world):
            gr = np.random.default_rng(np.random.SeedSequence([0, r]))
            mom = {k: (0.1 * gr.standard_normal(c, dtype=np.float32)).astype(np.float64)
                   for k, c in names.items()}
            grad = {k: (base[k] + gr.laplace(0.0, 1.0, c).astype(np.float32)).astype(np.float64)
                    for k, c in names.items()}
            self.states.append(O.WorkerState(params={k: v.copy() for k, v in theta.items()},
                                             momentum=mom, iteration=0))
            self.grads.append(grad)
        self.rngs = [np.random.default_rng(100 + r) for r in range(world)]

    def run(self, steps: int) -> list:
        """``steps`` reference steps on every rank thread; per-step time =
        max over ranks (seconds)."""
        O, CC, T = self.O, self.CC, self.T
        per_rank = [None] * self.world

        def fn(topo):
            r = topo.rank
            st, times = self.states[r], []
            for _ in range(steps):
                t0 = time.perf_counter()
                st = O.distributed_lion_step(st, self.grads[r], self.h_ref(), self.spec, topo,
                                             self.algo, rng=self.rngs[r])
                if self.policy is not None:
                    st = O.maybe_sync_momentum(st, self.policy, topo)
                times.append(time.perf_counter() - t0)
            self.states[r] = st
            per_rank[r] = times
            return None

        CC.run_ranks(self.world, fn, transport=T.InprocTransport(self.world), timeout=600.0)
        return [max(per_rank[r][i] for r in range(self.world)) for i in range(steps)]

    def h_ref(self):
        return self.O.LionHyper(beta1=0.9, beta2=0.99, lr=1e-4, weight_decay=0.0)

    def describe(self) -> str:
        b = "" if self.bits is None else f", bits={self.bits}"
        sy = "" if self.policy is None else \
            f" + maybe_sync_momentum(period={self.policy.period})"
        return (f"unmodified lioncomm (baseline/_ref) distributed_lion_step({self.algo}{b}){sy} "
                f"via run_ranks({self.world}, InprocTransport) on a {self.sample}-param flat "
                f"sample per rank, float64 numpy, {self.world} rank thread(s)")

    def timed(self, budget_s: float) -> dict:
        self.run(1)
        times = []
        t_end = time.perf_counter() + budget_s
        while not times or time.perf_counter() < t_end or len(times) < 3:
            times += self.run(1)
        t = min(times)  # best of the budget (best of 3)
        return {"value": self.world * self.sample / t, "unit": "params/s",
                "cores": self.cores, "kind": "reference", "sample": self.describe(),
                "ms_per_step_sample": t * 1e3, "extrapolated": True,
                "extrapolation": "linear in params: params/s of the sample applied to the "
                                 "workload (the reference needs ~77 B/param/rank of host RAM)"}


def sync_fraction(shapes: dict, sync) -> float:
    """Fraction of the params a firing sync averages (per firing step)."""
    if sync is None:
        return 0.0
    _, layers = sync
    n = numel(shapes)
    return 1.0 if layers == "all" else sum(math.prod(shapes[k]) for k in layers) / n


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    layout_fn, algo, bits, sync, desc = WORKLOADS[args.workload]
    shapes = layout_fn()
    n = numel(shapes)
    world = args.gpus
    sample = min(n, args.ref_sample)
    cfg = {"workload": args.workload, "description": desc, "params": n, "algo": algo,
           "bits": bits, "world": world, "sample_params_per_rank": sample,
           "same_config": False,
           "extrapolation": f"params/s measured on a {sample}-param per-rank sample, "
                            "applied linearly to the workload's params"}
    if load_lioncomm() is not None:
        ref = LioncommReference(world, algo, bits, sync, sync_fraction(shapes, sync), sample)
        ref.run(args.warmup)
        timed = ref.run(args.steps)
        kind, cores, descr = "reference", ref.cores, ref.describe()
    else:  # no pip install in baseline/_ref: the oracle port (labelled)
        ref = CpuReference(world, algo, bits, sample)
        for _ in range(args.warmup):
            ref.step()
        timed = [ref.step() for _ in range(args.steps)]
        kind, cores, descr = "port", ref.cores, ref.describe()
    t = sum(timed) / len(timed)
    value = world * sample / t
    line = {"metric": METRIC, "value": value, "unit": "params/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "ms_per_step_extrapolated": world * n / value * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference", "config": cfg,
            "cpu_baseline": {"value": value, "unit": "params/s", "cores": cores,
                             "kind": kind, "sample": descr},
            "e2e": {"value": value, "unit": "params/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


METRIC = "Lion Cub step time (ms) & params/s at 1/2/4/8 B200, % of HBM/NVLink roofline"


# ---------------------------------------------------------------------------
# The B200 arm
# ---------------------------------------------------------------------------

L2_BYTES = 126 * 1000 * 1000


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="flat7b_1bit_sync", choices=sorted(WORKLOADS))
    ap.add_argument("--ref-sample", type=int, default=1 << 22)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=1 << 23)
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="timed e2e steps (0: --steps, capped at 5 above 1e9 params)")
    ap.add_argument("--graph", action="store_true",
                    help="replay the single-GPU step as a CUDA graph (launch-bound sizes)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2411_16462_b200 as lc
    from paper_2411_16462_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if rank == 0:
            print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _lib.load()
    if world > 1:
        import datetime
        dist.init_process_group("nccl", device_id=dev,
                                timeout=datetime.timedelta(seconds=240))
        transport = lc.NcclTransport.init_process(rank, world, dev)
    else:
        transport = lc.LocalTransport(1, device=dev)
    topo = lc.Topology(world_size=world, rank=rank, transport=transport)

    layout_fn, algo, bits, sync, desc = WORKLOADS[args.workload]
    shapes = layout_fn()
    n = numel(shapes)
    qkw = quant_kwargs(bits)
    spec = None if qkw is None else lc.QuantSpec(**qkw)
    nbits = None if qkw is None else qkw["bits"]
    rng = np.random.default_rng(rank) if spec is not None and spec.rounding == "stochastic" \
        else None
    policy = None
    sync_frac = 0.0
    if sync is not None:
        period, layers = sync
        policy = lc.SyncPolicy(period=period, layers=layers if isinstance(layers, str)
                               else frozenset(layers))
        sync_frac = sync_fraction(shapes, sync) / period
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=1e-4, weight_decay=0.0)

    # synthetic state: theta shared (seed 0), m and g per rank; g = base +
    # noise (Laplace-correlated workers, runner.py:289-297).  Generated in
    # 2^27-element chunks so a 7e9 buffer never needs more than its own
    # 3 x 28 GB plus one chunk of temporaries.
    layout = lc.Layout(shapes)
    theta = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    mom = torch.empty_like(theta)
    grad = torch.empty_like(theta)
    gen = torch.Generator(device=dev)
    CH = 1 << 27

    def laplace(out, g_):
        out.exponential_(generator=g_)
        out.mul_(torch.where(torch.rand(out.shape, generator=g_, device=dev) < 0.5, -1.0, 1.0))

    for ci, a in enumerate(range(0, max(n, 1), CH)):
        b = min(max(n, 1), a + CH)
        gen.manual_seed(ci * 2 + 1)               # shared across ranks
        theta[a:b].normal_(generator=gen)
        laplace(grad[a:b], gen)                    # the shared base
        gen.manual_seed(1_000_003 * (rank + 1) + ci * 2)
        mom[a:b].normal_(generator=gen).mul_(0.1)
        noise = torch.empty(b - a, dtype=torch.float32, device=dev)
        laplace(noise, gen)
        grad[a:b].add_(noise)
        del noise
    st = lc.WorkerState(params=layout.views(theta), momentum=layout.views(mom), iteration=0)
    del mom  # the state owns it (a P2P sync may re-home it; do not pin the old buffer)
    g = layout.views(grad)
    stream = topo.stream
    torch.cuda.synchronize()

    graph = None
    if args.graph and world == 1 and (nbits is None or nbits == 1):
        graph = lc.StepGraph(st, g, h, spec, topo, algo)  # CUDA-graph replay of the P=1 step

    def step(state):
        if graph is not None:
            return graph.step()
        # sync=policy: distributed_lion_step + maybe_sync_momentum, with the
        # sync fused into the step's kernels where it can be (layers="all")
        return lc.distributed_lion_step(state, g, h, spec, topo, algo, rng=rng, sync=policy)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        st = step(st)
    barrier()
    # untimed soak so the clock sampler sees the part under load; the step
    # count is agreed across ranks (every rank must issue the same exchanges)
    t_probe = time.perf_counter()
    st = step(st)
    barrier()
    probe = torch.tensor([time.perf_counter() - t_probe], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(probe, op=dist.ReduceOp.MAX)
    soak = max(1, min(5000, int(0.4 / max(float(probe.item()), 1e-5))))
    for _ in range(soak):
        st = step(st)
    barrier()

    def timed_pass(record_kernels: bool):
        """K steps between a barrier + synchronize on both sides; returns
        (ms per step, host enqueue ms per step, our launches, kernel events)."""
        nonlocal st
        _lib.phase_events = {} if record_kernels else None
        l0 = _lib.launches
        t0 = time.perf_counter()
        if flush is None:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                st = step(st)
            e1.record(stream)
        else:
            evs = []
            for _ in range(args.steps):
                with torch.cuda.stream(stream):
                    flush.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                st = step(st)
                b.record(stream)
                evs.append((a, b))
        enq = (time.perf_counter() - t0) * 1e3 / args.steps
        barrier()
        nl = _lib.launches - l0
        ph = _lib.phase_events
        _lib.phase_events = None
        if flush is None:
            t = e0.elapsed_time(e1) / args.steps
        else:
            t = sum(a.elapsed_time(b) for a, b in evs) / args.steps
        return t, enq, nl, ph

    # state + gradient bytes a step touches; below 2x the 126 MB L2 every
    # timed step is preceded by an (untimed) L2 flush and timed alone
    flush = None
    if 12 * n < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    # the step time comes from a pass without per-kernel events (an event
    # between two kernels would break their programmatic-launch overlap);
    # a second pass of K steps records every kernel for the roofline
    w0 = time.perf_counter()
    ms, host_ms, launches, _ = timed_pass(False)
    w1 = time.perf_counter()
    ms_kpass, _, _, phases = timed_pass(True)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks = sampler.summary(w0, w1)
    sampler.stop()

    # per-kernel average durations over the timed region
    kern = {}
    for name, evs in phases.items():
        d = [a.elapsed_time(b) for a, b in evs]
        kern[name] = {"launches": len(d), "avg_ms": sum(d) / len(d), "total_ms": sum(d)}
    if graph is not None:
        # one fused kernel per replay: its duration is bounded by the step time
        launches = args.steps
        kern["lc_fused_local_step"] = {"launches": args.steps, "avg_ms": ms,
                                       "total_ms": ms * args.steps,
                                       "note": "CUDA-graph replay; step time used as kernel time"}
    cand = {k: v for k, v in kern.items() if k != "lc_barrier"}
    dominant = max(cand, key=lambda k: cand[k]["total_ms"]) if cand else None

    peaks, peak_src = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    P = world
    if algo == "compressed1bit":
        kind, F = "1bit", 1
    elif nbits is None:
        kind, F = "f64", 64
    elif nbits == 1 and P > 1 and transport.p2p:
        kind, F = "1bit", 1   # sum-of-signs ships 1-bit signs over peer memory
    else:
        kind = "fields"
        F = lc.field_bits(P, 1 if nbits == 1 else 2 * ((1 << (nbits - 1)) - 1))
    roof = None
    if dominant:
        bpl = kernel_bytes(dominant, n, P, F, kind, norm_bytes(bits))
        ach = bpl / (kern[dominant]["avg_ms"] * 1e-3) / 1e9
        ttab = traffic_table()
        tt = ttab.get(f"{args.workload}/P{P}/{dominant}")
        roof = {"kernel": dominant, "bound": "hbm", "achieved": ach, "peak": hbm_peak,
                "unit": "GB/s", "frac": ach / hbm_peak, "traffic": tt,
                "traffic_source": None if tt is None else
                ttab.get("_sources", {}).get(f"{args.workload}/P{P}/{dominant}",
                                             "profiles/traffic.json"),
                "algorithmic_bytes_per_launch": bpl,
                "avg_launch_ms": kern[dominant]["avg_ms"],
                "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs" if peak_src ==
                "measured" else "fallback 6650 GB/s (B200_PROFILING.md)"}
        if dominant == "lc_encode" and kind == "f64" and P > 1 and transport.p2p:
            # full-precision arm over peer memory: K1 is bound by its (P-1)/P x
            # 8 B/param of remote f64 stores
            per_launch = (P - 1) / P * 8.0 * n
            ach = per_launch / (kern[dominant]["avg_ms"] * 1e-3) / 1e9
            roof.update({"bound": "nvlink", "achieved": ach, "peak": NVL_GBS, "frac": ach / NVL_GBS,
                         "frac_of_nominal_900": ach / NVL_NOMINAL_GBS,
                         "algorithmic_bytes_per_launch": per_launch,
                         "peak_source": "B200_PROFILING.md NVLink per direction (measured)"})
        if dominant in ("lc_encode_sync", "lc_vote_apply_sync") and P > 1:
            # NVLink-bound halves of the fused momentum sync: (P-1)/P of the
            # m' rows leave in K1, (P-1)/P of the means leave in the vote kernel
            per_launch = (P - 1) / P * (4.0 + 1.0 / 8.0) * n
            ach = per_launch / (kern[dominant]["avg_ms"] * 1e-3) / 1e9
            roof.update({"bound": "nvlink", "achieved": ach, "peak": NVL_GBS, "frac": ach / NVL_GBS,
                         "frac_of_nominal_900": ach / NVL_NOMINAL_GBS,
                         "algorithmic_bytes_per_launch": per_launch,
                         "peak_source": "B200_PROFILING.md NVLink per direction (measured)"})
        if dominant == "lc_mean_pull_f32" and P > 1:
            # the momentum sync is NVLink-bound (synced values over the timed
            # steps / launches in them)
            # per direction: the other owners pull this rank's blocks AND this
            # owner stores its mean into every other rank: 2 (P-1)/P x 4 B
            per_launch = 2 * (P - 1) / P * 4.0 * sync_frac * n * args.steps / max(
                1, kern[dominant]["launches"])
            ach = per_launch / (kern[dominant]["avg_ms"] * 1e-3) / 1e9
            roof.update({"bound": "nvlink", "achieved": ach, "peak": NVL_GBS, "frac": ach / NVL_GBS,
                         "frac_of_nominal_900": ach / NVL_NOMINAL_GBS,
                         "algorithmic_bytes_per_launch": per_launch,
                         "peak_source": "B200_PROFILING.md NVLink per direction"})
    sr = step_roofline(n, P, F, kind, sync_frac, hbm_peak, nb=norm_bytes(bits))
    sr["frac"] = max(sr["t_hbm_ms"], sr["t_nvlink_ms"]) / ms

    # end to end through the public API with host buffers: pinned host
    # gradients in, updated parameters out (distributed_lion_step_host
    # pipelines both copies with the kernels chunk by chunk)
    e2e = None
    # pinned host g and theta (8 B/param) per rank must fit the host's RAM
    # with every local rank doing the same (7e9 params x 8 ranks would need
    # 448 GB): otherwise the e2e leg is skipped and says why
    e2e_skip = None
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 0
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    if avail and 8 * n * local_world > 0.7 * avail:
        e2e_skip = (f"host RAM: {local_world} ranks x 8 B/param x {n} params = "
                    f"{8 * n * local_world / 1e9:.0f} GB pinned > 70% of the "
                    f"{avail / 1e9:.0f} GB available")
    if world > 1 and not args.no_e2e:
        # every rank takes the same branch (the e2e steps are collective)
        ok = torch.tensor([0 if e2e_skip else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not int(ok.item()) and e2e_skip is None:
            e2e_skip = "host RAM: another local rank could not pin its e2e buffers"
    if e2e_skip is not None:
        e2e = {"value": None, "unit": "params/s", "h2d_bytes_per_step": 4 * n,
               "d2h_bytes_per_step": 4 * n, "skipped": e2e_skip}
    if not args.no_e2e and e2e_skip is None:
        host_g = torch.empty(n, dtype=torch.float32, pin_memory=True)
        host_g.copy_(grad[:n])
        host_t = torch.empty(n, dtype=torch.float32, pin_memory=True)
        e2e_steps = args.e2e_steps or (min(args.steps, 5) if n > 1_000_000_000 else args.steps)

        def step_host(state):
            state = lc.distributed_lion_step_host(state, host_g, h, spec, topo, algo,
                                                  params_out=host_t, chunk=args.e2e_chunk,
                                                  rng=rng)
            if policy is not None:
                state = lc.maybe_sync_momentum(state, policy, topo)
            return state

        for _ in range(2):
            st = step_host(st)
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(e2e_steps):
            st = step_host(st)
        f1.record(stream)
        barrier()
        ems = f0.elapsed_time(f1) / e2e_steps
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": P * n / (ems * 1e-3), "unit": "params/s", "ms_per_step": ems,
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
               "steps": e2e_steps,
               "path": "distributed_lion_step_host: pinned host grads -> step -> pinned "
                       f"host params, {args.e2e_chunk}-element chunks pipelined",
               "host_state": "g in and theta out every step (8 B/param over PCIe); the "
                             "momentum stays resident on the device like a torch.optim "
                             "state -- the reference API passes the whole f64 state "
                             "(theta, m in and out) through host memory"}

    cpu = cpu_port = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(n, args.ref_sample)
        if load_lioncomm() is not None:
            cpu = LioncommReference(1, algo, bits, sync, sync_fraction(shapes, sync),
                                    sample).timed(args.cpu_budget)
        cpu_port = CpuReference(1, algo, bits, sample).timed(args.cpu_budget)
        if cpu is None:
            cpu = cpu_port

    if rank == 0:
        line = {"metric": METRIC, "value": P * n / (ms * 1e-3), "unit": "params/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "fp32 state, f64 math",
                "data": "synthetic (Laplace-correlated grads, runner.py:289-297 recipe)",
                "config": {"workload": args.workload, "description": desc, "params": n,
                           "tensors": len(shapes), "algo": algo, "bits": bits,
                           "parallelism": f"dp{world}", "field_bits": F,
                           "cuda_graph": graph is not None,
                           "exchange": ("nvlink peer memory" if world > 1 and transport.p2p
                                        else "nccl" if world > 1 else "none (P=1)"),
                           "l2": ("inputs larger than L2 (no flush needed)" if flush is None
                                  else "L2 flushed (252 MB write) before every timed step; "
                                       "steps timed individually, flush excluded")},
                "roofline": roof, "step_roofline": sr, "kernels": kern,
                "ms_per_step_kernel_pass": ms_kpass,
                # the exchange is fused into the kernels (peer-memory stores /
                # loads), so its rate is reported over the whole step: the
                # algorithmic NVLink bytes each rank moves per direction per
                # step / step time, against the per-direction link peak
                "nvlink": None if world == 1 else {
                    "bytes_per_rank_per_direction": sr["nvlink_bytes"],
                    "achieved_gbs_over_step": sr["nvlink_bytes"] / (ms * 1e-3) / 1e9,
                    "peak_gbs": NVL_GBS,
                    "frac_of_peak": sr["nvlink_bytes"] / (ms * 1e-3) / 1e9 / NVL_GBS,
                    "peak_gbs_nominal": NVL_NOMINAL_GBS,
                    "frac_of_nominal": sr["nvlink_bytes"] / (ms * 1e-3) / 1e9 / NVL_NOMINAL_GBS},
                "cpu_baseline": cpu, "cpu_baseline_port": cpu_port,
                "e2e": e2e, "gpu_launches": launches,
                "host_enqueue_ms_per_step": host_ms,
                "clocks": clocks}
        print(json.dumps(line))
    if world > 1:
        transport.close()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
