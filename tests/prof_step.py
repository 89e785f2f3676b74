"""Host-side cost of one multi-GPU step (a tuning tool, not a test).

    torchrun --nproc-per-node 2 tests/prof_step.py [--workload gpt2s_sumsigns] [--steps 300]

Runs the bench workload's step on synthetic state, reports the host time
per ``distributed_lion_step`` call in deferred-error mode (the enqueue cost
alone) and in step mode, and rank 0 prints the cProfile top functions of
the deferred run.
"""

import argparse
import cProfile
import io
import os
import pstats
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2411_16462_b200 as lc  # noqa: E402
from paper_2411_16462_b200 import transport as T  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt2s_sumsigns")
    ap.add_argument("--steps", type=int, default=300)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    tp = lc.NcclTransport.init_process(rank, world, dev)
    topo = lc.Topology(world_size=world, rank=rank, transport=tp)
    layout_fn, algo, bits, sync, _ = bench.WORKLOADS[args.workload]
    shapes = layout_fn()
    layout = lc.Layout(shapes)
    n = layout.n
    qkw = bench.quant_kwargs(bits)
    spec = None if qkw is None else lc.QuantSpec(**qkw)
    theta = torch.randn(n, device=dev)
    mom = torch.randn(n, device=dev)
    grad = torch.randn(n, device=dev)
    st = lc.WorkerState(params=layout.views(theta), momentum=layout.views(mom), iteration=0)
    g = layout.views(grad)
    h = lc.LionHyper(beta1=0.9, beta2=0.99, lr=1e-4, weight_decay=0.0)
    out = {}
    for mode in ("deferred", "step", "deferred"):
        tp.error_mode = mode
        for _ in range(20):
            st = lc.distributed_lion_step(st, g, h, spec, topo, algo)
        torch.cuda.synchronize()
        dist.barrier()
        prof = cProfile.Profile() if (mode == "deferred" and rank == 0 and "d" in out) else None
        t0 = time.perf_counter()
        if prof:
            prof.enable()
        for _ in range(args.steps):
            st = lc.distributed_lion_step(st, g, h, spec, topo, algo)
        if prof:
            prof.disable()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        key = "d" if mode == "deferred" and "d" not in out else ("s" if mode == "step" else "dprof")
        out[key] = ((t1 - t0) / args.steps * 1e6, (t2 - t0) / args.steps * 1e6)
        if prof:
            s = io.StringIO()
            pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(30)
            print(s.getvalue()[:6000])
    if rank == 0:
        print({k: tuple(round(x, 1) for x in v) for k, v in out.items()},
              "(host us/step enqueue, us/step incl. drain)")
    T.host_wait()
    tp.close() if hasattr(tp, "close") else None
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
