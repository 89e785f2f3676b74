"""Micro-benchmark of the peer-memory exchange pieces (torchrun, >= 2 GPUs).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/p2p_microbench.py

Prints per-rank JSON: back-to-back device barrier latency, host enqueue time
of one step, and per-phase device times of a 1-bit step with the ranks
re-aligned (host sync + dist.barrier) before every step.
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2411_16462_b200 as lc  # noqa: E402
from paper_2411_16462_b200 import _lib  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    tp = lc.NcclTransport.init_process(rank, world, dev)
    topo = lc.Topology(world, rank, tp)
    out = {"rank": rank}
    st = torch.cuda.current_stream()

    # (a) back-to-back barriers
    for _ in range(10):
        tp.device_barrier(rank, 0)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(200):
        tp.device_barrier(rank, 0)
    e1.record(st)
    torch.cuda.synchronize()
    out["barrier_us"] = e0.elapsed_time(e1) / 200 * 1e3

    # (b) a 1-bit step on n params, phases timed with ranks re-aligned
    n = int(os.environ.get("MB_N", str(64 << 20)))
    layout = lc.Layout({"w": (n,)})
    th = torch.randn(n, device=dev)
    m = torch.randn(n, device=dev) * 0.1
    g = torch.randn(n, device=dev)
    state = lc.WorkerState(params=layout.views(th), momentum=layout.views(m), iteration=0)
    gs = layout.views(g)
    h = lc.LionHyper(lr=1e-4)
    for _ in range(3):
        state = lc.distributed_lion_step(state, gs, h, None, topo, "compressed1bit")
    torch.cuda.synchronize()
    dist.barrier()
    host = []
    phases = {}
    steps = []
    for _ in range(10):
        torch.cuda.synchronize()
        dist.barrier()
        _lib.phase_events = {}
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        t0 = time.perf_counter()
        state = lc.distributed_lion_step(state, gs, h, None, topo, "compressed1bit")
        host.append(time.perf_counter() - t0)
        a1.record(st)
        torch.cuda.synchronize()
        steps.append(a0.elapsed_time(a1))
        for k, evs in _lib.phase_events.items():
            phases.setdefault(k, []).extend(a.elapsed_time(b) for a, b in evs)
        _lib.phase_events = None
    out["n"] = n
    out["host_enqueue_ms"] = sorted(host)[len(host) // 2] * 1e3
    out["step_ms_aligned"] = sorted(steps)[len(steps) // 2]
    out["phase_ms"] = {k: sum(v) / len(v) for k, v in phases.items()}

    # (c) free-running steps (no host sync between steps)
    torch.cuda.synchronize()
    dist.barrier()
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b0.record(st)
    t0 = time.perf_counter()
    for _ in range(20):
        state = lc.distributed_lion_step(state, gs, h, None, topo, "compressed1bit")
    t_host = time.perf_counter() - t0
    b1.record(st)
    torch.cuda.synchronize()
    out["step_ms_free"] = b0.elapsed_time(b1) / 20
    out["host_ms_per_step_free"] = t_host / 20 * 1e3
    print(json.dumps(out), flush=True)
    tp.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
