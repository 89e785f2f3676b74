"""Selective momentum sync under both error modes, multi-process (a
diagnostic, not a test):

    torchrun --nproc-per-node 2 tests/repro_sync_modes.py [--mode deferred] [--steps 40]

Runs the GPT-2 layout with SyncPolicy(period=3, wte + lm-head-sized layers)
through the production peer-memory path and prints one progress line per
step on rank 0, then the max |m_r - m_0| over the synced layers."""

import argparse
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2411_16462_b200 as lc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="deferred")
    ap.add_argument("--steps", type=int, default=39)
    ap.add_argument("--workload", default="gpt2s_sumsigns")
    ap.add_argument("--algo", default="compressed1bit")
    ap.add_argument("--watch", type=float, default=30.0)
    ap.add_argument("--drain-sync", action="store_true")
    ap.add_argument("--timeout", type=float, default=20.0)
    args = ap.parse_args()
    os.environ["LIONCUB_ERRORS"] = args.mode
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    tp = lc.NcclTransport.init_process(rank, world, dev)
    tp.timeout = args.timeout
    topo = lc.Topology(world_size=world, rank=rank, transport=tp)
    shapes = bench.WORKLOADS[args.workload][0]()
    layout = lc.Layout(shapes)
    names = sorted(shapes, key=lambda k: -int(torch.tensor(shapes[k]).prod()))[:2]
    pol = lc.SyncPolicy(period=3, layers=frozenset(names))
    n = layout.n
    torch.manual_seed(rank)
    theta = torch.randn(n, device=dev)
    dist.broadcast(theta, 0)
    mom = torch.randn(n, device=dev)
    grad = torch.randn(n, device=dev)
    st = lc.WorkerState(params=layout.views(theta), momentum=layout.views(mom), iteration=0)
    g = layout.views(grad)
    h = lc.LionHyper(lr=1e-4)
    t0 = time.time()
    for i in range(args.steps):
        st = lc.distributed_lion_step(st, g, h, None, topo, args.algo, sync=pol)
        if args.drain_sync and pol.fires(st.iteration):
            torch.cuda.synchronize()
        if rank == 0:
            print(f"step {i + 1} enqueued {time.time() - t0:.3f}s", flush=True)
    ev = torch.cuda.Event()
    ev.record(topo.stream)
    t1 = time.time()
    while not ev.query() and time.time() - t1 < args.watch:
        time.sleep(0.01)
    if not ev.query():
        # stuck: read the barrier state through the copy engine on a side stream
        s2 = torch.cuda.Stream(dev)
        with torch.cuda.stream(s2):
            err = tp._err[rank].to("cpu", non_blocking=True)
            fl = tp._flags(rank).local.to("cpu", non_blocking=True)
            ctr = [(k[3], w.counters.to("cpu", non_blocking=True))
                   for k, w in st.params.workspace.items()]
        s2.synchronize()
        print(f"STUCK rank {rank}: host epoch {tp._epoch[rank]} flags {fl.tolist()} "
              f"err {err.tolist()} counters {[(k, c.tolist()) for k, c in ctr]}", flush=True)
        os._exit(3)
    torch.cuda.synchronize()
    if rank == 0:
        print(f"drained {time.time() - t0:.3f}s", flush=True)
    for k in names:
        x = st.momentum[k].contiguous()
        ref = x.clone()
        dist.broadcast(ref, 0)
        d = (x - ref).abs().max().item()
        if rank == 0 or d:
            print(f"rank {rank} layer {k} max|m - m_0| after step {st.iteration}: {d}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
