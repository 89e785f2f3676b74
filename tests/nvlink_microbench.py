"""NVLink peer-memory bandwidth probes with the library's own kernels
(torchrun, >= 2 GPUs, one process per GPU).

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tests/nvlink_microbench.py

* push: every rank stores its P blocks of an fp32 vector into the owners'
  slots (lc_push_blocks_f32) -- remote writes, (P-1)/P of the bytes;
* pull: every owner loads its block from all P ranks (lc_mean_pull_f32 with a
  local-only output) -- remote reads;
* mcast: every owner stores its block once to the NVLS multicast address
  (lc_mean_pull_f32 with P=1 source, nout=-1) -- multicast writes.
Rank 0 prints one JSON line of GB/s (bytes leaving/entering each GPU over
NVLink per second, max time over ranks).
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2411_16462_b200 as lc  # noqa: E402
from paper_2411_16462_b200 import _lib  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    tp = lc.NcclTransport.init_process(rank, world, dev)
    n = int(os.environ.get("NB_N", str(1 << 28)))
    s = -(-n // world)
    s = -(-s // 4) * 4
    src = torch.randn(n, device=dev)
    stage = tp.sym_buffer(rank, ("nb_stage",), world * s, torch.float32)
    vec = tp.sym_buffer(rank, ("nb", "momentum"), n, torch.float32)  # torch symm -> mc
    vec.local.copy_(src)
    st = torch.cuda.current_stream().cuda_stream
    res = {}

    def timed(name, fn, remote_bytes, reps=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = {"ms": float(t.item()), "GBps": remote_bytes / float(t.item()) / 1e6}

    dst = _lib.table([stage.peers[j] + rank * s * 4 for j in range(world)])
    timed("push", lambda: _lib.call("lc_push_blocks_f32", src.data_ptr(), n, s, dst, world, st),
          (world - 1) / world * n * 4)
    cnt = max(0, min(s, n - rank * s))
    local_out = _lib.table([vec.local.data_ptr()])
    timed("pull", lambda: _lib.call("lc_mean_pull_f32", _lib.table(vec.peers), world,
                                    rank * s, cnt, _lib.table([stage.local.data_ptr()]), 1, None, st),
          (world - 1) * cnt * 4)
    if vec.mc:
        timed("mcast", lambda: _lib.call("lc_mean_pull_f32", local_out, 1, rank * s, cnt,
                                         _lib.table([vec.mc]), -1, None, st), cnt * 4)
    # the fused sync's owner mean: P local staged rows -> fp32 mean stored into
    # every rank (k_sync_mean), at several grid sizes (CTAs per SM)
    work = torch.zeros(1, dtype=torch.int32, device=dev)
    mean_out = _lib.table([p + rank * s * 4 for p in vec.peers])
    cnt_m = max(0, min(s, n - rank * s))
    for cps in (1, 2, 4, 8):
        timed(f"sync_mean_cps{cps}", lambda c=cps: _lib.call(
            "lc_sync_mean", None, stage.local.data_ptr(), mean_out, world, s, cnt_m,
            work.data_ptr(), c, st), (world - 1) * cnt_m * 4)
    peers_out = _lib.table(vec.peers)
    timed("store_all", lambda: _lib.call("lc_mean_pull_f32", local_out, 1, rank * s, cnt,
                                         peers_out, world, None, st), (world - 1) * cnt * 4)
    if rank == 0:
        res["n"] = n
        res["world"] = world
        print(json.dumps(res), flush=True)
    tp.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
