"""Probe: does torch symmetric memory give an NVLS multicast address here?"""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
try:
    symm_mem.enable_symm_mem_for_group(dist.group.WORLD.group_name)
except Exception as e:
    print("enable:", e)
print("backend", symm_mem.get_backend(torch.device("cuda", rank)) if hasattr(symm_mem, "get_backend") else None)
t = symm_mem.empty(1 << 20, dtype=torch.uint8, device=f"cuda:{rank}")
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print(rank, "mc", getattr(h, "multicast_ptr", None), "has_mc", getattr(h, "has_multicast_support", None),
      "ptrs", list(h.buffer_ptrs), "sig", getattr(h, "signal_pad_ptrs", None) is not None,
      [a for a in dir(h) if not a.startswith("_")])
dist.destroy_process_group()
