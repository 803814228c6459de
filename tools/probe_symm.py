"""Probe: does torch symmetric memory give a multicast (NVLS) pointer on this box with 1 rank?"""
import os
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
try:
    import torch.distributed._symmetric_memory as symm_mem
    t = symm_mem.empty(1024, dtype=torch.int32, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print("symm ok; multicast_ptr", getattr(h, "multicast_ptr", None), "buffer ptrs", getattr(h, "buffer_ptrs", None))
    print("has_multicast_support", symm_mem.has_multicast_support if hasattr(symm_mem, "has_multicast_support") else "n/a")
except Exception as e:
    print("symm failed:", repr(e))
dist.destroy_process_group()
