"""Probe torch SymmetricMemory / NVLS multicast on this box (torchrun, N ranks)."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
grp = dist.group.WORLD
print(rank, "backend", symm_mem.get_backend(dev) if hasattr(symm_mem, "get_backend") else "?", flush=True)
t = symm_mem.empty(1 << 20, dtype=torch.float32, device=dev)
h = symm_mem.rendezvous(t, grp.group_name)
attrs = [a for a in dir(h) if not a.startswith("_")]
print(rank, "attrs", attrs, flush=True)
print(rank, "multicast_ptr", getattr(h, "multicast_ptr", None), "buffer_ptrs", getattr(h, "buffer_ptrs", None)[:4] if hasattr(h, "buffer_ptrs") else None,
      "signal_pad_ptrs", (getattr(h, "signal_pad_ptrs", None) or [])[:2], "signal_pad_size", getattr(h, "signal_pad_size", None), flush=True)
dist.barrier()
dist.destroy_process_group()
