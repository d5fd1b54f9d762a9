"""Probe: torch symmetric memory across 2 processes on the SAME GPU (gloo group)."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
g = dist.group.WORLD
try:
    symm_mem.set_backend("CUDA")
except Exception as e:
    print("set_backend", e)
t = symm_mem.empty(1024, dtype=torch.float32, device="cuda")
t.fill_(rank + 1)
h = symm_mem.rendezvous(t, g.group_name)
print(rank, "world", h.world_size, "mc", h.multicast_ptr, "ptrs", h.buffer_ptrs, flush=True)
torch.cuda.synchronize()
dist.barrier()
peer = h.get_buffer(1 - rank, (1024,), torch.float32)
print(rank, "peer value", float(peer[0]), flush=True)
dist.barrier()
dist.destroy_process_group()
