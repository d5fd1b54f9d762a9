"""Probe: torch symmetric memory + NVLS multicast with a world-size-1 NCCL group."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29531")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
g = dist.group.WORLD
print("backend", symm_mem.get_backend(torch.device("cuda")) if hasattr(symm_mem, "get_backend") else "?")
try:
    symm_mem.enable_symm_mem_for_group(g.group_name)
except Exception as e:
    print("enable:", e)
t = symm_mem.empty(64 * 4096, dtype=torch.bfloat16, device="cuda")
h = symm_mem.rendezvous(t, g)
print("rank", h.rank, "world", h.world_size)
for a in ("multicast_ptr", "buffer_ptrs_dev", "signal_pad_ptrs_dev", "buffer_ptrs", "signal_pad_ptrs", "signal_pad_size"):
    try:
        print(a, getattr(h, a))
    except Exception as e:
        print(a, "ERR", e)
print("mc supported attr:", torch.cuda.get_device_properties(0))
dist.destroy_process_group()
