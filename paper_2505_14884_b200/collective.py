"""Peer-memory all-reduce fused with the residual add.

``P2PAllReduce`` gives every tensor-parallel rank two bf16 partial buffers
(alternating from call to call) and an inbox of flags, maps every rank's
buffers into every other rank's address space with CUDA IPC (the handles
travel over the process group with ``all_gather_object``), and runs
``ps_allreduce_add_bf16``: one launch that waits for every rank's partial
(flags + a device epoch, so it replays inside CUDA graphs) and adds the sum
into the f32 residual stream.  It replaces ``dist.all_reduce(part)`` +
``x.add_(part)`` after the O- and down-projections (parallel.py).

On one node the IPC mappings are NVLink peer memory; ranks sharing one GPU
(the tests) map the same device.  The group only carries the handles, so a
gloo group is enough.
"""

from __future__ import annotations

import torch

from . import _lib


def _share(t: torch.Tensor):
    from torch.multiprocessing.reductions import reduce_tensor

    return reduce_tensor(t)


def _open(shared):
    fn, args = shared
    return fn(*args)


class P2PAllReduce:
    MAX_WORLD = 8

    def __init__(self, group, rank: int, world: int, numel: int, device):
        if not 1 <= world <= self.MAX_WORLD:
            raise ValueError(f"P2PAllReduce supports 1..{self.MAX_WORLD} ranks, got {world}")
        self.rank, self.world, self.numel = rank, world, numel
        dev = torch.device(device)
        self.bufs = [torch.zeros(numel, dtype=torch.bfloat16, device=dev) for _ in range(2)]
        self.inbox = torch.zeros(self.MAX_WORLD, dtype=torch.int32, device=dev)
        self.state = torch.zeros(4, dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)
        mine = (_share(self.bufs[0]), _share(self.bufs[1]), _share(self.inbox))
        if world > 1:
            import torch.distributed as dist

            allh = [None] * world
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        self._peers = []  # keep the mapped peer tensors alive
        ptr_slots = [[], []]
        flag_ptrs = []
        for r, h in enumerate(allh):
            if r == rank:
                b0, b1, ib = self.bufs[0], self.bufs[1], self.inbox
            else:
                b0, b1, ib = _open(h[0]), _open(h[1]), _open(h[2])
                self._peers += [b0, b1, ib]
            ptr_slots[0].append(b0.data_ptr())
            ptr_slots[1].append(b1.data_ptr())
            flag_ptrs.append(ib.data_ptr())
        self.buf_ptrs = [torch.tensor(p, dtype=torch.int64, device=dev) for p in ptr_slots]
        self.flag_ptrs = torch.tensor(flag_ptrs, dtype=torch.int64, device=dev)
        self._call = 0
        if world > 1:
            import torch.distributed as dist

            dist.barrier(group=group)

    def next_buffer(self, shape) -> torch.Tensor:
        """The bf16 buffer the next call reduces (write the partial here)."""
        n = 1
        for s in shape:
            n *= int(s)
        if n > self.numel:
            raise ValueError(f"partial of {n} elements exceeds the {self.numel}-element buffers")
        return self.bufs[self._call % 2][:n].view(*shape)

    def add_into(self, x: torch.Tensor) -> None:
        """x (f32 (B, d)) += sum over ranks of their current partials."""
        B, d = x.shape
        slot = self._call % 2
        self._call += 1
        _lib.call("ps_allreduce_add_bf16", _lib.ptr(self.buf_ptrs[slot]), _lib.ptr(self.flag_ptrs),
                  _lib.ptr(self.inbox), _lib.ptr(self.state), self.rank, self.world, B, d, _lib.ptr(x),
                  x.stride(0), _lib.stream_ptr())
