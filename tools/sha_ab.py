"""A/B of the SHA kernel: this tree's libpolar_b200.so vs another build of
the library (``tools/micro/libpolar_r01.so`` by default: the round-1
kernel whose tile count came from the host hint), same process, same
caches (rotated over buffers larger than L2), graph-replayed.

    python tools/sha_ab.py [other.so]
"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200 import _lib  # noqa: E402
from tools.kbench import timeit  # noqa: E402

other = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tools", "micro", "libpolar_r01.so")
OTHER = ctypes.CDLL(other)
for n in ("ps_sha_workspace_bytes", "ps_sha_decode"):
    getattr(OTHER, n).restype, getattr(OTHER, n).argtypes = _lib.SIGNATURES[n]
NEW = _lib.load()
dev = torch.device("cuda")
for (B, H, H_kv, ctx, kh) in [(64, 32, 32, 1920, 16), (64, 32, 32, 1920, 32), (256, 32, 8, 1920, 4),
                              (1, 32, 32, 1920, 16), (16, 32, 32, 1920, 16)]:
    n = 4
    caches = []
    for i in range(n):
        c = pb.KVCache(B, H_kv, ctx + 64, 128, device=dev)
        c.fill_random(i, ctx)
        caches.append(c)
    q = torch.randn(B, H * 128, device=dev).bfloat16()
    out = torch.empty(B, H * 128, dtype=torch.bfloat16, device=dev)
    sel = torch.stack([torch.randperm(H_kv, device=dev)[:kh].sort().values for _ in range(B)]).to(torch.int32)
    nb = B * kh * ctx * 128 * 4
    res = []
    for name, L in (("new", NEW), ("r01", OTHER), ("new", NEW)):
        nbytes = L.ps_sha_workspace_bytes(B, H, H_kv, 128, kh, 0)
        ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev)

        def f(i, L=L, ws=ws, nbytes=nbytes):
            c = caches[i % n]
            rc = L.ps_sha_decode(q.data_ptr(), H * 128, c.keys.data_ptr(), c.values.data_ptr(), c.lengths.data_ptr(),
                                 sel.data_ptr(), 0, B, H, H_kv, c.capacity, 128, kh, 0.088, 0, ctx + 1,
                                 out.data_ptr(), H * 128, 1, ws.data_ptr(), nbytes,
                                 torch.cuda.current_stream().cuda_stream)
            assert rc == 0, rc
        us = timeit(f, 16)
        res.append(f"{name}: {us:6.1f}us {nb / us / 1e3:5.0f}GB/s")
    print(f"B={B} H_kv={H_kv} k={kh} ctx={ctx}: " + "  ".join(res), flush=True)
