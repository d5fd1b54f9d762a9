"""SHA throughput vs head density and CTA count (OPT-6.7B decode shape:
B=64, H=H_kv=32, d_h=128, ctx 1920), graph replays over rotating caches
(> L2).  GB/s = algorithmic K+V bytes / time."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200 import kernels as pk  # noqa: E402
from tools.kbench import timeit  # noqa: E402

dev = torch.device("cuda")
B, H, ctx = int(os.environ.get("B", 64)), 32, 1920
H_kv = int(os.environ.get("H_KV", 32))
caches = []
for i in range(3):
    c = pb.KVCache(B, H_kv, ctx + 1, 128, device=dev)
    c.fill_random(i, ctx)
    caches.append(c)
q = torch.randn(B, H * 128, device=dev).bfloat16()
out = torch.empty(B, H * 128, dtype=torch.bfloat16, device=dev)
cases = [(H_kv, "dense"), (H_kv // 2, "random")] if os.environ.get("SHORT") else \
    [(32, "dense"), (16, "random"), (16, "first half"), (16, "strided")]
for kh, how in cases:
    if how == "random":
        g = torch.Generator(device=dev).manual_seed(0)
        sel = torch.stack([torch.randperm(H_kv, device=dev, generator=g)[:kh].sort().values for _ in range(B)])
    elif how == "strided":
        sel = torch.arange(0, H, 2, device=dev).repeat(B, 1)
    else:
        sel = torch.arange(kh, device=dev).repeat(B, 1)
    sel = sel.to(torch.int32).contiguous()
    nb = B * kh * ctx * 128 * 4
    res = []
    for s in [int(v) for v in os.environ.get('SPLITS', '0,-148,-296,-444,-592').split(',')]:
        f = lambda i: pk.sha_decode_into(q, H * 128, caches[i % 3], sel, H, 0.088, out, H * 128,  # noqa: E731
                                         num_splits=s, max_len_hint=ctx)
        us = timeit(f, 12)
        res.append(f"{s or 'auto'}:{us:6.1f}us {nb / us / 1e3:5.0f}GB/s")
    print(f"k={kh:2d} {how:10s}: " + "  ".join(res), flush=True)
