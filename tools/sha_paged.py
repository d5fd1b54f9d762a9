"""SHA kernel time, contiguous vs paged caches (same contents), at decode shapes."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import kernels as pk  # noqa
from tools.kbench import timeit  # noqa
dev = torch.device("cuda")
for (B, H, H_kv, ctx, kh) in [(64, 32, 32, 1920, 16), (256, 32, 8, 1920, 4), (64, 32, 32, 1920, 32)]:
    n = 3
    caches = []
    for i in range(n):
        c = pb.KVCache(B, H_kv, ctx + 64, 128, device=dev)
        c.fill_random(i, ctx)
        caches.append(c)
    q = torch.randn(B, H * 128, device=dev).bfloat16()
    out = torch.empty(B, H * 128, dtype=torch.bfloat16, device=dev)
    sel = torch.stack([torch.randperm(H_kv, device=dev)[:kh].sort().values for _ in range(B)]).to(torch.int32)
    nb = B * kh * ctx * 128 * 4
    res = [f"B={B} H_kv={H_kv} k={kh}:"]
    f = lambda i: pk.sha_decode_into(q, H * 128, caches[i % n], sel, H, 0.088, out, H * 128, max_len_hint=ctx)  # noqa
    us = timeit(f, 12)
    res.append(f"contig {us:6.1f}us/{nb / us / 1e3:5.0f}GB/s")
    for P in (int(x) for x in os.environ.get("PAGES", "32,64,256").split(",")):
        for shuffled in ((True,) if os.environ.get("PAGES") else (False, True)):
            pcs = [pb.PagedKVCache.from_contiguous(c, page_rows=P, seed=(7 if shuffled else None)) for c in caches]
            g = lambda i: pk.sha_decode_into(q, H * 128, pcs[i % n], sel, H, 0.088, out, H * 128, max_len_hint=ctx)  # noqa
            us = timeit(g, 12)
            res.append(f"P={P}{'s' if shuffled else 'o'} {us:6.1f}us/{nb / us / 1e3:5.0f}")
            del pcs
    print("  ".join(res), flush=True)
    del caches
    torch.cuda.empty_cache()
