"""mlp_into: bf16 vs f32 output, and shard-sum vs full (TP MLP partials)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2505_14884_b200 as pb
from paper_2505_14884_b200 import _lib
from paper_2505_14884_b200.kernels import PackedMLP, mlp_into, ROW_PAD, _round_up

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
for (B, d, D, k) in [(8, 256, 1024, 300), (8, 256, 512, 200), (64, 4096, 16384, 6000)]:
    w1 = (torch.randn(D, d, device=dev, generator=g) * 0.05).bfloat16()
    w2 = (torch.randn(D, d, device=dev, generator=g) * 0.05).bfloat16()
    b1 = torch.randn(D, device=dev, generator=g) * 0.05
    b2 = torch.randn(d, device=dev, generator=g) * 0.05
    x = torch.randn(B, d, device=dev, generator=g).bfloat16()
    ids = torch.randperm(D, device=dev, generator=g)[:k].sort().values.int()
    Dp = _round_up(D, ROW_PAD)
    idx = torch.full((Dp,), int(ids[-1]), dtype=torch.int32, device=dev); idx[:k] = ids
    cnt = torch.tensor([k], dtype=torch.int32, device=dev)
    pk = PackedMLP(w1, b1, w2, b2)
    hid = torch.zeros(B, Dp, dtype=torch.bfloat16, device=dev)
    o32 = torch.zeros(B, d, device=dev); o16 = torch.zeros(B, d, dtype=torch.bfloat16, device=dev)
    mlp_into(pk, x, idx, cnt, hid, o32)
    mlp_into(pk, x, idx, cnt, hid, o16)
    hr = torch.relu(x.float() @ w1[ids.long()].float().t() + b1[ids.long()]).bfloat16().float()
    ref = hr @ w2[ids.long()].float() + b2
    torch.cuda.synchronize()
    e32 = float((o32 - ref).norm() / ref.norm()); e16 = float((o16.float() - ref).norm() / ref.norm())
    print(B, d, D, k, "f32 rel", e32, "bf16 rel", e16, flush=True)
    # shard sum (2 shards, own neurons only, b2 on shard 0)
    tot = torch.zeros(B, d, device=dev)
    for r in range(2):
        lo, hi = r * D // 2, (r + 1) * D // 2
        sid = ids[(ids >= lo) & (ids < hi)] - lo
        kk = sid.numel()
        Dl = D // 2; Dlp = _round_up(Dl, ROW_PAD)
        idl = torch.full((Dlp,), int(sid[-1]), dtype=torch.int32, device=dev); idl[:kk] = sid
        cl = torch.tensor([kk], dtype=torch.int32, device=dev)
        pkl = PackedMLP(w1[lo:hi].contiguous(), b1[lo:hi].contiguous(), w2[lo:hi].contiguous(), b2 if r == 0 else torch.zeros_like(b2))
        hl = torch.zeros(B, Dlp, dtype=torch.bfloat16, device=dev)
        part = torch.zeros(B, d, dtype=torch.bfloat16, device=dev)
        mlp_into(pkl, x, idl, cl, hl, part)
        tot += part.float()
    torch.cuda.synchronize()
    print("   shard-sum rel", float((tot - ref).norm() / ref.norm()), flush=True)
