"""SHA with group_base on a local cache slice vs the full SHA; select_union [lo,hi) vs full."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2505_14884_b200 as pb
from paper_2505_14884_b200 import _lib
from paper_2505_14884_b200.kernels import sha_decode_into, ROW_PAD, _round_up

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
for (B, H, H_kv, d_h, N, k, world) in [(8, 8, 8, 32, 256, 4, 2), (8, 8, 2, 32, 256, 1, 2), (8, 32, 8, 128, 256, 4, 2),
                                       (8, 8, 8, 32, 256, 8, 2)]:
    G = H // H_kv
    full = pb.KVCache(B, H_kv, N + 8, d_h, device=dev)
    full.keys.copy_(torch.randn(full.keys.shape, device=dev, generator=g).bfloat16())
    full.values.copy_(torch.randn(full.values.shape, device=dev, generator=g).bfloat16())
    full.set_lengths([N] * B)
    q = torch.randn(B, H * d_h, device=dev, generator=g).bfloat16()
    sel = torch.stack([torch.randperm(H_kv, device=dev, generator=g)[:k].sort().values for _ in range(B)]).int()
    out = torch.zeros(B, H * d_h, dtype=torch.bfloat16, device=dev)
    sha_decode_into(q, H * d_h, full, sel, H, 0.1, out, H * d_h, max_len_hint=N + 1)
    torch.cuda.synchronize()
    hl = H_kv // world
    for r in range(world):
        loc = pb.KVCache(B, hl, N + 8, d_h, device=dev)
        loc.keys.copy_(full.keys[:, r * hl:(r + 1) * hl])
        loc.values.copy_(full.values[:, r * hl:(r + 1) * hl])
        loc.set_lengths([N] * B)
        ql = q[:, r * hl * G * d_h:(r + 1) * hl * G * d_h].contiguous()
        ol = torch.full((B, hl * G * d_h), 7.0, dtype=torch.bfloat16, device=dev)
        sha_decode_into(ql, ql.shape[1], loc, sel, hl * G, 0.1, ol, ol.shape[1], group_base=r * hl, max_len_hint=N + 1)
        torch.cuda.synchronize()
        ref = out[:, r * hl * G * d_h:(r + 1) * hl * G * d_h]
        print(B, H, H_kv, d_h, k, "rank", r, "max|d|", float((ol.float() - ref.float()).abs().max()), flush=True)

# select_union [lo, hi)
L = _lib.load()
for (rows, cols, k, lo, hi) in [(8, 1024, 128, 0, 512), (8, 1024, 128, 512, 1024), (64, 16384, 1638, 8192, 16384)]:
    lg = torch.randn(rows, cols, device=dev, generator=g)
    nb = int(L.ps_select_union_workspace_bytes(rows, cols))
    ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
    idx = torch.zeros(_round_up(cols, ROW_PAD), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("ps_select_union", _lib.ptr(lg), None, rows, cols, cols, k, 0.0, _lib.ptr(ws), nb, lo, hi, ROW_PAD,
              _lib.ptr(idx), _lib.ptr(cnt), _lib.stream_ptr())
    torch.cuda.synchronize()
    top = torch.topk(lg, k, dim=1).indices
    u = torch.unique(top)
    u = u[(u >= lo) & (u < hi)] - lo
    c = int(cnt.item())
    print("union", rows, cols, k, lo, hi, "count", c, "ref", u.numel(), "eq", bool(c == u.numel() and torch.equal(idx[:c].long(), u)), flush=True)
