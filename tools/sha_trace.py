"""Per-CTA timeline of the SHA tensor-core kernel (ps_debug_sha_trace) at the
OPT-6.7B decode shape (B=64, 32 groups, ctx 1920): polar (16 of 32) and
dense, inside a CUDA graph of 3 launches over rotating caches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa: E402

dev = torch.device("cuda")
L = _lib.load()
B, H, ctx = int(os.environ.get("B", 64)), 32, 1920
caches = []
for i in range(3):
    c = pb.KVCache(B, H, ctx + 1, 128, device=dev)
    c.fill_random(i, ctx)
    caches.append(c)
q = torch.randn(B, H * 128, device=dev).bfloat16()
out = torch.empty(B, H * 128, dtype=torch.bfloat16, device=dev)
bufs = [torch.zeros(8 * 4096, dtype=torch.int64, device=dev) for _ in range(3)]
for kh in (16, 32):
    g = torch.Generator(device=dev).manual_seed(0)
    sel = torch.stack([torch.randperm(H, device=dev, generator=g)[:kh].sort().values for _ in range(B)]).int()

    def f(i, tr=True):
        if tr:
            L.ps_debug_sha_trace(bufs[i].data_ptr())
        pk.sha_decode_into(q, H * 128, caches[i], sel, H, 0.088, out, H * 128, max_len_hint=ctx)
        L.ps_debug_sha_trace(None)
    for i in range(3):
        f(i, False)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(gr, stream=st):
        for i in range(3):
            f(i)
    torch.cuda.current_stream().wait_stream(st)
    gr.replay()
    torch.cuda.synchronize()
    for b in bufs:
        b.zero_()
    gr.replay()
    torch.cuda.synchronize()
    t = bufs[1].view(-1, 8).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    work = t[t[:, 3] > 0]
    print(f"k={kh}: {len(t)} CTAs ({len(work)} stream-K), span {(t[:, 1:].max() - t0) / 1e3:.1f} us")
    for j, nm in [(0, "start"), (1, "dep wait"), (2, "partition"), (4, "1st tile"), (3, "end")]:
        v = work[:, j]
        v = v[v > 0]
        d = (v - t0) / 1e3
        print(f"   {nm:10s} min {d.min():8.2f} p10 {np.percentile(d, 10):8.2f} med {np.median(d):8.2f} "
              f"p90 {np.percentile(d, 90):8.2f} max {d.max():8.2f}")
    # which CTAs form the tail?  (rows are indexed by blockIdx; the first B
    # stream-K CTAs also zero the unselected heads of sequence bid)
    rows = bufs[1].view(-1, 8).cpu().numpy()
    bid = np.arange(len(rows))
    ok = (rows[:, 0] > 0) & (rows[:, 3] > 0)
    end = (rows[:, 3] - t0) / 1e3
    part = (rows[:, 2] - t0) / 1e3
    zf = ok & (bid < B)
    nz = ok & (bid >= B)
    print(f"   zero-fill CTAs (bid < {B}): partition med {np.median(part[zf]):.2f} end med {np.median(end[zf]):.2f} "
          f"max {end[zf].max():.2f} | others: partition med {np.median(part[nz]):.2f} end med "
          f"{np.median(end[nz]):.2f} max {end[nz].max():.2f}")
    late = np.argsort(end * ok)[-12:]
    print("   latest CTAs (bid:end):", " ".join(f"{i}:{end[i]:.1f}" for i in late))
