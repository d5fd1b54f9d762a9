"""Per-kernel micro-benchmark at a decode shape (CUDA events, L2-cold
weights via per-iteration buffer rotation).

    python tools/kbench.py [--batch 64] [--d 4096] [--D 16384] [--union 0.5] [--only gg]
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa: E402


def timeit(fn, iters=20, warm=3, graph=True):
    """Device time per call (us).  The calls are captured into one CUDA graph
    and replayed, so host launch overhead (ctypes, tensor-map encode) is not
    measured -- exactly how the decode step runs."""
    for _ in range(warm):
        fn(0)
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=st):
            for i in range(iters):
                fn(i)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    if graph:
        g.replay()
    else:
        for i in range(iters):
            fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--D", type=int, default=16384)
    ap.add_argument("--union", type=float, default=0.5)
    ap.add_argument("--copies", type=int, default=6)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--splits-up", type=int, default=0)
    ap.add_argument("--splits-down", type=int, default=0)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    dev = torch.device("cuda")
    B, d, D = a.batch, a.d, a.D
    n = a.copies  # rotate weight copies so every iteration streams from HBM
    rows = []

    def rep(name, us, nbytes):
        rows.append((name, us, nbytes / (us * 1e-6) / 1e9))
        print(f"{name:40s} {us:9.1f} us  {nbytes / 1e6:9.1f} MB  {nbytes / (us * 1e-6) / 1e9:8.1f} GB/s", flush=True)

    x = torch.randn(B, d, device=dev).bfloat16()
    if not a.only or "gg" in a.only:
        mlps = [pb.PackedMLP((torch.randn(D, d, device=dev) * 0.02).bfloat16(), torch.zeros(D, device=dev),
                             (torch.randn(D, d, device=dev) * 0.02).bfloat16(), torch.zeros(d, device=dev))
                for _ in range(n)]
        k = int(a.union * D)
        idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, k, replace=False))).to(dev, torch.int32)
        nit = pb.NeuronIndexTensor(0, idx, validate=False)
        hidden = torch.empty(B, mlps[0].D_pad, dtype=torch.bfloat16, device=dev)
        y = torch.empty(B, d, dtype=torch.float32, device=dev)
        up = lambda i: pk.gather_gemm_into(mlps[i % n].w1t, nit.buffer, nit.count, x, d, mlps[i % n].b1, B,  # noqa
                                           mlps[0].D_pad, d, _lib.PS_ACT_RELU, hidden, hidden.stride(0),
                                           splits=a.splits_up)
        down = lambda i: pk.gather_gemm_t_into(mlps[i % n].w2t, nit.buffer, nit.count, hidden, hidden.stride(0),  # noqa
                                               mlps[i % n].b2, B, d, mlps[0].D_pad, y, d, splits=a.splits_down)
        wb = k * d * 2
        rep(f"gather_gemm UP   |S|={k}", timeit(up, a.iters), wb + B * d * 2 + B * k * 2)
        rep(f"gather_gemm DOWN |S|={k}", timeit(down, a.iters), wb + B * k * 2 + B * d * 4)
        ar = torch.arange(k, dtype=torch.int32, device=dev)
        nit_ar = pb.NeuronIndexTensor(0, ar, validate=False)
        up_ar = lambda i: pk.gather_gemm_into(mlps[i % n].w1t, nit_ar.buffer, nit_ar.count, x, d, None, B,  # noqa
                                              mlps[0].D_pad, d, _lib.PS_ACT_RELU, hidden, hidden.stride(0))
        rep(f"gather_gemm UP gather4 of rows 0..{k}", timeit(up_ar, a.iters), wb)
        up_dk = lambda i: pk.gather_gemm_into(mlps[i % n].w1t, None, None, x, d, None, B, k, d,  # noqa
                                              _lib.PS_ACT_RELU, hidden, hidden.stride(0))
        rep(f"gather_gemm UP dense tiles M={k}", timeit(up_dk, a.iters), wb)
        dense_up = lambda i: pk.gather_gemm_into(mlps[i % n].w1t, None, None, x, d, mlps[i % n].b1, B, D, d,  # noqa
                                                 _lib.PS_ACT_RELU, hidden, hidden.stride(0), splits=a.splits_up)
        rep(f"gather_gemm UP dense D={D}", timeit(dense_up, a.iters), D * d * 2)
        # cuBLAS reference point for the same dense weight stream
        ws = [m.w1t for m in mlps]
        cub = lambda i: torch.matmul(x, ws[i % n].t())  # noqa
        rep(f"cuBLAS x @ W1 (dense D={D})", timeit(cub, a.iters), D * d * 2)
    if not a.only or "sha" in a.only:
        H, ctx = 32, 1920
        caches = []
        for i in range(n):
            c = pb.KVCache(B, H, ctx + 1, 128, device=dev)
            c.fill_random(i, ctx)
            caches.append(c)
        q = torch.randn(B, H * 128, device=dev).bfloat16()
        out = torch.empty(B, H * 128, dtype=torch.bfloat16, device=dev)
        for kh in (16, 32):
            sel = torch.stack([torch.randperm(H, device=dev)[:kh].sort().values for _ in range(B)]).to(torch.int32)
            f = lambda i: pk.sha_decode_into(q, H * 128, caches[i % n], sel, H, 0.088, out, H * 128)  # noqa
            nb = B * kh * ctx * 128 * 4
            rep(f"sha_decode k={kh}/{H} ctx={ctx}", timeit(f, a.iters), nb)
    if not a.only or "sel" in a.only:
        logits = torch.randn(B, D, device=dev)
        nb = int(_lib.load().ps_select_union_workspace_bytes(B, D))
        ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
        buf = torch.empty(D, dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int32, device=dev)
        st = lambda: _lib.stream_ptr()  # noqa
        f = lambda i: _lib.call("ps_select_union", logits.data_ptr(), None, B, D, D, int(a.union * D), 0.0, ws.data_ptr(),  # noqa
                                nb, 0, D, 128, buf.data_ptr(), cnt.data_ptr(), st())
        rep(f"select_union (topk+union+compact) {B}x{D} k={int(a.union * D)}", timeit(f, a.iters), B * D * 4)
        hr = pb.HeadRouter(d, 32, seed=1)
        sel = torch.empty(B, 16, dtype=torch.int32, device=dev)
        h = lambda i: hr.select_into(x, 16, sel)  # noqa
        rep("head_router_topk d x 32", timeit(h, a.iters), d * 32 * 2 + B * d * 2)


if __name__ == "__main__" and "--trace" not in sys.argv:
    main()


def trace_main():
    """python tools/kbench.py --trace: per-CTA timeline of one UP / DOWN launch."""
    ap = argparse.ArgumentParser()
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--D", type=int, default=16384)
    ap.add_argument("--union", type=float, default=0.5)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--target", type=int, default=0)
    ap.add_argument("--splits", type=int, default=0)
    a = ap.parse_args()
    dev = torch.device("cuda")
    B, d, D = a.batch, a.d, a.D
    L = _lib.load()
    buf = torch.zeros(16 * 4000, dtype=torch.int64, device=dev)
    w = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
    x = torch.randn(B, d, device=dev).bfloat16()
    k = int(a.union * D)
    idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, k, replace=False))).to(dev, torch.int32)
    nit = pb.NeuronIndexTensor(0, idx, validate=False)
    hidden = torch.zeros(B, D, dtype=torch.bfloat16, device=dev)
    y = torch.empty(B, d, dtype=torch.float32, device=dev)
    runs = {
        "UP sparse": lambda i: pk.gather_gemm_into(w[i % 4], nit.buffer, nit.count, x, d, None, B, D, d, 1, hidden, D,
                                                   splits=a.splits),
        "UP dense": lambda i: pk.gather_gemm_into(w[i % 4], None, None, x, d, None, B, D, d, 1, hidden, D,
                                                  splits=a.splits),
        "DOWN sparse": lambda i: pk.gather_gemm_t_into(w[i % 4], nit.buffer, nit.count, hidden, D, None, B, d, D, y, d,
                                                       splits=a.splits),
    }
    for name, fn in runs.items():
        L.ps_debug_gemm_trace(None, a.stages, a.target)
        us = timeit(fn, 10)
        buf.zero_()
        L.ps_debug_gemm_trace(buf.data_ptr(), a.stages, a.target)
        fn(1)
        torch.cuda.synchronize()
        L.ps_debug_gemm_trace(None, 0, 0)
        t = buf.view(-1, 8).cpu().numpy()
        t = t[t[:, 5] > 0]
        t0 = t[:, 0].min()
        rel = (t[:, :6] - t0) / 1e3
        its = t[:, 6]
        print(f"{name}: {us:.1f} us/launch (graph), CTAs={len(t)}  traced span={rel[:, 5].max():.1f} us  "
              f"SMs={len(np.unique(t[:, 7]))}")
        print("   start max %.2f | setup med %.2f | first stage med %.2f | MMA loop med %.1f max %.1f | "
              "epi-end med %.1f max %.1f" % (rel[:, 0].max(), np.median(rel[:, 1] - rel[:, 0]),
                                              np.median(rel[:, 2] - rel[:, 1]), np.median(rel[:, 3] - rel[:, 2]),
                                              (rel[:, 3] - rel[:, 2]).max(), np.median(rel[:, 5] - rel[:, 3]),
                                              (rel[:, 5] - rel[:, 3]).max()))
        per = (rel[:, 3] - rel[:, 2]) / np.maximum(its - 1, 1)
        print("   iters/CTA med %d  us/iter med %.3f -> per-CTA %.1f GB/s (A operand)" %
              (np.median(its), np.median(per), 16384 / (np.median(per) * 1e-6) / 1e9))


if __name__ == "__main__" and "--trace" in sys.argv:
    trace_main()
    sys.exit(0)
