"""Selective MLP and router MLP timing: one chained launch (ps_sparse_mlp /
ps_router_mlp) vs the two-launch tcgen05 path (mlp_into) vs cuBLAS, inside a
CUDA graph of L launches over 8 distinct weight sets (inputs >> L2).

    python tools/chain_bench.py [--batches 1,16,64,128,256] [--union 0.4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2505_14884_b200 import MlpRouter  # noqa: E402
from paper_2505_14884_b200.kernels import PackedMLP, ROW_PAD, _round_up, mlp_into, sparse_mlp_into  # noqa: E402


def graph_time(fn, L, reps=5):
    s = torch.cuda.Stream()
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(L):
                fn(i)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / L)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,16,64,128,256")
    ap.add_argument("--union", type=float, default=0.4)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--D", type=int, default=16384)
    ap.add_argument("--L", type=int, default=32)
    ap.add_argument("--router", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda")
    d, D, L = a.d, a.D, a.L
    g = torch.Generator(device=dev).manual_seed(0)
    mlps = [PackedMLP((torch.randn(D, d, device=dev, generator=g) * 0.02).bfloat16(),
                      torch.randn(D, device=dev, generator=g) * 0.02,
                      (torch.randn(D, d, device=dev, generator=g) * 0.02).bfloat16(),
                      torch.zeros(d, device=dev)) for _ in range(8)]
    Dp = _round_up(D, ROW_PAD)
    for B in [int(b) for b in a.batches.split(",")]:
        k = int(a.union * D)
        ids = torch.randperm(D, device=dev, generator=g)[:k].sort().values.int()
        idx = torch.full((Dp,), int(ids[-1]), dtype=torch.int32, device=dev)
        idx[:k] = ids
        cnt = torch.tensor([k], dtype=torch.int32, device=dev)
        x = torch.randn(B, d, device=dev, generator=g).bfloat16()
        hid = torch.zeros(B, Dp, dtype=torch.bfloat16, device=dev)
        out = torch.zeros(B, d, device=dev)
        byt = 2 * k * d * 2 + 2 * B * d * 2 + B * d * 8
        t_chain = graph_time(lambda i: sparse_mlp_into(mlps[i % 8], x, idx, cnt, hid, out, residual=out), L)
        t_two = graph_time(lambda i: mlp_into(mlps[i % 8], x, idx, cnt, hid, out, residual=out, expected=k), L)
        print(f"MLP B={B:4d} |S|={k}: chain {t_chain:7.1f} us ({byt / t_chain / 1e3:6.0f} GB/s)   "
              f"two-launch {t_two:7.1f} us ({byt / t_two / 1e3:6.0f} GB/s)", flush=True)
    if a.router:
        rs = [MlpRouter.random_device(d, D, seed=i, device=dev) for i in range(8)]
        for B in [int(b) for b in a.batches.split(",")]:
            x = torch.randn(B, d, device=dev, generator=g).bfloat16()
            h = rs[0].hidden_dim_
            hid = torch.zeros(B, h, dtype=torch.bfloat16, device=dev)
            lg = torch.zeros(B, D, device=dev)
            byt = (d * h + h * D) * 2 + B * D * 4
            t_chain = graph_time(lambda i: rs[i % 8].logits_into(x, hid, lg, with_bias=False), L)
            t_two = graph_time(lambda i: rs[i % 8].logits_into(x, hid, lg, with_bias=False, fused=False), L)

            def cub(i):
                r = rs[i % 8]
                torch._addmm_activation(r.b_in.bfloat16(), x, r.w_in_t.t(), out=hid)
                torch.mm(hid, r.w_out_t.t(), out_dtype=torch.float32, out=lg)
            t_cub = graph_time(cub, L)
            print(f"router B={B:4d}: chain {t_chain:6.1f} us ({byt / t_chain / 1e3:5.0f} GB/s)  two-launch "
                  f"{t_two:6.1f} us  cuBLAS {t_cub:6.1f} us", flush=True)


if __name__ == "__main__":
    main()
