"""Small-batch gathered UP GEMV (gemv_up_kernel, N <= 4) timed alone with CUDA
events: |S| gathered rows of a (D, d) bf16 matrix, rotating over enough
matrices that nothing is L2-resident, 200 launches replayed from a CUDA graph.  Prints us per launch and
the algorithmic HBM rate (|S| * d * 2 bytes per launch).

    PS_LIB_PATH=tools/micro/libpolar_oldgemv.so python tools/gemv_bench.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa: E402

dev = torch.device("cuda")


def run(N, d, D, rows, n_mats=8, iters=200):
    ws = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(n_mats)]
    rng = np.random.default_rng(0)
    nits = [pb.NeuronIndexTensor(0, torch.from_numpy(np.sort(rng.choice(D, rows, replace=False))).to(dev, torch.int32),
                                 validate=False) for _ in range(n_mats)]
    x = torch.randn(N, d, device=dev).bfloat16()
    out = torch.empty(N, D + 128, dtype=torch.bfloat16, device=dev)

    def one(i):
        pk.gather_gemm_into(ws[i % n_mats], nits[i % n_mats].buffer, nits[i % n_mats].count, x, d, None, N, D, d,
                            _lib.PS_ACT_RELU, out, out.stride(0), splits=rows)

    for i in range(20):
        one(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()  # launches from a graph: the host is not the bound
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=st):
        for i in range(iters):
            one(i)
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    gbs = rows * d * 2 / (us * 1e-6) / 1e9
    print(f"N={N} d={d} D={D} rows={rows}: {us:.2f} us/launch, {gbs:.0f} GB/s")


if __name__ == "__main__":
    print("lib:", os.environ.get("PS_LIB_PATH", "in-tree"))
    for N, d, D, rows in [(1, 4096, 16384, 1638), (1, 4096, 16384, 4096), (2, 4096, 16384, 2600),
                          (4, 4096, 16384, 3500), (1, 9216, 36864, 3686), (1, 8192, 28672, 2867)]:
        run(N, d, D, rows)
