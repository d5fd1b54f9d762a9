"""Reconcile per-launch GEMM timings: single launches vs graph replay."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa
dev = torch.device("cuda")
B, d, D = 64, 4096, 16384
ws = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
x = torch.randn(B, d, device=dev).bfloat16()
hidden = torch.zeros(B, D, dtype=torch.bfloat16, device=dev)
L = _lib.load()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa
for grid in (0, 148, 74):
    L.ps_debug_gemm_trace(None, 0, grid)
    f = lambda i: pk.gather_gemm_into(ws[i % 4], None, None, x, d, None, B, D, d, 1, hidden, D)  # noqa
    for i in range(3):
        f(i)
    torch.cuda.synchronize()
    single = []
    for i in range(6):
        s, e = ev(), ev()
        torch.cuda.synchronize()
        s.record(); f(i); e.record()
        torch.cuda.synchronize()
        single.append(s.elapsed_time(e) * 1e3)
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=st):
        for i in range(8):
            f(i)
    g.replay(); torch.cuda.synchronize()
    s, e = ev(), ev()
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    print(f"grid={grid or 'default'}: single launches (us) {np.round(single, 1).tolist()}  graph avg {s.elapsed_time(e) * 1e3 / 8:.1f}")
    s, e = ev(), ev()
    s.record()
    for i in range(8):
        torch.matmul(x, ws[i % 4].t())
    e.record(); torch.cuda.synchronize()
    print(f"   cuBLAS eager avg {s.elapsed_time(e) * 1e3 / 8:.1f} us")
