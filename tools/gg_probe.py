"""Probe fixed per-launch cost and epilogue tail of the gathered GEMM."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kbench import timeit  # noqa
dev = torch.device("cuda")
L = _lib.load()
B = 64
for (M, K) in [(128, 64), (128, 4096), (1024, 4096), (4096, 4096), (16384, 4096)]:
    ws = [(torch.randn(M, K, device=dev) * 0.02).bfloat16() for _ in range(4)]
    x = torch.randn(B, K, device=dev).bfloat16()
    out = torch.zeros(B, M, dtype=torch.bfloat16, device=dev)
    f = lambda i: pk.gather_gemm_into(ws[i % 4], None, None, x, K, None, B, M, K, 0, out, M)  # noqa
    us = timeit(f, 20)
    c = lambda i: torch.matmul(x, ws[i % 4].t())  # noqa
    uc = timeit(c, 20)
    buf = torch.zeros(16 * 400, dtype=torch.int64, device=dev)
    L.ps_debug_gemm_trace(buf.data_ptr(), 0, 0)
    f(1)
    torch.cuda.synchronize()
    L.ps_debug_gemm_trace(None, 0, 0)
    t = buf.view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    epi = t[:, 4][t[:, 4] > 0]
    mma = t[:, 3][t[:, 3] > 0]
    w = t[t[:, 8] > 0]
    if len(w):
        print("   first segment: acc ready - last MMA issue med %.2f | drain med %.2f | finish med %.2f us" % (
            np.median(w[:, 8] - w[:, 3]) / 1e3, np.median(w[:, 9] - w[:, 8]) / 1e3, np.median(w[:, 10] - w[:, 9]) / 1e3))
    print(f"M={M:6d} K={K}: ours {us:7.1f} us  cuBLAS {uc:6.1f} us | CTAs {len(t)} | last MMA issue "
          f"{(mma.max() - t0) / 1e3 if len(mma) else -1:.1f} us | last epilogue done {(epi.max() - t0) / 1e3 if len(epi) else -1:.1f} us",
          flush=True)
