"""Gathered / dense GEMM timings vs batch (cluster split-K kernel) next to cuBLAS."""
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
d, D = 4096, 16384
ws = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
for frac in (0.5, 0.25, 0.1):
    k = int(frac * D)
    idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, k, replace=False))).to(dev, torch.int32)
    nit = pb.NeuronIndexTensor(0, idx, validate=False)
    for B in (16, 64, 256):
        x = torch.randn(B, d, device=dev).bfloat16()
        out = torch.zeros(B, D, dtype=torch.bfloat16, device=dev)
        h = torch.randn(B, D, device=dev).bfloat16()
        y = torch.zeros(B, d, dtype=torch.float32, device=dev)
        f = lambda i: pk.gather_gemm_into(ws[i % 4], None, None, x, d, None, B, D, d, 0, out, D)  # noqa
        g = lambda i: pk.gather_gemm_into(ws[i % 4], nit.buffer, nit.count, x, d, None, B, D, d, 0, out, D, splits=k)  # noqa
        dn = lambda i: pk.gather_gemm_t_into(ws[i % 4], nit.buffer, nit.count, h, D, None, B, d, D, y, d, splits=k)  # noqa
        c = lambda i: torch.matmul(x, ws[i % 4].t())  # noqa
        ud, ug, un, uc = timeit(f, 10), timeit(g, 10), timeit(dn, 10), timeit(c, 10)
        wb = k * d * 2 / 1e3
        print(f"|S|/D={frac:.2f} B={B:3d}: UP dense {ud:6.1f} us ({134.2e3 / ud:5.0f} GB/s) | UP gather {ug:6.1f} us "
              f"({wb / ug:5.0f} GB/s) | DOWN gather {un:6.1f} us ({wb / un:5.0f} GB/s) | cuBLAS dense {uc:6.1f} us",
              flush=True)
