"""Dense / gathered UP GEMM time vs batch (B-operand bytes per stage)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kbench import timeit  # noqa
dev = torch.device("cuda")
d, D = 4096, 16384
ws = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, D // 2, replace=False))).to(dev, torch.int32)
nit = pb.NeuronIndexTensor(0, idx, validate=False)
for B in (16, 32, 64, 128, 256):
    x = torch.randn(B, d, device=dev).bfloat16()
    out = torch.zeros(B, D, dtype=torch.bfloat16, device=dev)
    f = lambda i: pk.gather_gemm_into(ws[i % 4], None, None, x, d, None, B, D, d, 0, out, D)  # noqa
    g = lambda i: pk.gather_gemm_into(ws[i % 4], nit.buffer, nit.count, x, d, None, B, D, d, 0, out, D)  # noqa
    c = lambda i: torch.matmul(x, ws[i % 4].t())  # noqa
    ud, ug, uc = timeit(f, 10), timeit(g, 10), timeit(c, 10)
    print(f"B={B:4d}: dense {ud:6.1f} us ({134.2e6 / ud / 1e3:5.0f} GB/s)  gather-50% {ug:6.1f} us "
          f"({67.1e6 / ug / 1e3:5.0f} GB/s)  cuBLAS {uc:6.1f} us ({134.2e6 / uc / 1e3:5.0f} GB/s)", flush=True)
