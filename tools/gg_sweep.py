"""Sweep pipeline depth x persistent grid for the dense and gathered UP GEMM."""
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
B, d, D = 64, 4096, 16384
ws = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
x = torch.randn(B, d, device=dev).bfloat16()
out = torch.zeros(B, D, dtype=torch.bfloat16, device=dev)
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, D // 2, replace=False))).to(dev, torch.int32)
nit = pb.NeuronIndexTensor(0, idx, validate=False)
for stages, grid in [(4, 296), (2, 296), (3, 296), (8, 148), (6, 148), (4, 148), (8, 74)]:
    L.ps_debug_gemm_trace(None, stages, grid)
    f = lambda i: pk.gather_gemm_into(ws[i % 4], None, None, x, d, None, B, D, d, 0, out, D)  # noqa
    g = lambda i: pk.gather_gemm_into(ws[i % 4], nit.buffer, nit.count, x, d, None, B, D, d, 0, out, D)  # noqa
    try:
        ud = timeit(f, 10)
        ug = timeit(g, 10)
        print(f"stages={stages} grid={grid}: dense 134MB {ud:6.1f} us ({134.2e6 / ud / 1e3:5.0f} GB/s)   "
              f"gather 67MB {ug:6.1f} us ({67.1e6 / ug / 1e3:5.0f} GB/s)", flush=True)
    except Exception as e:
        print(stages, grid, "failed", e)
L.ps_debug_gemm_trace(None, 0, 0)
