"""Stages x grid sweep for the LSU-fed gathered UP/DOWN GEMM (B=64, |S|=D/2)."""
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
d, D, B = 4096, 16384, int(os.environ.get('B', 64))
ws = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, D // 2, replace=False))).to(dev, torch.int32)
nit = pb.NeuronIndexTensor(0, idx, validate=False)
x = torch.randn(B, d, device=dev).bfloat16()
out = torch.zeros(B, D, dtype=torch.bfloat16, device=dev)
h = torch.randn(B, D, device=dev).bfloat16()
y = torch.zeros(B, d, dtype=torch.float32, device=dev)
for stages, grid in [(0, 0), (3, 296), (2, 296), (4, 148), (5, 148), (6, 148), (7, 148)]:
    L.ps_debug_gemm_trace(None, stages, grid)
    g = lambda i: pk.gather_gemm_into(ws[i % 4], nit.buffer, nit.count, x, d, None, B, D, d, 0, out, D, splits=D // 2)  # noqa
    dn = lambda i: pk.gather_gemm_t_into(ws[i % 4], nit.buffer, nit.count, h, D, None, B, d, D, y, d, splits=D // 2, flags=1)  # noqa
    try:
        ug, un = timeit(g, 10), timeit(dn, 10)
        print(f"stages={stages} grid={grid}: UP gather {ug:6.1f} us ({67.1e6 / ug / 1e3:5.0f} GB/s)  DOWN gather "
              f"{un:6.1f} us ({67.1e6 / un / 1e3:5.0f} GB/s)", flush=True)
    except Exception as e:
        print(stages, grid, "failed:", e, flush=True)
L.ps_debug_gemm_trace(None, 0, 0)
