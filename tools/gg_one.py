"""Run one dense and one gathered UP launch (for ncu captures)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa
dev = torch.device("cuda")
B, d, D = 64, 4096, 16384
w = (torch.randn(D, d, device=dev) * 0.02).bfloat16()
x = torch.randn(B, d, device=dev).bfloat16()
hidden = torch.zeros(B, D, dtype=torch.bfloat16, device=dev)
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, D // 2, replace=False))).to(dev, torch.int32)
nit = pb.NeuronIndexTensor(0, idx, validate=False)
for _ in range(3):
    pk.gather_gemm_into(w, None, None, x, d, None, B, D, d, 1, hidden, D)
    pk.gather_gemm_into(w, nit.buffer, nit.count, x, d, None, B, D, d, 1, hidden, D)
torch.cuda.synchronize()
