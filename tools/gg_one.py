"""A tiny dense launch and a sparse-MLP-shaped UP/DOWN pair (for ncu captures)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa
dev = torch.device("cuda")
B, d, D = 64, 4096, 16384
w = (torch.randn(D, d, device=dev) * 0.02).bfloat16()
b1 = torch.randn(D, device=dev) * 0.02
x = torch.randn(B, d, device=dev).bfloat16()
hidden = torch.zeros(B, D, dtype=torch.bfloat16, device=dev)
y = torch.zeros(B, d, dtype=torch.float32, device=dev)
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, D // 2, replace=False))).to(dev, torch.int32)
nit = pb.NeuronIndexTensor(0, idx, validate=False)
wt = w[:128, :64].contiguous()
xt = x[:, :64].contiguous()
ot = torch.zeros(B, 128, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    pk.gather_gemm_into(wt, None, None, xt, 64, None, B, 128, 64, 0, ot, 128)
    pk.gather_gemm_into(w, nit.buffer, nit.count, x, d, b1, B, D, d, 1, hidden, D)
    pk.gather_gemm_t_into(w, nit.buffer, nit.count, hidden, D, None, B, d, D, y, d, residual=y, res_ld=d)
torch.cuda.synchronize()
