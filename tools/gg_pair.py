"""One gathered UP and one DOWN launch of the bench's sparse-MLP shape at
batch B (env B, default 256; |S| = D/2), after a warm-up pair -- for ncu."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import kernels as pk  # noqa
dev = torch.device("cuda")
B, d, D = int(os.environ.get("B", 256)), 4096, 16384
w1 = (torch.randn(D, d, device=dev) * 0.02).bfloat16()
w2 = (torch.randn(D, d, device=dev) * 0.02).bfloat16()
b1 = torch.randn(D, device=dev) * 0.02
x = torch.randn(B, d, device=dev).bfloat16()
hidden = torch.zeros(B, D + 128, dtype=torch.bfloat16, device=dev)
y = torch.zeros(B, d, dtype=torch.float32, device=dev)
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, D // 2, replace=False))).to(dev, torch.int32)
nit = pb.NeuronIndexTensor(0, idx, validate=False)
for _ in range(2):
    pk.gather_gemm_into(w1, nit.buffer, nit.count, x, d, b1, B, D + 128, d, 1, hidden, D + 128, splits=D // 2)
    pk.gather_gemm_t_into(w2, nit.buffer, nit.count, hidden, D + 128, None, B, d, D + 128, y, d, residual=y,
                          res_ld=d, splits=D // 2, flags=1)
torch.cuda.synchronize()
