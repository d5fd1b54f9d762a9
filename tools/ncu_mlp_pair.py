import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2505_14884_b200 import _lib
from paper_2505_14884_b200.kernels import PackedMLP, ROW_PAD, gather_gemm_into, gather_gemm_t_into
dev = torch.device("cuda")
B, d, D, S = 64, 4096, 16384, 6656
pk = PackedMLP((torch.randn(D, d, device=dev) * 0.02).bfloat16(), torch.zeros(D, device=dev),
               (torch.randn(D, d, device=dev) * 0.02).bfloat16(), torch.zeros(d, device=dev))
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, S, replace=False)).astype(np.int32)).to(dev)
idx = torch.cat([idx, idx[-1:].repeat(ROW_PAD)])
cnt = torch.full((1,), S, dtype=torch.int32, device=dev)
x = torch.randn(B, d, device=dev).bfloat16()
hid = torch.zeros(B, pk.D_pad, dtype=torch.bfloat16, device=dev)
out = torch.zeros(B, d, dtype=torch.float32, device=dev)
for i in range(4):
    gather_gemm_into(pk.w1t, idx, cnt, x, d, pk.b1, B, pk.D_pad, d, _lib.PS_ACT_RELU, hid, hid.stride(0), splits=S + 256, tag="gg_up")
    gather_gemm_t_into(pk.w2t, idx, cnt, hid, hid.stride(0), pk.b2, B, d, pk.D_pad, out, d, residual=out, res_ld=d, splits=S + 256, tag="gg_down", flags=_lib.PS_GG_A_READY)
torch.cuda.synchronize()
