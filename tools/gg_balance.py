"""Gathered UP / DOWN time vs union size at B=64 (tiles x cluster = CTAs):
does the per-SM balance of the split-K clusters set the streaming rate?
Graph-replayed launches, 4 rotating weight sets (L2-cold), CUDA events."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kbench import timeit  # noqa
dev = torch.device("cuda")
B, d, D = int(os.environ.get("GB_B", 64)), 4096, 16384
w1 = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
w2 = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
x = torch.randn(B, d, device=dev).bfloat16()
h = torch.randn(B, D + 128, device=dev).bfloat16()
out_up = torch.zeros(B, D + 128, dtype=torch.bfloat16, device=dev)
out_dn = torch.zeros(B, d, dtype=torch.float32, device=dev)
L = _lib.load()
tgt = int(os.environ.get("GB_TARGET", 0))
if tgt:
    L.ps_debug_gemm_trace(None, 0, tgt)
    print("CTA slot target", tgt)
for S in [int(v) for v in os.environ.get("GB_S", "4736 4864 6272 6400 8192 9472").split()]:
    idx = torch.from_numpy(np.sort(np.random.default_rng(S).choice(D, S, replace=False))).to(dev, torch.int32)
    nit = pb.NeuronIndexTensor(0, idx, validate=False)
    up = lambda i: pk.gather_gemm_into(w1[i % 4], nit.buffer, nit.count, x, d, None, B, D + 128, d, 1, out_up,  # noqa
                                       out_up.stride(0), splits=S, tag="gb_up")
    dn = lambda i: pk.gather_gemm_t_into(w2[i % 4], nit.buffer, nit.count, h, h.stride(0), None, B, d, D + 128,  # noqa
                                         out_dn, d, splits=S, tag="gb_dn", flags=_lib.PS_GG_A_READY)
    tu, td = timeit(up, 20), timeit(dn, 20)
    mb = S * d * 2 / 1e6
    print(f"|S|={S:5d} tiles={-(-S // 128):3d}: UP {tu:6.1f} us ({mb / tu:5.2f} TB/s)  DOWN {td:6.1f} us "
          f"({mb / td:5.2f} TB/s)", flush=True)
