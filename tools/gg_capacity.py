"""Where do the split-K clusters stop being co-resident?  DOWN (C = 8) time
vs output tiles M/128, UP (C = 4) time vs union tiles, B = 64; a jump in time
per tile marks a second wave of clusters.  Graph-replayed, L2-cold weights."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kbench import timeit  # noqa
dev = torch.device("cuda")
B, D = 64, 16384
S = 6272
idx = torch.from_numpy(np.sort(np.random.default_rng(1).choice(D, S, replace=False))).to(dev, torch.int32)
nit = pb.NeuronIndexTensor(0, idx, validate=False)
h = torch.randn(B, D + 128, device=dev).bfloat16()
for M in (2048, 3072, 3584, 3840, 3968, 4096, 4224, 4608):
    w2 = [(torch.randn(D, M, device=dev) * 0.02).bfloat16() for _ in range(4)]
    out = torch.zeros(B, M, dtype=torch.float32, device=dev)
    dn = lambda i: pk.gather_gemm_t_into(w2[i % 4], nit.buffer, nit.count, h, h.stride(0), None, B, M, D + 128,  # noqa
                                         out, M, splits=S, tag="gc_dn", flags=_lib.PS_GG_A_READY)
    t = timeit(dn, 20)
    print(f"DOWN M={M} tiles={M // 128}: {t:6.1f} us  ({t / (M // 128):5.2f} us/tile)", flush=True)
    del w2
d = 4096
w1 = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
x = torch.randn(B, d, device=dev).bfloat16()
out_up = torch.zeros(B, D + 128, dtype=torch.bfloat16, device=dev)
for T in (52, 56, 60, 62, 64, 66, 68, 72):
    S2 = T * 128
    idx2 = torch.from_numpy(np.sort(np.random.default_rng(T).choice(D, S2, replace=False))).to(dev, torch.int32)
    nit2 = pb.NeuronIndexTensor(0, idx2, validate=False)
    up = lambda i: pk.gather_gemm_into(w1[i % 4], nit2.buffer, nit2.count, x, d, None, B, D + 128, d, 1, out_up,  # noqa
                                       out_up.stride(0), splits=S2, tag="gc_up")
    t = timeit(up, 20)
    print(f"UP tiles={T}: {t:6.1f} us  ({t / T:5.2f} us/tile)", flush=True)
