"""One launch of every remaining libpolar kernel at a bench shape, for an ncu
metrics capture (profiles/r01_ncu_other_kernels.csv): LayerNorm, embed, KV
append (contiguous and paged), SwiGLU, the small-batch gathered GEMV, paged
SHA, the paged fused head-router append, and the threshold / union kernels."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa
dev = torch.device("cuda")
L = _lib.load()
st = _lib.stream_ptr
B, d, D, H, Hkv, dh, ctx = 64, 4096, 16384, 32, 32, 128, 1920
x = torch.randn(B, d, device=dev)
g, b_ = torch.ones(d, device=dev), torch.zeros(d, device=dev)
h = torch.empty(B, d, dtype=torch.bfloat16, device=dev)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
_lib.call("ps_add_layernorm", _lib.ptr(x), d, None, _lib.ptr(g), _lib.ptr(b_), B, d, _lib.ptr(h), d, st())
emb = torch.randn(50272, d, device=dev).bfloat16()
pos = torch.randn(2048, d, device=dev).bfloat16()
tok = torch.randint(0, 50272, (B,), dtype=torch.int32, device=dev)
c = pb.KVCache(B, Hkv, ctx + 8, dh, device=dev)
c.fill_random(0, ctx)
_lib.call("ps_embed", _lib.ptr(tok), _lib.ptr(c.lengths), _lib.ptr(emb), _lib.ptr(pos), B, d, _lib.ptr(x), st())
kn = torch.randn(B, Hkv, dh, device=dev).bfloat16()
c.append_step(kn, kn)
pc = pb.PagedKVCache.from_contiguous(c, page_rows=64, seed=1)
pc.append_step(kn, kn)
gu = torch.randn(B, 2 * 14336, device=dev).bfloat16()
hid = torch.empty(B, 14336, dtype=torch.bfloat16, device=dev)
_lib.call("ps_swiglu", _lib.ptr(gu), gu.stride(0), B, 14336, _lib.ptr(hid), hid.stride(0), st())
w1t = (torch.randn(D, d, device=dev) * 0.02).bfloat16()
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, D // 2, replace=False))).to(dev, torch.int32)
nit = pb.NeuronIndexTensor(0, idx, validate=False)
x2 = torch.randn(2, d, device=dev).bfloat16()
hid2 = torch.empty(2, D + 128, dtype=torch.bfloat16, device=dev)
pk.gather_gemm_into(w1t, nit.buffer, nit.count, x2, d, None, 2, D + 128, d, _lib.PS_ACT_RELU, hid2, D + 128,
                    splits=D // 2)
q = torch.randn(B, H * dh, device=dev).bfloat16()
out = torch.empty(B, H * dh, dtype=torch.bfloat16, device=dev)
sel = torch.stack([torch.randperm(Hkv, device=dev)[:16].sort().values for _ in range(B)]).to(torch.int32)
pk.sha_decode_into(q, H * dh, pc, sel, H, 0.088, out, H * dh, max_len_hint=ctx + 2)
hr = pb.HeadRouter(d, Hkv, seed=1)
sel2 = torch.empty(B, 16, dtype=torch.int32, device=dev)
qkv = torch.randn(B, 3 * d, device=dev).bfloat16()
for b in range(B):
    pc.reserve(b, int(pc.host_lengths[b]) + 1)
hr.select_append_into(h, 16, sel2, pc, qkv[:, d:], qkv[:, 2 * d:], qkv.stride(0))
lg = torch.randn(B, D, device=dev)
pb.union_from_logits(lg, threshold=2.0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
