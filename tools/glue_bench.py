"""In-graph (CUDA graph replay) per-op times of the decode-step glue at the
bench shape: LayerNorm, KV append, head router(+append), cuBLAS projections,
router layers, SwiGLU.  Weights rotate over copies larger than L2."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib  # noqa
from tools.kbench import timeit  # noqa
dev = torch.device("cuda")
B, d, D, H = int(os.environ.get("B", 64)), 4096, 16384, 32
L = _lib.load()
st = lambda: _lib.stream_ptr()  # noqa
x = torch.randn(B, d, device=dev)
h = torch.empty(B, d, dtype=torch.bfloat16, device=dev)
g, bta = torch.ones(d, device=dev), torch.zeros(d, device=dev)
res = []
def rep(name, us):
    res.append((name, us)); print(f"{name:44s} {us:7.1f} us", flush=True)
rep("layernorm", timeit(lambda i: L.ps_layernorm(x.data_ptr(), d, g.data_ptr(), bta.data_ptr(), B, d, h.data_ptr(), d, st()), 20))
rep("add_layernorm", timeit(lambda i: L.ps_add_layernorm(x.data_ptr(), d, bta.data_ptr(), g.data_ptr(), bta.data_ptr(), B, d, h.data_ptr(), d, st()), 20))
n = 6
wq = [(torch.randn(3 * d, d, device=dev) * 0.02).bfloat16() for _ in range(n)]
bq = torch.zeros(3 * d, device=dev).bfloat16()
qkv = torch.empty(B, 3 * d, dtype=torch.bfloat16, device=dev)
rep("QKV cuBLAS addmm (100 MB)", timeit(lambda i: torch.addmm(bq, h, wq[i % n].t(), out=qkv), 20))
wo = [(torch.randn(d, d, device=dev) * 0.02).bfloat16() for _ in range(n)]
attn = torch.randn(B, d, device=dev).bfloat16()
rep("O-proj cuBLAS addmm residual f32 (33 MB)", timeit(lambda i: torch.addmm(x, attn, wo[i % n].t(), out_dtype=torch.float32, out=x), 20))
c = pb.KVCache(B, H, 64, 128, device=dev)
kq, vq = qkv[:, d:], qkv[:, 2 * d:]
def app(i):
    if i % 16 == 0:
        c.lengths.zero_()
    L.ps_kv_append(c.keys.data_ptr(), c.values.data_ptr(), c.lengths.data_ptr(), kq.data_ptr(), vq.data_ptr(), 3 * d, B, H, 64, 128, c._err.data_ptr(), st())
rep("kv_append", timeit(app, 16))
hr = pb.HeadRouter(d, H, seed=1, device=dev)
sel = torch.empty(B, 16, dtype=torch.int32, device=dev)
rep("head_router_topk", timeit(lambda i: hr.select_into(h, 16, sel), 20))
def hra(i):
    if i % 16 == 0:
        c.lengths.zero_()
    hr.select_append_into(h, 16, sel, c, kq, vq, 3 * d)
rep("head_router_topk_append", timeit(hra, 16))
win = [(torch.randn(1024, d, device=dev) * 0.02).bfloat16() for _ in range(n)]
bin_ = torch.zeros(1024, device=dev).bfloat16()
rhid = torch.empty(B, 1024, dtype=torch.bfloat16, device=dev)
rep("router W_in cuBLAS relu (8 MB)", timeit(lambda i: torch._addmm_activation(bin_, h, win[i % n].t(), out=rhid), 20))
wout = [(torch.randn(D, 1024, device=dev) * 0.02).bfloat16() for _ in range(n)]
lg = torch.empty(B, D, device=dev)
rep("router W_out cuBLAS f32 (33 MB)", timeit(lambda i: torch.mm(rhid, wout[i % n].t(), out_dtype=torch.float32, out=lg), 20))
