import os, sys, ctypes
import torch
sys.path.insert(0, "/root/repo")
import paper_2505_14884_b200 as pb
from paper_2505_14884_b200 import _lib, kernels as pk
dev = torch.device("cuda")
OLD = ctypes.CDLL("tools/micro/libsha_old.so")
for _n in ("ps_sha_workspace_bytes", "ps_sha_decode"):
    getattr(OLD, _n).restype, getattr(OLD, _n).argtypes = _lib.SIGNATURES[_n]
B, H, H_kv, ctx, kh = 64, 32, 32, 1920, 32
c = pb.KVCache(B, H_kv, ctx + 1, 128, device=dev); c.fill_random(0, ctx)
q = torch.randn(B, H * 128, device=dev).bfloat16()
out = torch.empty(B, H * 128, dtype=torch.bfloat16, device=dev)
sel = torch.arange(H_kv, device=dev, dtype=torch.int32).repeat(B, 1).contiguous()
for _ in range(2):
    pk.sha_decode_into(q, H * 128, c, sel, H, 0.088, out, H * 128, num_splits=1, max_len_hint=ctx)
    nb = OLD.ps_sha_workspace_bytes(B, H, H_kv, 128, kh, 1)
    ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
    OLD.ps_sha_decode(q.data_ptr(), H * 128, c.keys.data_ptr(), c.values.data_ptr(), c.lengths.data_ptr(), sel.data_ptr(),
                      0, B, H, H_kv, ctx + 1, 128, kh, 0.088, 1, ctx, out.data_ptr(), H * 128, 1, ws.data_ptr(), nb,
                      torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
