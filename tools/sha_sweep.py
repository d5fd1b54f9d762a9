"""Split-count sweep of the SHA kernel at decode shapes (graph replay over
rotating caches larger than L2)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import kernels as pk  # noqa
from tools.kbench import timeit  # noqa
dev = torch.device("cuda")
if os.environ.get("PS_PDL") == "0":
    from paper_2505_14884_b200 import _lib as _l  # noqa: E402
    _l.load().ps_set_pdl(0)
import ctypes  # noqa: E402
_old = os.path.join(os.path.dirname(os.path.abspath(__file__)), "micro", "libsha_old.so")
OLD = ctypes.CDLL(_old) if os.path.exists(_old) else None
if OLD is not None:
    from paper_2505_14884_b200 import _lib  # noqa: E402
    for _n in ("ps_sha_workspace_bytes", "ps_sha_decode"):
        getattr(OLD, _n).restype, getattr(OLD, _n).argtypes = _lib.SIGNATURES[_n]
for (B, H, H_kv, ctx, ks) in ([(int(b), 32, 8, 1920, (4, 8)) for b in os.environ["SWEEP_B"].split(",")] if os.environ.get("SWEEP_B") else [(64, 32, 32, 1920, (16,)), (256, 32, 8, 1920, (4, 8)), (64, 32, 8, 1920, (4, 8))]):
    n = 2 if B >= 512 else 4
    caches = []
    for i in range(n):
        c = pb.KVCache(B, H_kv, ctx + 1, 128, device=dev)
        c.fill_random(i, ctx)
        caches.append(c)
    q = torch.randn(B, H * 128, device=dev).bfloat16()
    out = torch.empty(B, H * 128, dtype=torch.bfloat16, device=dev)
    for kh in ks:
        sel = torch.stack([torch.randperm(H_kv, device=dev)[:kh].sort().values for _ in range(B)]).to(torch.int32)
        nb = B * kh * ctx * 128 * 4
        res = []
        for s in (0, 1, 2, -444, -888):
            f = lambda i: pk.sha_decode_into(q, H * 128, caches[i % n], sel, H, 0.088, out, H * 128, num_splits=s,  # noqa
                                             max_len_hint=ctx)
            us = timeit(f, 12)
            res.append(f"s={s or 'auto'}:{us:6.1f}us/{nb / us / 1e3:5.0f}")
        print(f"B={B} H_kv={H_kv} k={kh} ctx={ctx}: " + "  ".join(res), flush=True)
        if False and OLD is not None:  # the previous (per-unit split) kernel, same process / box
            res = []
            for sp in (1, 2, 3, 4):
                nbytes = OLD.ps_sha_workspace_bytes(B, H, H_kv, 128, kh, sp)
                ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
                g = lambda i: OLD.ps_sha_decode(q.data_ptr(), H * 128, caches[i % n].keys.data_ptr(),  # noqa
                                                caches[i % n].values.data_ptr(), caches[i % n].lengths.data_ptr(),
                                                sel.data_ptr(), 0, B, H, H_kv, ctx + 1, 128, kh, 0.088,
                                                sp, ctx, out.data_ptr(), H * 128, 1, ws.data_ptr(),
                                                nbytes, torch.cuda.current_stream().cuda_stream)
                us = timeit(g, 12)
                res.append(f"s={sp}:{us:6.1f}us/{nb / us / 1e3:5.0f}")
            print("   old kernel: " + "  ".join(res), flush=True)
