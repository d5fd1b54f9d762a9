"""Gap analysis of back-to-back gathered-GEMM launches inside one CUDA graph:
per-CTA globaltimer stamps (ps_debug_gemm_trace) of two consecutive launches."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa
from paper_2505_14884_b200 import _lib, kernels as pk  # noqa
dev = torch.device("cuda")
L = _lib.load()
B, d, D = int(os.environ.get("B", 64)), 4096, 16384
ws = [(torch.randn(D, d, device=dev) * 0.02).bfloat16() for _ in range(4)]
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, D // 2, replace=False))).to(dev, torch.int32)
nit = pb.NeuronIndexTensor(0, idx, validate=False)
x = torch.randn(B, d, device=dev).bfloat16()
hid = torch.zeros(B, D, dtype=torch.bfloat16, device=dev)
y = torch.zeros(B, d, dtype=torch.float32, device=dev)
bufs = [torch.zeros(16 * 4096, dtype=torch.int64, device=dev) for _ in range(4)]
up = lambda i: pk.gather_gemm_into(ws[i % 4], nit.buffer, nit.count, x, d, None, B, D, d, 1, hid, D)  # noqa
dn = lambda i: pk.gather_gemm_t_into(ws[i % 4], nit.buffer, nit.count, hid, D, None, B, d, D, y, d)  # noqa
for stages, target in [(0, 0), (7, 148)]:
    seq = [up, dn, up, dn]
    for i, f in enumerate(seq):
        L.ps_debug_gemm_trace(None, stages, target)
        f(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=st):
        for i, f in enumerate(seq):
            L.ps_debug_gemm_trace(bufs[i].data_ptr(), stages, target)
            f(i)
    L.ps_debug_gemm_trace(None, 0, 0)
    for b in bufs:
        b.zero_()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    tot = s.elapsed_time(e) * 1e3
    ts = [b.view(-1, 16).cpu().numpy() for b in bufs]
    ts = [t[t[:, 0] > 0] for t in ts]
    t0 = ts[0][:, 0].min()
    print(f"stages={stages} target={target}: graph of 4 launches {tot:.1f} us")
    for i, t in enumerate(ts):
        rel = (t[:, :10].astype(np.int64) - t0) / 1e3
        print(f"  launch {i} ({'UP' if i % 2 == 0 else 'DOWN'}): CTAs={len(t)} start min {rel[:, 0].min():6.1f} max {rel[:, 0].max():6.1f} | "
              f"setup med {np.median(rel[:, 1]):6.1f} | 1st stage med {np.median(rel[:, 2][t[:, 2] > 0]):6.1f} | "
              f"MMA done med {np.median(rel[:, 3][t[:, 3] > 0]):6.1f} max {rel[:, 3][t[:, 3] > 0].max():6.1f} | "
              f"epi done max {rel[:, 4][t[:, 4] > 0].max():6.1f} | end max {rel[:, 5].max():6.1f}")
        rr = (t[:, :16].astype(np.int64) - t0) / 1e3
        ok = t[:, 13] > 0
        if ok.any():
            dd = lambda a, b: np.median(rr[ok, b] - rr[ok, a])  # noqa
            print(f"     epilogue (median deltas, us): MMA-issued->acc-ready {dd(3, 8):.2f} | TMEM->stg {dd(8, 10):.2f} | "
                  f"rdy wait {dd(10, 11):.2f} | reduce+store {dd(11, 12):.2f} | fre wait {dd(12, 13):.2f} | ->end {dd(13, 5):.2f}")
