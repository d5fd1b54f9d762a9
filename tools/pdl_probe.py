"""Does PDL overlap consecutive libpolar launches?  Builds short launch
sequences (select_union -> UP -> DOWN, with and without a cuBLAS GEMM in
front), eagerly and inside a CUDA graph, and prints each traced kernel's CTA
start window against its predecessor's end (globaltimer stamps)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14884_b200 import _lib, _ws  # noqa: E402
from paper_2505_14884_b200.kernels import PackedMLP, ROW_PAD, mlp_into  # noqa: E402

dev = torch.device("cuda")
L = _lib.load()
B, d, D, k = 64, 4096, 16384, 1638
g = torch.Generator(device=dev)
g.manual_seed(0)
logits = torch.randn(B, D, device=dev, generator=g)
logits[:, torch.randperm(D, device=dev, generator=g)[:1180]] += 6.0
pk = PackedMLP((torch.randn(D, d, device=dev) * 0.02).bfloat16(), torch.zeros(D, device=dev),
               (torch.randn(D, d, device=dev) * 0.02).bfloat16(), torch.zeros(d, device=dev))
x = (torch.randn(B, d, device=dev)).bfloat16()
hid = torch.zeros(B, pk.D_pad, dtype=torch.bfloat16, device=dev)
out = torch.zeros(B, d, dtype=torch.float32, device=dev)
idx = torch.zeros(D + ROW_PAD, dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int32, device=dev)
nb = int(L.ps_select_union_workspace_bytes(B, D))
sws = torch.zeros(nb, dtype=torch.uint8, device=dev)
wr = (torch.randn(D, 1024, device=dev) * 0.02).bfloat16()
rh = torch.randn(B, 1024, device=dev).bfloat16()
bufs = {}


POOL = [torch.zeros(16 * 2048, dtype=torch.int64, device=dev) for _ in range(64)]


def tb(name):
    b = POOL.pop()  # preallocated: no memset node inside the capture
    bufs.setdefault(name, []).append(b)
    return b


def seq(with_mm, traced, parts=("topk", "up", "down"), a_ready=True):
    from paper_2505_14884_b200.kernels import gather_gemm_into, gather_gemm_t_into
    if "topk" not in parts:
        if traced:
            L.ps_debug_gemm_trace(tb("up").data_ptr(), 0, 0)
        gather_gemm_into(pk.w1t, idx, cnt, x, d, pk.b1, B, pk.D_pad, d, _lib.PS_ACT_RELU, hid, hid.stride(0),
                         splits=7000, tag="gg_up")
        if traced:
            L.ps_debug_gemm_trace(tb("down").data_ptr(), 0, 0)
        gather_gemm_t_into(pk.w2t, idx, cnt, hid, hid.stride(0), pk.b2, B, d, pk.D_pad, out, d, splits=7000,
                           tag="gg_down", flags=_lib.PS_GG_A_READY if a_ready else 0)
        L.ps_debug_gemm_trace(None, 0, 0)
        return
    if with_mm:
        torch.mm(rh, wr.t(), out_dtype=torch.float32, out=logits)
    if traced:
        L.ps_debug_topk_trace(tb("topk").data_ptr())
    _lib.call("ps_select_union", logits.data_ptr(), None, B, D, D, k, 0.0, sws.data_ptr(), nb, 0, D, ROW_PAD,
              idx.data_ptr(), cnt.data_ptr(), _lib.stream_ptr())
    L.ps_debug_topk_trace(None)
    if traced:
        L.ps_debug_gemm_trace(tb("up").data_ptr(), 0, 0)
    from paper_2505_14884_b200.kernels import gather_gemm_into, gather_gemm_t_into
    gather_gemm_into(pk.w1t, idx, cnt, x, d, pk.b1, B, pk.D_pad, d, _lib.PS_ACT_RELU, hid, hid.stride(0),
                     splits=7000, tag="gg_up")
    if traced:
        L.ps_debug_gemm_trace(tb("down").data_ptr(), 0, 0)
    gather_gemm_t_into(pk.w2t, idx, cnt, hid, hid.stride(0), pk.b2, B, d, pk.D_pad, out, d, splits=7000,
                       tag="gg_down", flags=_lib.PS_GG_A_READY)
    L.ps_debug_gemm_trace(None, 0, 0)


def report(label):
    tk, up, dn = bufs["topk"][-1], bufs["up"][-1], bufs["down"][-1]
    t = tk.view(-1, 16).cpu().numpy(); t = t[t[:, 0] > 0]
    u = up.view(-1, 16).cpu().numpy(); u = u[u[:, 0] > 0]
    w = dn.view(-1, 16).cpu().numpy(); w = w[w[:, 0] > 0]
    t0 = t[:, 0].min()
    tk_end = np.maximum(t[:, 5], t[:, 7]).max()
    up_end = u[:, 4].max()
    f = lambda v: (v - t0) / 1e3  # noqa
    print(f"{label:28s} topk {f(t0):6.2f}..{f(tk_end):6.2f} | UP start {f(u[:, 0].min()):6.2f}/{f(np.median(u[:, 0])):6.2f}"
          f" setup {f(np.median(u[:, 1])):6.2f} 1st {f(np.median(u[:, 2][u[:, 2] > 0])):6.2f} end {f(up_end):6.2f} |"
          f" DOWN start {f(w[:, 0].min()):6.2f}/{f(np.median(w[:, 0])):6.2f} 1st {f(np.median(w[:, 2])):6.2f}"
          f" end {f(w[:, 4].max()):6.2f}")


def report2(label):
    up, dn = bufs["up"][-1], bufs["down"][-1]
    u = up.view(-1, 16).cpu().numpy(); u = u[u[:, 0] > 0]
    w = dn.view(-1, 16).cpu().numpy(); w = w[w[:, 0] > 0]
    t0 = u[:, 0].min()
    f = lambda v: (v - t0) / 1e3  # noqa
    print(f"{label:28s} UP {len(u)} CTAs start ..{f(u[:, 0].max()):6.2f} 1st {f(np.median(u[:, 2][u[:, 2] > 0])):6.2f} "
          f"end {f(u[:, 4].max()):6.2f} | DOWN {len(w)} CTAs start {f(w[:, 0].min()):6.2f}/{f(np.median(w[:, 0])):6.2f}"
          f"/{f(w[:, 0].max()):6.2f} 1st {f(np.median(w[:, 2])):6.2f} end {f(w[:, 4].max()):6.2f}")


seq(False, False)  # idx / count for the UP>DOWN-only graphs
torch.cuda.synchronize()
for pdl in (1, 0):
    L.ps_set_pdl(pdl)
    for a_ready in (True, False):
        for _ in range(2):
            seq(False, False, parts=("up", "down"), a_ready=a_ready)
        gr = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(gr, stream=st):
            seq(False, True, parts=("up", "down"), a_ready=a_ready)
        torch.cuda.current_stream().wait_stream(st)
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        for v in bufs.values():
            v[-1].zero_()
        gr.replay()
        torch.cuda.synchronize()
        report2(f"graph UP>DOWN pdl={pdl} a_ready={a_ready}")
L.ps_set_pdl(1)

for with_mm in (False, True):
    for _ in range(2):
        seq(with_mm, False)
    torch.cuda.synchronize()
    seq(with_mm, True)
    torch.cuda.synchronize()
    report(f"eager mm={with_mm}")
    gr = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(gr, stream=st):
        seq(with_mm, True)
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    for v in bufs.values():
        v[-1].zero_()
    gr.replay()
    torch.cuda.synchronize()
    report(f"graph mm={with_mm}")
print("union count", int(cnt.item()))
