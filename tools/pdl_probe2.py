"""PDL overlap of two trivial kernels launched from Python: plain stream vs
torch.cuda.graph capture (tools/micro/pdl_lib.cu)."""
import ctypes
import os

import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "micro", "libpdl_probe.so"))
lib.pdl_a.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
lib.pdl_b.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
a = torch.zeros(4096, dtype=torch.int64, device="cuda")
b = torch.zeros(4096, dtype=torch.int64, device="cuda")


def seq():
    s = torch.cuda.current_stream().cuda_stream
    assert lib.pdl_a(a.data_ptr(), 64, 20000, s) == 0
    assert lib.pdl_b(b.data_ptr(), 148, s) == 0


def rep(label):
    ha, hb = a.cpu()[:128].view(64, 2), b.cpu()[:148]
    a0 = int(ha[:, 0].min())
    print(f"{label:30s} A ..{(int(ha[:, 1].max()) - a0) / 1e3:6.2f} us  B start {(int(hb.min()) - a0) / 1e3:6.2f}"
          f"..{(int(hb.max()) - a0) / 1e3:6.2f}")


for _ in range(3):
    seq()
torch.cuda.synchronize()
a.zero_(); b.zero_()
seq()
torch.cuda.synchronize()
rep("stream")
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=st):
    seq()
torch.cuda.current_stream().wait_stream(st)
g.replay()
torch.cuda.synchronize()
a.zero_(); b.zero_()
g.replay()
torch.cuda.synchronize()
rep("torch graph")

# mixed: micro kernel A -> library UP GEMM (does UP launch early?), and
# library select_union -> micro kernel B (does select_union trigger?)
import sys  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2505_14884_b200 import _lib as PL  # noqa: E402
from paper_2505_14884_b200.kernels import PackedMLP, ROW_PAD, gather_gemm_into  # noqa: E402
P = PL.load()
B_, d, D, k = 64, 4096, 16384, 1638
logits = torch.randn(B_, D, device="cuda")
pk = PackedMLP((torch.randn(D, d, device="cuda") * 0.02).bfloat16(), torch.zeros(D, device="cuda"),
               (torch.randn(D, d, device="cuda") * 0.02).bfloat16(), torch.zeros(d, device="cuda"))
x = torch.randn(B_, d, device="cuda").bfloat16()
hid = torch.zeros(B_, pk.D_pad, dtype=torch.bfloat16, device="cuda")
idx = torch.arange(D + ROW_PAD, dtype=torch.int32, device="cuda") % D
cnt = torch.full((1,), 6656, dtype=torch.int32, device="cuda")
nb = int(P.ps_select_union_workspace_bytes(B_, D))
sws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
tr = torch.zeros(16 * 4096, dtype=torch.int64, device="cuda")


def up():
    gather_gemm_into(pk.w1t, idx, cnt, x, d, pk.b1, B_, pk.D_pad, d, PL.PS_ACT_RELU, hid, hid.stride(0),
                     splits=7000, tag="gg_up")


def topk():
    PL.call("ps_select_union", logits.data_ptr(), None, B_, D, D, k, 0.0, sws.data_ptr(), nb, 0, D, ROW_PAD,
            idx.data_ptr(), cnt.data_ptr(), PL.stream_ptr())


def graph_of(fn):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=st):
        fn()
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    return g


def a_then_up():
    s = torch.cuda.current_stream().cuda_stream
    lib.pdl_a(a.data_ptr(), 64, 20000, s)
    up()


P.ps_debug_gemm_trace(tr.data_ptr(), 0, 0)
g = graph_of(a_then_up)
P.ps_debug_gemm_trace(None, 0, 0)
a.zero_(); tr.zero_()
g.replay()
torch.cuda.synchronize()
t = tr.view(-1, 16).cpu().numpy(); t = t[t[:, 0] > 0]
ha = a.cpu()[:128].view(64, 2)
a0 = int(ha[:, 0].min())
print(f"microA -> UP gemm: A ..{(int(ha[:, 1].max()) - a0) / 1e3:6.2f} us, UP CTA start {(t[:, 0].min() - a0) / 1e3:6.2f}"
      f"..{(t[:, 0].max() - a0) / 1e3:6.2f} ({len(t)} CTAs)")

idx.copy_(torch.arange(D + ROW_PAD, dtype=torch.int32, device="cuda") % D)


def a_then_topk():
    s = torch.cuda.current_stream().cuda_stream
    lib.pdl_a(a.data_ptr(), 64, 20000, s)
    topk()


def topk_then_b():
    topk()
    lib.pdl_b(b.data_ptr(), 148, torch.cuda.current_stream().cuda_stream)


P.ps_debug_topk_trace(tr.data_ptr())
g = graph_of(topk_then_b)
P.ps_debug_topk_trace(None)
b.zero_(); tr.zero_()
g.replay()
torch.cuda.synchronize()
t = tr.view(-1, 16).cpu().numpy(); t = t[t[:, 0] > 0]
hb = b.cpu()[:148]
t0 = t[:, 0].min()
print(f"topk -> microB: topk ..{(np.maximum(t[:, 5], t[:, 7]).max() - t0) / 1e3:6.2f} us, B start "
      f"{(int(hb.min()) - t0) / 1e3:6.2f}..{(int(hb.max()) - t0) / 1e3:6.2f}")


def topk_then_up():
    topk()
    up()


tr2 = torch.zeros(16 * 4096, dtype=torch.int64, device="cuda")
for rows in (64, 16, 1):
    B_ = rows
    P.ps_debug_topk_trace(tr.data_ptr())
    P.ps_debug_gemm_trace(tr2.data_ptr(), 0, 0)
    g = graph_of(topk_then_up)
    P.ps_debug_topk_trace(None)
    P.ps_debug_gemm_trace(None, 0, 0)
    tr.zero_(); tr2.zero_()
    g.replay()
    torch.cuda.synchronize()
    t = tr.view(-1, 16).cpu().numpy(); t = t[t[:, 0] > 0]
    u = tr2.view(-1, 16).cpu().numpy(); u = u[u[:, 0] > 0]
    t0 = t[:, 0].min()
    print(f"topk({rows} rows) -> UP: topk ..{(np.maximum(t[:, 5], t[:, 7]).max() - t0) / 1e3:6.2f} us, UP CTA start "
          f"{(u[:, 0].min() - t0) / 1e3:6.2f}..{(u[:, 0].max() - t0) / 1e3:6.2f} ({len(u)} CTAs), setup med "
          f"{(np.median(u[:, 1]) - t0) / 1e3:6.2f}")
