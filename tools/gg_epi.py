"""Epilogue anatomy of the gathered GEMM: UP alone, DOWN alone and UP->DOWN
inside a CUDA graph (B=64, |S|=6656 union rows), per-CTA stamp deltas
relative to each CTA's own accumulator-ready time (ps_debug_gemm_trace)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14884_b200 import _lib  # noqa: E402
from paper_2505_14884_b200.kernels import PackedMLP, ROW_PAD, gather_gemm_into, gather_gemm_t_into  # noqa: E402

dev = torch.device("cuda")
L = _lib.load()
B = int(os.environ.get("B", 64))
d, D, S = 4096, 16384, int(os.environ.get("S", 6656))
pks = [PackedMLP((torch.randn(D, d, device=dev) * 0.02).bfloat16(), torch.zeros(D, device=dev),
                 (torch.randn(D, d, device=dev) * 0.02).bfloat16(), torch.zeros(d, device=dev)) for _ in range(3)]
idx = torch.from_numpy(np.sort(np.random.default_rng(0).choice(D, S, replace=False)).astype(np.int32)).to(dev)
idx = torch.cat([idx, idx[-1:].repeat(ROW_PAD)])
cnt = torch.full((1,), S, dtype=torch.int32, device=dev)
x = torch.randn(B, d, device=dev).bfloat16()
hid = torch.zeros(B, pks[0].D_pad, dtype=torch.bfloat16, device=dev)
out = torch.zeros(B, d, dtype=torch.float32, device=dev)
POOL = [torch.zeros(16 * 2048, dtype=torch.int64, device=dev) for _ in range(16)]


def up(i, tr=None):
    if tr is not None:
        L.ps_debug_gemm_trace(tr.data_ptr(), 0, 0)
    gather_gemm_into(pks[i].w1t, idx, cnt, x, d, pks[i].b1, B, pks[i].D_pad, d, _lib.PS_ACT_RELU, hid,
                     hid.stride(0), splits=S + 256, tag="gg_up")
    L.ps_debug_gemm_trace(None, 0, 0)


def down(i, tr=None, a_ready=True):
    if tr is not None:
        L.ps_debug_gemm_trace(tr.data_ptr(), 0, 0)
    gather_gemm_t_into(pks[i].w2t, idx, cnt, hid, hid.stride(0), pks[i].b2, B, d, pks[i].D_pad, out, d,
                       residual=out, res_ld=d, splits=S + 256, tag="gg_down",
                       flags=_lib.PS_GG_A_READY if a_ready else 0)
    L.ps_debug_gemm_trace(None, 0, 0)


SLOTS = [(2, "1st stage"), (3, "mma issued"), (8, "acc ready"), (10, "staged"), (11, "peers in"), (12, "reduced"),
         (9, "tile0 done"), (4, "epi done")]


def show(label, tr):
    t = tr.view(-1, 16).cpu().numpy()
    t = t[(t[:, 0] > 0) & (t[:, 8] > 0)]
    a = t[:, 8]
    t0 = t[:, 0].min()
    print(f"  {label}: {len(t)} CTAs, acc ready {np.median(a - t0) / 1e3:6.2f} (max {(a.max() - t0) / 1e3:6.2f}) us"
          f" after the first CTA start")
    sm = t[:, 7]
    u, c = np.unique(sm, return_counts=True)
    per = dict(zip(u.tolist(), c.tolist()))
    two = np.array([per[x] >= 2 for x in sm])
    if two.any() and (~two).any():
        print(f"     SMs with 2 CTAs: {int((c >= 2).sum())}, with 1: {int((c == 1).sum())}; acc ready (from launch) "
              f"med {np.median(a[two] - t0) / 1e3:.2f} (2/SM) vs {np.median(a[~two] - t0) / 1e3:.2f} (1/SM) us")
    for j, nm in SLOTS:
        v = t[:, j]
        ok = v > 0
        if ok.any():
            dd = (v[ok] - a[ok]) / 1e3
            print(f"     {nm:11s} - acc ready: min {dd.min():6.2f} med {np.median(dd):6.2f} max {dd.max():6.2f} us")


def graph_run(fn):
    fn(False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=st):
        fn(True)
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for b in POOL:
        b.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3


if os.environ.get("LSU_MODE"):
    L.ps_debug_gemm_lsu_mode(int(os.environ["LSU_MODE"]))
print(f"B={B} |S|={S} PS_GG_PUSH={os.environ.get('PS_GG_PUSH', '1')} LSU_MODE={os.environ.get('LSU_MODE', '1')}")
us = graph_run(lambda tr: [up(i, POOL[i] if tr else None) for i in range(3)])
print(f"UP x3 graph: {us:.1f} us ({us / 3:.1f} per launch)")
show("UP #2", POOL[1])
us = graph_run(lambda tr: [down(i, POOL[i] if tr else None) for i in range(3)])
print(f"DOWN x3 graph: {us:.1f} us ({us / 3:.1f} per launch)")
show("DOWN #2", POOL[1])
us = graph_run(lambda tr: [f(i, POOL[2 * i + k] if tr else None) for i in range(3) for k, f in enumerate((up, down))])
print(f"(UP, DOWN) x3 graph: {us:.1f} us ({us / 3:.1f} per pair)")
show("UP #2", POOL[2])
show("DOWN #2", POOL[3])
