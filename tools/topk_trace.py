"""Phase timeline of the top-k kernel (ps_debug_topk_trace)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14884_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
L = _lib.load()
names = ["start", "loaded", "bracket", "counted", "kth", "selected", "barrier1", "union", "or-loaded", "scanned",
         "-", "-", "br-hist1", "br-sel1", "br-hist2"]
for rows, cols, k, dist, use_bias in [(64, 16384, 1638, "hotcold", True), (1, 16384, 1638, "hotcold", True),
                                     (16, 16384, 1638, "hotcold", True), (128, 16384, 1638, "hotcold", True),
                                     (64, 16384, 8192, "hot", False), (64, 16384, 8192, "hot", True),
                                     (64, 1024, 512, "normal", False), (256, 16384, 8192, "hot", False)]:
    g = torch.Generator(device=dev); g.manual_seed(0)
    lg = torch.randn(rows, cols, device=dev, generator=g)
    if dist == "hotcold":  # bench.py recipe: 1180 hot columns always in every row's top-1638
        lg[:, torch.randperm(cols, device=dev, generator=g)[:1180]] += 6.0
    if dist == "hot":
        lg[:, torch.randperm(cols, device=dev, generator=g)[: cols // 2]] += 20.0
    bias = torch.randn(cols, device=dev, generator=g) if use_bias else None
    bm = torch.zeros((cols + 31) // 32, dtype=torch.int32, device=dev)
    nb = int(_lib.load().ps_select_union_workspace_bytes(rows, cols))
    ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
    buf = torch.empty(cols, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    tk = torch.zeros(1, dtype=torch.int32, device=dev)
    tr = torch.zeros(rows * 8 * 16, dtype=torch.int64, device=dev)
    f = lambda: _lib.call("ps_select_union", lg.data_ptr(), None if bias is None else bias.data_ptr(), rows, cols, cols, k, 0.0, ws.data_ptr(),  # noqa
                          nb, 0, cols, 128, buf.data_ptr(), cnt.data_ptr(), _lib.stream_ptr())
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    L.ps_debug_topk_trace(tr.data_ptr())
    f()
    torch.cuda.synchronize()
    L.ps_debug_topk_trace(None)
    t = tr.view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    print(f"== {rows}x{cols} k={k} {dist} bias={use_bias}: CTAs={len(t)}  span={(max(t[:, 5].max(), t[:, 7].max()) - t0) / 1e3:.1f} us  "
          f"fallbacks={int((t[:, 11] == 1).sum())}  cand(med)={int(np.median(t[:, 10] >> 32))} "
          f"eq(max)={int((t[:, 10] & 0xffffffff).max())}")
    order = [1, 12, 13, 14, 2, 3, 4, 5, 6, 8, 9, 7]
    if os.environ.get("PS_TOPK_V2", "1") != "0":  # topk_union.cu stamps
        names[:8] = ["start", "loaded", "round1", "round2", "round3", "selected", "last-in", "union"]
        names[10:12] = ["r1-hist", "r2-hist"]
        order = [1, 10, 2, 11, 3, 4, 5, 6, 7]
    for j in order:
        v = t[:, j]
        ok = v > 0
        if ok.any():
            d = (v[ok] - t0) / 1e3
            print(f"   {names[j]:9s} min {d.min():7.2f}  med {np.median(d):7.2f}  max {d.max():7.2f} us")
    if os.environ.get("PS_TOPK_V2", "1") != "0" and (t[:, 9] > 0).any():
        f = (t[:, 9] - t[:, 8]) / np.maximum(t[:, 5] - t[:, 0], 1)
        print(f"   SM clock (start->selected) med {np.median(f) * 1e3:.0f} MHz")
    print(f"   start     min {0:7.2f}  med {np.median((t[:, 0] - t0) / 1e3):7.2f}  max {(t[:, 0].max() - t0) / 1e3:7.2f}")
