"""Timing probe of the selection kernels (CUDA-graph replay, warm)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_14884_b200 import _lib  # noqa: E402
from tools.kbench import timeit  # noqa: E402

dev = torch.device("cuda")
st = lambda: _lib.stream_ptr()  # noqa: E731
for rows, cols, k, dist in [(64, 16384, 8192, "hot"), (64, 16384, 8192, "normal"), (64, 16384, 1638, "normal"),
                            (256, 16384, 8192, "hot"), (8, 16384, 8192, "hot"), (64, 1024, 512, "normal")]:
    g = torch.Generator(device=dev); g.manual_seed(0)
    lg = torch.randn(rows, cols, device=dev, generator=g)
    if dist == "hot":
        hot = torch.randperm(cols, device=dev, generator=g)[: cols // 2]
        lg[:, hot] += 20.0
    bm = torch.zeros((cols + 31) // 32, dtype=torch.int32, device=dev)
    nb = int(_lib.load().ps_select_union_workspace_bytes(rows, cols))
    ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
    buf = torch.empty(cols, dtype=torch.int32, device=dev)
    ids = torch.empty(rows, k, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    tk = torch.zeros(1, dtype=torch.int32, device=dev)
    f_union = lambda i: _lib.call("ps_select_union", lg.data_ptr(), None, rows, cols, cols, k, 0.0, ws.data_ptr(),  # noqa
                                  nb, 0, cols, 128, buf.data_ptr(), cnt.data_ptr(), st())
    f_bm = lambda i: _lib.call("ps_topk_rows", lg.data_ptr(), rows, cols, cols, k, None, bm.data_ptr(), st())  # noqa
    f_ids = lambda i: _lib.call("ps_topk_rows", lg.data_ptr(), rows, cols, cols, k, ids.data_ptr(), None, st())  # noqa
    f_thr = lambda i: _lib.call("ps_threshold_rows", lg.data_ptr(), rows, cols, cols, 1.0, bm.data_ptr(), st())  # noqa
    f_cmp = lambda i: _lib.call("ps_bitmap_compact", bm.data_ptr(), cols, 0, cols, 128, buf.data_ptr(),  # noqa
                                cnt.data_ptr(), st())
    res = {n: timeit(f, 20) for n, f in [("select_union", f_union), ("topk->bitmap", f_bm), ("topk->ids", f_ids),
                                          ("threshold", f_thr), ("compact", f_cmp)]}
    print(f"{rows}x{cols} k={k} {dist}: " + "  ".join(f"{n} {v:.1f}us" for n, v in res.items()), flush=True)
