"""Per-CTA timeline of one ps_sparse_mlp launch (ps_debug_chain_trace)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_14884_b200 import _lib
from paper_2505_14884_b200.kernels import PackedMLP, ROW_PAD, _round_up, sparse_mlp_into

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
S = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = torch.device("cuda")
d, D, k = 4096, 16384, 6553
g = torch.Generator(device=dev).manual_seed(0)
pk = PackedMLP((torch.randn(D, d, device=dev, generator=g) * 0.02).bfloat16(), torch.zeros(D, device=dev),
               (torch.randn(D, d, device=dev, generator=g) * 0.02).bfloat16(), torch.zeros(d, device=dev))
ids = torch.randperm(D, device=dev, generator=g)[:k].sort().values.int()
idx = torch.full((_round_up(D, ROW_PAD),), int(ids[-1]), dtype=torch.int32, device=dev); idx[:k] = ids
cnt = torch.tensor([k], dtype=torch.int32, device=dev)
x = torch.randn(B, d, device=dev, generator=g).bfloat16()
hid = torch.zeros(B, _round_up(D, ROW_PAD), dtype=torch.bfloat16, device=dev)
out = torch.zeros(B, d, device=dev)
L = _lib.load()
L.ps_debug_chain_stages(S)
print("B", B, "stages", S)
for _ in range(3):
    sparse_mlp_into(pk, x, idx, cnt, hid, out)
tr = torch.zeros(148 * 16, dtype=torch.int64, device=dev)
L.ps_debug_chain_trace(tr.data_ptr())
sparse_mlp_into(pk, x, idx, cnt, hid, out)
torch.cuda.synchronize()
L.ps_debug_chain_trace(None)
t = tr.view(148, 16).cpu().numpy().astype(np.float64)
t0 = t[:, 0].min()
names = ["start", "after_wait", "first_stage", "last_ph0_acc", "ph1_wait_begin", "first_flag", "epi_done", "end",
         "smid", "p0_tfull", "p0_ticket", "p0_done", "p0_publish", "fin_loads_done", "ld_first_issue", "tma_first_issue"]
for i, n in enumerate(names):
    if n == "smid":
        continue
    col = t[:, i]
    col = col[col > 0]
    if len(col):
        print(f"{n:15s} min {(col.min()-t0)/1e3:8.2f} us  median {(np.median(col)-t0)/1e3:8.2f}  max {(col.max()-t0)/1e3:8.2f}")
