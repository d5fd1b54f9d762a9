"""In-graph timeline of one polar decode step: every traced libpolar launch
(gathered GEMMs, select_union) gets its own per-CTA globaltimer buffer at
capture time, so one replay shows when each kernel's CTAs started, passed
their setup, landed their first stage and exited -- the gaps between them are
the untraced kernels (SHA, cuBLAS, LN, head router).  Profiling aid only.

    python tools/timeline.py [--batch 64] [--layers-shown 2]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200 import _lib  # noqa: E402
from paper_2505_14884_b200.engine import DecodeEngine, SparsityPolicy  # noqa: E402
from paper_2505_14884_b200.model import SHAPES, DeviceModel  # noqa: E402

TRACED = {"ps_gather_gemm": "gemm", "ps_gather_gemm_t": "gemm", "ps_select_union": "topk",
          "ps_select_union_bitmap": "topk",
          "ps_router_mlp_fused": "router", "ps_sha_decode": "sha",
          "ps_sparse_mlp": "chain", "ps_router_mlp": "chain"}


class Proxy:
    def __init__(self, lib, dev, n=512):
        self.lib, self.dev, self.bufs = lib, dev, []
        # preallocated: a torch.zeros inside the capture would add a memset
        # node between two kernels and break their PDL edge
        self.pool = [torch.zeros(16 * 2048, dtype=torch.int64, device=dev) for _ in range(n)]

    def __getattr__(self, name):
        fn = getattr(self.lib, name)
        kind = TRACED.get(name)
        if kind is None:
            return fn

        def wrapped(*a):
            buf = self.pool.pop()
            self.bufs.append((name, buf))
            if kind == "gemm":
                self.lib.ps_debug_gemm_trace(buf.data_ptr(), 0, 0)
            elif kind == "topk":
                self.lib.ps_debug_topk_trace(buf.data_ptr())
            elif kind == "router":
                self.lib.ps_debug_router_trace(buf.data_ptr())
            elif kind == "sha":
                self.lib.ps_debug_sha_trace(buf.data_ptr())
            else:
                self.lib.ps_debug_chain_trace(buf.data_ptr())
            r = fn(*a)
            if kind == "gemm":
                self.lib.ps_debug_gemm_trace(None, 0, 0)
            elif kind == "topk":
                self.lib.ps_debug_topk_trace(None)
            elif kind == "router":
                self.lib.ps_debug_router_trace(None)
            elif kind == "sha":
                self.lib.ps_debug_sha_trace(None)
            else:
                self.lib.ps_debug_chain_trace(None)
            return r
        return wrapped


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=1920)
    ap.add_argument("--rho", type=float, default=0.5)
    ap.add_argument("--union", type=float, default=0.5)
    ap.add_argument("--k-frac", type=float, default=0.1)
    ap.add_argument("--hot-frac", type=float, default=0.072)
    ap.add_argument("--union-recipe", default="hot-cold")
    ap.add_argument("--router-backend", default=None)
    ap.add_argument("--mlp-backend", default="split")
    ap.add_argument("--dense-backend", default="cublas")
    ap.add_argument("--layers-shown", type=int, default=2)
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--dot", default="", help="dump the captured graph (cudaGraphDebugDotPrint) here")
    a = ap.parse_args()
    import bench

    dev = torch.device("cuda", 0)
    cfg = SHAPES[a.config]
    L, H_kv, D = cfg.layers, cfg.kv_heads, cfg.ffn_dim
    k_mlp, n_hot = bench.neuron_recipe(a, D)
    gen = np.random.default_rng(7)
    model = DeviceModel.random(cfg, seed=1234, device=dev)
    hr = [pb.HeadRouter(cfg.model_dim, H_kv, seed=100 + e, device=dev) for e in range(L)]
    mr = [pb.MlpRouter.random_device(cfg.model_dim, D, seed=200 + e, device=dev,
                                     hot=gen.choice(D, n_hot, replace=False) if n_hot else None,
                                     center=a.union_recipe == "hot-cold") for e in range(L)]
    pol = SparsityPolicy(mode="polar", head_density=a.rho, mlp_k_table={e: k_mlp for e in range(L)})
    eng = DecodeEngine(model, a.batch, a.ctx + 64, pol, head_routers=hr, mlp_routers=mr,
                       router_backend=a.router_backend, mlp_backend=a.mlp_backend, dense_backend=a.dense_backend)
    eng.fill_random(a.ctx, seed=99)
    eng.tokens.copy_(torch.randint(0, cfg.vocab, (a.batch,), dtype=torch.int32))
    lib = _lib.load()
    if a.no_pdl:
        lib.ps_set_pdl(0)
    if a.dot:
        orig_graph = torch.cuda.CUDAGraph

        class DbgGraph(orig_graph):
            def __init__(self, *x, **k):
                super().__init__(*x, **k)
                self.enable_debug_mode()
        torch.cuda.CUDAGraph = DbgGraph
    proxy = Proxy(lib, dev)
    _lib._LIB = proxy
    try:
        eng.capture()
    finally:
        _lib._LIB = lib
    if a.dot:
        eng.graph.debug_dump(a.dot)
    for _ in range(3):
        eng.graph.replay()
    torch.cuda.synchronize()
    for _, b in proxy.bufs:
        b.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    eng.graph.replay()
    e.record()
    torch.cuda.synchronize()
    step_us = s.elapsed_time(e) * 1e3
    rows = []
    for name, b in proxy.bufs:
        t = b.view(-1, 16).cpu().numpy()
        t = t[t[:, 0] > 0]
        if len(t) == 0:
            continue
        if name == "ps_select_union":
            end = np.maximum(t[:, 5], t[:, 7])
            rows.append((name, len(t), t[:, 0].min(), np.median(t[:, 0]), None, None, end.max()))
        elif name.startswith("ps_gather"):
            f = t[:, 2][t[:, 2] > 0]
            rows.append((name, len(t), t[:, 0].min(), np.median(t[:, 0]), np.median(t[:, 1]),
                         np.median(f) if len(f) else None, t[:, 5].max()))
        elif name == "ps_router_mlp_fused":
            rows.append((name, len(t), t[:, 0].min(), np.median(t[:, 0]), None, None, t[:, 6].max()))
        elif name == "ps_sha_decode":
            t8 = b.view(-1, 8).cpu().numpy()
            t8 = t8[t8[:, 0] > 0]
            rows.append((name, len(t8), t8[:, 0].min(), np.median(t8[:, 0]), None, None, t8[:, 3].max()))
        else:
            rows.append((name, len(t), t[:, 0].min(), np.median(t[:, 0]), None, None, t.max()))
    t0 = min(r[2] for r in rows)
    # detail of the last layer's traced launches (per-CTA stamp distributions)
    gl = [(n, b) for n, b in proxy.bufs if b.view(-1, 16)[:, 0].gt(0).any()]
    per = len(gl) // L
    for name, b in gl[-per:]:
        t = b.view(-1, 8 if name == "ps_sha_decode" else 16).cpu().numpy()
        t = t[t[:, 0] > 0]
        slots = {"ps_select_union": [(0, "start"), (5, "selected"), (7, "union")],
                 "ps_sha_decode": [(0, "start"), (1, "dep wait"), (2, "partition"), (4, "1st tile"), (3, "end")],
                 "ps_router_mlp_fused": [(0, "start"), (1, "prefetched"), (7, "dep. wait"), (12, "p1 mma"),
                                         (13, "p1 done"), (2, "p1 written"), (3, "barrier1"), (10, "reduce in"), (11, "reduce out"),
                                         (4, "barrier2"), (8, "p2 mma0"), (9, "p2 mmaN"), (5, "acc2 ready"),
                                         (6, "done")]}.get(
            name, [(0, "start"), (1, "setup"), (2, "1st stage"), (3, "mma issued"), (8, "acc ready"),
                   (10, "staged"), (11, "peers in"), (12, "reduced"), (13, "fre"), (9, "tile0 done"),
                   (4, "epi done"), (5, "end")])
        print(f"  {name} ({len(t)} CTAs)")
        for j, lab in slots:
            v = t[:, j]
            v = v[v > 0]
            if len(v):
                d = (v - t0) / 1e3
                print(f"     {lab:10s} n={len(v):4d} min {d.min():9.2f} med {np.median(d):9.2f} max {d.max():9.2f}")
    print(f"step {step_us:.1f} us ({step_us / L:.1f} us/layer), {len(rows)} traced launches, B={a.batch}")
    per_layer = len(rows) // L
    show = rows[-per_layer * a.layers_shown:]
    prev_end = None
    print(f"{'kernel':18s} {'CTAs':>5s} {'gap':>7s} {'start0':>8s} {'startmed':>8s} {'setup':>8s} {'1st':>8s} {'end':>8s} {'dur':>7s}")
    for name, n, st, sm, su, f1, en in show:
        rel = lambda v: f"{(v - t0) / 1e3:8.2f}" if v is not None else "       -"  # noqa
        gap = f"{(st - prev_end) / 1e3:7.2f}" if prev_end is not None else "      -"
        print(f"{name:18s} {n:5d} {gap} {rel(st)} {rel(sm)} {rel(su)} {rel(f1)} {rel(en)} {(en - st) / 1e3:7.2f}")
        prev_end = en
    # per-layer spans between consecutive select_union ends (one layer)
    ends = [r[6] for r in rows if r[0] == "ps_select_union"]
    if len(ends) > 2:
        d = np.diff(ends) / 1e3
        print(f"layer period (select_union to select_union): median {np.median(d):.1f} us")
    for kind in sorted(set(r[0] for r in rows)):
        durs = [(r[6] - r[2]) / 1e3 for r in rows if r[0] == kind]
        print(f"{kind:18s} median span {np.median(durs):6.2f} us  (n={len(durs)})")


if __name__ == "__main__":
    main()
