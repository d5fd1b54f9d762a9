"""In-graph cost attribution of one decode step: the step is re-captured with
one component removed at a time and the replay time difference is that
component's effective cost inside the graph (its kernels + the launch gaps
they bring).  Profiling aid only -- a step with a component removed computes
garbage.

    python tools/attrib.py [--batch 64] [--config opt-6.7b] [--mode polar]
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200 import _lib, engine as E  # noqa: E402
from paper_2505_14884_b200.engine import DecodeEngine, SparsityPolicy  # noqa: E402
from paper_2505_14884_b200.model import SHAPES, DeviceModel  # noqa: E402


class _LibProxy:
    def __init__(self, lib, drop):
        self._lib, self._drop = lib, drop

    def __getattr__(self, name):
        if name in self._drop:
            return lambda *a, **k: 0
        return getattr(self._lib, name)


class _TorchProxy:
    def __init__(self, eng):
        self._eng = eng

    def mm(self, a, b, *args, out=None, **kw):
        if out is self._eng.r_logits:
            return out
        return torch.mm(a, b, *args, out=out, **kw)

    def __getattr__(self, name):
        return getattr(torch, name)


def time_graph(eng, caches_len, reps=10):
    ts = []
    for _ in range(reps):
        for c, ln in zip(eng.caches, caches_len):
            c.lengths.copy_(ln)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        eng.graph.replay()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.median(ts))


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
    ap.add_argument("--mode", default="polar")
    ap.add_argument("--mlp-backend", default="split")
    ap.add_argument("--only", default="", help="comma list of components to drop (default: all)")
    a = ap.parse_args()
    import bench  # the bench's neuron recipe (hot/cold, centered router)
    dev = torch.device("cuda", 0)
    cfg = SHAPES[a.config]
    L, H_kv, D = cfg.layers, cfg.kv_heads, cfg.ffn_dim
    k_mlp, n_hot = bench.neuron_recipe(a, D)
    gen = np.random.default_rng(7)
    model = DeviceModel.random(cfg, seed=1234, device=dev)
    relu = cfg.activation == "relu"
    hr = [pb.HeadRouter(cfg.model_dim, H_kv, seed=100 + e, device=dev) for e in range(L)]
    mr = None
    if relu:
        mr = [pb.MlpRouter.random_device(cfg.model_dim, D, seed=200 + e, device=dev,
                                         hot=gen.choice(D, n_hot, replace=False) if n_hot else None,
                                         center=a.union_recipe == "hot-cold") for e in range(L)]
    if a.mode == "polar":
        pol = SparsityPolicy(mode="polar", head_density=a.rho,
                             mlp_k_table={e: k_mlp for e in range(L)} if relu else None)
    else:
        pol = SparsityPolicy(mode="dense")
    eng = DecodeEngine(model, a.batch, a.ctx + 16, pol, head_routers=hr, mlp_routers=mr, mlp_backend=a.mlp_backend)
    eng.fill_random(a.ctx, seed=99)
    eng.tokens.copy_(torch.randint(0, cfg.vocab, (a.batch,), dtype=torch.int32))
    lens = [c.lengths.clone() for c in eng.caches]


    orig = {"sha": E.sha_decode_into, "mlp": E.mlp_into, "smlp": E.sparse_mlp_into, "lib": _lib.load, "torch": E.torch,
            "lb": eng._linear_bf16, "lf": eng._linear_f32, "ln": eng._ln, "hs": eng._head_select}
    lib = _lib.load()

    def restore():
        E.sha_decode_into, E.mlp_into, E.torch = orig["sha"], orig["mlp"], orig["torch"]
        E.sparse_mlp_into = orig["smlp"]
        _lib.load = orig["lib"]
        eng._linear_bf16, eng._linear_f32, eng._ln, eng._head_select = orig["lb"], orig["lf"], orig["ln"], orig["hs"]

    def drop(what):
        if what == "sha":
            E.sha_decode_into = lambda *x, **k: None
        elif what == "mlp(up+down)":
            E.mlp_into = lambda *x, **k: None
            E.sparse_mlp_into = lambda *x, **k: None
        elif what == "select_union":
            _lib.load = lambda: _LibProxy(lib, {"ps_select_union"})
        elif what == "router_gemms":
            E.torch = _TorchProxy(eng)
            eng._linear_bf16 = lambda x2d, w_t, bias, out, act_relu=False, tag="gg": (
                0 if (act_relu and tag == "gg") else orig["lb"](x2d, w_t, bias, out, act_relu, tag))
        elif what == "qkv":
            eng._linear_bf16 = lambda x2d, w_t, bias, out, act_relu=False, tag="gg": (
                0 if tag == "gg_qkv" else orig["lb"](x2d, w_t, bias, out, act_relu, tag))
        elif what == "o_proj":
            eng._linear_f32 = lambda x2d, w_t, bias, out, residual=False, tag="gg", defer_bias=False: (
                ((0, bias) if defer_bias else 0) if tag == "gg_o" else
                orig["lf"](x2d, w_t, bias, out, residual, tag, defer_bias))
        elif what == "layernorm":
            eng._ln = lambda g, b, pending: 0
        elif what == "head_router+append":
            eng._head_select = lambda ell, k_h, append=None: eng.sel_full[:, :k_h]

    items = ["none", "sha", "mlp(up+down)", "select_union", "router_gemms", "qkv", "o_proj", "layernorm",
             "head_router+append"]
    if a.only:
        items = ["none"] + a.only.split(",")
    base = None
    for what in items:
        restore()
        if what != "none":
            drop(what)
        eng.graph = None
        try:
            eng.capture()
            t = time_graph(eng, lens)
        except Exception as ex:  # noqa: BLE001
            print(f"{what:20s} failed: {ex}", flush=True)
            continue
        finally:
            restore()
        if base is None:
            base = t
            print(f"full step {t:9.1f} us  ({t / L:6.1f} us/layer)", flush=True)
        else:
            print(f"-{what:20s} {t:9.1f} us  saves {base - t:8.1f} us  ({(base - t) / L:6.1f} us/layer)", flush=True)


if __name__ == "__main__":
    main()
