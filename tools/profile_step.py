"""One polar (or dense) decode step of the bench workload between
cudaProfilerStart/Stop, for ncu:

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python tools/profile_step.py

The engine is built exactly as bench.py builds it; the step is replayed from
its CUDA graph (ncu profiles graph kernel nodes one by one).
"""

from __future__ import annotations

import argparse
import dataclasses
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200.engine import DecodeEngine, SparsityPolicy  # noqa: E402
from paper_2505_14884_b200.model import SHAPES, DeviceModel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=1920)
    ap.add_argument("--rho", type=float, default=0.5)
    ap.add_argument("--union", type=float, default=0.5)
    ap.add_argument("--k-frac", type=float, default=0.1)
    ap.add_argument("--hot-frac", type=float, default=0.072)
    ap.add_argument("--union-recipe", default="hot-cold", choices=["hot-cold", "hot-set"])
    ap.add_argument("--mode", default="polar")
    ap.add_argument("--layers", type=int, default=0, help="truncate to this many layers (0 = all)")
    ap.add_argument("--no-graph", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = SHAPES[a.config]
    if a.layers:
        cfg = dataclasses.replace(cfg, layers=a.layers)
    L, H_kv, D = cfg.layers, cfg.kv_heads, cfg.ffn_dim
    import bench  # the bench's neuron recipe (hot/cold by default)

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
    eng = DecodeEngine(model, a.batch, a.ctx + 16, pol, head_routers=hr, mlp_routers=mr)
    eng.fill_random(a.ctx, seed=99)
    eng.tokens.copy_(torch.randint(0, cfg.vocab, (a.batch,), dtype=torch.int32))
    if not a.no_graph:
        eng.capture()
    for _ in range(3):
        if a.no_graph:
            eng.step_launches()
            eng._advance()
        else:
            eng.graph.replay()
            eng._advance()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    if a.no_graph:
        eng.step_launches()
        eng._advance()
    else:
        eng.graph.replay()
        eng._advance()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled one", a.mode, "step; launches/step =", eng.launches_per_step, "k_heads", math.ceil(a.rho * H_kv))


if __name__ == "__main__":
    main()
