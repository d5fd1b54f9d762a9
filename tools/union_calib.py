"""Measured batch-union density of the hot/cold neuron recipe (bench.py) vs
hot-set size, OPT-6.7B shape, a few eager decode steps.

    python tools/union_calib.py [--batch 64] [--hot 0,500,1000,1500] [--center 1]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200.engine import DecodeEngine, SparsityPolicy  # noqa: E402
from paper_2505_14884_b200.model import SHAPES, DeviceModel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", default="64")
ap.add_argument("--hot", default="0,500,1000,1300,1500")
ap.add_argument("--center", type=int, default=1)
ap.add_argument("--k", type=int, default=1638)
ap.add_argument("--layers", type=int, default=8)
a = ap.parse_args()
cfg = SHAPES["opt-6.7b"]
from dataclasses import replace  # noqa: E402
cfg = replace(cfg, layers=a.layers)
dev = torch.device("cuda")
model = DeviceModel.random(cfg, seed=1234, device=dev)
D = cfg.ffn_dim
for B in [int(x) for x in a.batch.split(",")]:
    for n_hot in [int(x) for x in a.hot.split(",")]:
        gen = np.random.default_rng(7)
        hr = [pb.HeadRouter(cfg.model_dim, cfg.kv_heads, seed=100 + e, device=dev) for e in range(cfg.layers)]
        mr = [pb.MlpRouter.random_device(cfg.model_dim, D, seed=200 + e, device=dev,
                                         hot=gen.choice(D, n_hot, replace=False) if n_hot else None,
                                         center=bool(a.center)) for e in range(cfg.layers)]
        pol = SparsityPolicy(mode="polar", head_density=0.5, mlp_k_table={e: a.k for e in range(cfg.layers)})
        eng = DecodeEngine(model, B, 1960, pol, head_routers=hr, mlp_routers=mr)
        eng.fill_random(1920, seed=99)
        tok = torch.randint(0, cfg.vocab, (B,), generator=torch.Generator().manual_seed(5))
        dens = []
        for s in range(3):
            eng.step(tok if s == 0 else None)
            dens.append(eng.union_counts.float().cpu().numpy() / D)
        d = np.array(dens)
        print(f"B={B} hot={n_hot} center={a.center}: |S|/D mean {d.mean():.3f} per layer "
              f"{np.round(d.mean(0), 3).tolist()}", flush=True)
        del eng
