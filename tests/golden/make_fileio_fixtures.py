"""Generate the on-disk-format fixtures under tests/golden/fileio/ with the
REFERENCE's own writers (sparsedecode/fileio.py save_model / save_router,
calibration.LayerKTable.save, save_run_config, save_token_stream), plus an
npz of the arrays they hold, so tests/test_fileio.py pins this package's
readers to the reference byte layout without importing it.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fileio_fixtures.py
"""
import os

import numpy as np

from sparsedecode import fileio as F
from sparsedecode.calibration import LayerKTable
from sparsedecode.engine import SparsityPolicy
from sparsedecode.model import TransformerConfig, random_model
from sparsedecode.routers import HeadRouter, MlpRouter

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fileio")
os.makedirs(OUT, exist_ok=True)
arrays = {}
for tag, act, kvh in (("relu", "relu", 2), ("swiglu", "swiglu", 1)):
    cfg = TransformerConfig(layers=2, model_dim=64, ffn_dim=128, heads=2, kv_heads=kvh, vocab=40, max_seq=12,
                            activation=act)
    m = random_model(cfg, seed=7)
    F.save_model(m, os.path.join(OUT, f"model_{tag}.pswt"))
    arrays[f"{tag}_embed"] = m.embed
    arrays[f"{tag}_pos_embed"] = m.pos_embed
    arrays[f"{tag}_unembed"] = m.unembed
    arrays[f"{tag}_lnf_g"] = m.lnf_g
    arrays[f"{tag}_lnf_b"] = m.lnf_b
    for ell, lw in enumerate(m.layers):
        for name in lw.array_names(cfg):
            arrays[f"{tag}_l{ell}_{name}"] = getattr(lw, name)
mr = MlpRouter(64, 128, hidden_dim=16, seed=3)
mr.set_weights({k: np.random.default_rng(5 + i).normal(size=v.shape)
                for i, (k, v) in enumerate(mr.weights().items())})
F.save_router(mr, os.path.join(OUT, "router_mlp.psrt"))
for k, v in mr.weights().items():
    arrays[f"mlp_router_{k}"] = v
hr = HeadRouter(64, 2, seed=4)
hr.set_weights({k: np.random.default_rng(9 + i).normal(size=v.shape)
                for i, (k, v) in enumerate(hr.weights().items())})
F.save_router(hr, os.path.join(OUT, "router_head.psrt"))
for k, v in hr.weights().items():
    arrays[f"head_router_{k}"] = v
kt = LayerKTable(rows=((0, 20, 0.95), (1, 24, 0.9)))
kt.save(os.path.join(OUT, "k_table.tsv"))
pol = SparsityPolicy(mode="polar", mlp_k_table=kt, head_density=0.5)
F.save_run_config(TransformerConfig(2, 64, 128, 2, 2, 40, 12, "relu"), pol, os.path.join(OUT, "run_config.json"))
F.save_token_stream(np.array([3, 1, 4, 1, 5, 9, 2, 6]), os.path.join(OUT, "tokens.txt"))
np.savez_compressed(os.path.join(OUT, "expected.npz"), **{k: np.asarray(v, np.float32) for k, v in arrays.items()})
print("wrote", sorted(os.listdir(OUT)))
