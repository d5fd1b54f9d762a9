"""A model, routers and k-table loaded from the reference's file formats
(fixtures written by its own writers) drive the GPU decode step; the step
matches the CPU oracle on the same arrays (selections bit-exact given the
device router logits, logits within the bf16 tolerance)."""

import os

import numpy as np
import pytest
import torch

from oracle import polar_oracle as po

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200 import fileio as F  # noqa: E402
from paper_2505_14884_b200.engine import DecodeEngine  # noqa: E402

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fileio")
B, CTX = 4, 8


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("tag", ["relu", "swiglu"])
@pytest.mark.parametrize("mode", ["dense", "polar"])
def test_loaded_model_step_matches_oracle(tag, mode):
    path = os.path.join(G, f"model_{tag}.pswt")
    host = F.read_model(path)
    cfg = host["config"]
    model = F.load_model(path)
    _, pol = F.load_run_config(os.path.join(G, "run_config.json"))
    if mode == "dense":
        pol = type(pol)(mode="dense")
    _, hw = F.read_router(os.path.join(G, "router_head.psrt"))
    _, mw = F.read_router(os.path.join(G, "router_mlp.psrt"))
    hr = [F.load_router(os.path.join(G, "router_head.psrt"))] * cfg.layers
    if cfg.kv_heads != hw["w"].shape[1]:  # GQA fixture: route over its KV groups
        hw = {"w": hw["w"][:, :cfg.kv_heads], "b": hw["b"][:cfg.kv_heads]}
        hr = [pb.HeadRouter.from_weights(hw["w"], hw["b"])] * cfg.layers
    mr = [F.load_router(os.path.join(G, "router_mlp.psrt"))] * cfg.layers
    eng = DecodeEngine(model, B, cfg.max_seq, pol, head_routers=hr, mlp_routers=mr)
    eng.record = {}
    rng = np.random.default_rng(3)
    for c in eng.caches:
        c.fill_random(rng, CTX)
    tokens = F.load_token_stream(os.path.join(G, "tokens.txt"))[:B]
    logits = eng.step(tokens).cpu().numpy()

    ref_host = dict(host, config=cfg.to_dict())
    rng = np.random.default_rng(3)
    caches = []
    for _ in range(cfg.layers):
        c = po.KVCache(B, cfg.kv_heads, cfg.max_seq, cfg.head_dim)
        c.fill_random(rng, CTX)
        caches.append(c)
    kw = {}
    if mode == "polar":
        rec = eng.record
        k_h = pol.head_budget(cfg.kv_heads)
        for hl, sel in zip(rec.get("head_logits", []), rec.get("heads", [])):
            assert np.array_equal(sel.cpu().numpy(), po.topk_indices_rows(hl.cpu().numpy(), k_h))
        forced = {"heads": {1: rec["heads"][0].cpu().numpy()}}
        if tag == "relu":
            for ell in range(cfg.layers):
                ml = rec["mlp_logits"][ell].cpu().numpy()
                ref_u = po.union_neuron_indices(list(po.topk_indices_rows(ml, pol.k_for(ell))))
                assert np.array_equal(rec["union"][ell].cpu().numpy(), ref_u)
            forced["union"] = {e: rec["union"][e].cpu().numpy() for e in range(cfg.layers)}
        kw = dict(mode="polar", head_density=pol.head_density,
                  k_table={e: pol.k_for(e) for e in range(cfg.layers)} if tag == "relu" else None,
                  head_routers=[hw] * cfg.layers, mlp_routers=[mw] * cfg.layers, forced=forced)
    ref = po.decode_step(ref_host, caches, tokens, **kw)
    assert _rel(logits, ref) <= 2e-2
    assert np.abs(logits - ref).max() <= 2e-2 * max(1.0, np.abs(ref).max())
