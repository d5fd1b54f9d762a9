"""The reference-facing adapter: a reference-shaped engine module (the
oracle's ``decode_step``, which resolves its kernels as module globals like
sparsedecode/engine.py:25-35) decodes on the B200 kernels after
``adapter.install`` and agrees with its own CPU run."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import polar_oracle as po  # noqa: E402

pytestmark = pytest.mark.gpu


def _run(model, tokens, seed, **kw):
    rng = np.random.default_rng(seed)
    caches = []
    for _ in range(model["config"]["layers"]):
        c = po.KVCache(8, model["config"]["kv_heads"], 64, model["config"]["model_dim"] // model["config"]["heads"])
        c.fill_random(rng, 40)
        caches.append(c)
    rec = {}
    out = po.decode_step(model, caches, tokens, record=rec, **kw)
    return out, rec


@pytest.mark.parametrize("kv_heads", [8, 4])
def test_reference_engine_on_gpu_kernels(kv_heads):
    from paper_2505_14884_b200 import adapter

    model = po.random_model(2, 128, 512, 8, kv_heads, 256, 96, seed=5)
    routers = dict(head_routers=[po.init_head_router(128, kv_heads, seed=60 + e) for e in range(2)],
                   mlp_routers=[po.init_mlp_router(128, 512, seed=70 + e) for e in range(2)])
    kw = dict(mode="polar", head_density=0.5, k_table={0: 64, 1: 64}, **routers)
    tokens = np.arange(8) * 3
    ref, rec_ref = _run(model, tokens, 1, **kw)
    saved = adapter.install(po)
    try:
        got, rec_got = _run(model, tokens, 1, **kw)
    finally:
        adapter.uninstall(po, saved)
    assert po.gqa_selective_attention_decode is saved["gqa_selective_attention_decode"]
    # the device path rounds activations to bf16, so later layers see slightly
    # different router inputs: selections must agree up to a few boundary
    # flips (bit-exactness given identical logits is tests/test_gpu_parity.py)
    for a, b in zip(rec_ref["heads"], rec_got["heads"]):
        assert (np.asarray(a) == np.asarray(b)).all(axis=1).mean() >= 0.75
    for a, b in zip(rec_ref["union"], rec_got["union"]):
        a, b = set(np.asarray(a).tolist()), set(np.asarray(b).tolist())
        assert len(a & b) >= 0.95 * max(len(a), len(b))
    # numerics: the CPU run forced onto the device run's selections
    forced = {"heads": {e: h for e, h in enumerate(rec_got["heads"]) if e > 0},
              "union": dict(enumerate(rec_got["union"]))}
    ref2, _ = _run(model, tokens, 1, forced=forced, **kw)
    rel = np.linalg.norm(got - ref2) / np.linalg.norm(ref2)
    assert rel <= 2e-2, rel
