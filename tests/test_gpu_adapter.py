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


def _import_reference():
    import os
    import sys

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "sparsedecode")) and ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import sparsedecode
    except Exception:
        return None
    return sparsedecode


def test_unmodified_reference_engine_on_gpu_kernels():
    """adapter.install on the REAL reference engine module
    (sparsedecode.engine, pip-installed unmodified into baseline/_ref): its
    own decode_step runs on this package's CUDA kernels and agrees with its
    own CPU run (forced onto the same selections through the reference's
    rebinding hook, tests/test_engine.py:55-64)."""
    sd = _import_reference()
    if sd is None:
        pytest.skip("baseline/_ref (the unmodified reference install) is not present")
    from sparsedecode import engine as sde, model as sdm

    from paper_2505_14884_b200 import adapter

    cfg = sdm.TransformerConfig(2, 128, 512, 8, 4, 256, 96, "relu")
    model = sdm.random_model(cfg, 5)

    def session(seed):
        rng = np.random.default_rng(seed)
        caches = []
        for _ in range(2):
            c = sd.KVCache(8, 4, 96, 16)
            c.fill_random(rng, 40)
            caches.append(c)
        policy = sd.SparsityPolicy(mode="polar", mlp_k_table=sd.LayerKTable(((0, 64, 1.0), (1, 64, 1.0))),
                                   head_density=0.5)
        return sd.DecodeSession(caches=caches, policy=policy,
                                mlp_routers=[sd.MlpRouter(128, 512, seed=70 + e) for e in range(2)],
                                head_routers=[sd.HeadRouter(128, 4, seed=60 + e) for e in range(2)])

    tokens = np.arange(8) * 3
    BHI = sde.BatchHeadIndex

    class _Heads:  # records / replays the head selections (BatchHeadIndex.from_logits)
        full = staticmethod(BHI.full)
        replay = None

        @staticmethod
        def from_logits(logits, k):
            if _Heads.replay is not None:
                return next(_Heads.replay)
            out = BHI.from_logits(logits, k)
            seen["bhi"].append(out)
            return out

    # record the selections of the GPU run, then replay them on the CPU run
    seen = {"heads": [], "union": [], "bhi": []}
    saved = adapter.install(sde)
    try:
        topk, union = sde.topk_indices_rows, sde.union_neuron_indices

        def spy_topk(scores, k):
            out = topk(scores, k)
            seen["heads"].append(np.asarray(out))
            return out

        def spy_union(sets, layer=0):
            out = union(sets, layer)
            seen["union"].append(np.asarray(out))
            return out
        sde.topk_indices_rows, sde.union_neuron_indices = spy_topk, spy_union
        sde.BatchHeadIndex = _Heads
        got = sde.decode_step(session(1), model, tokens)
    finally:
        adapter.uninstall(sde, saved)
        sde.BatchHeadIndex = BHI
    assert sde.gqa_selective_attention_decode is saved["gqa_selective_attention_decode"]
    assert seen["union"] and seen["bhi"], "the reference engine did not route through the installed kernels"
    it_h, it_u = iter(seen["heads"]), iter(seen["union"])
    orig_topk, orig_union = sde.topk_indices_rows, sde.union_neuron_indices
    try:
        sde.topk_indices_rows = lambda scores, k: next(it_h)
        sde.union_neuron_indices = lambda sets, layer=0: next(it_u)
        _Heads.replay = iter(seen["bhi"])
        sde.BatchHeadIndex = _Heads
        ref = sde.decode_step(session(1), model, tokens)
    finally:
        sde.topk_indices_rows, sde.union_neuron_indices = orig_topk, orig_union
        sde.BatchHeadIndex = BHI
    rel = np.linalg.norm(np.asarray(got) - np.asarray(ref)) / np.linalg.norm(np.asarray(ref))
    assert rel <= 2e-2, rel
