"""GPU decode step (engine.py) vs the reference on BASELINE.json configs[0]:
tiny OPT-style decoder, 2 layers, d=256, 8 heads, ReLU MLP, batch 8, ctx 256.

* head and neuron selections are bit-exact to the reference rule applied
  to the GPU router's own logits (top-k / union given identical logits);
* logits match the reference's (golden) within bf16 tolerance;
* the CUDA-graph replay matches the eager step (to f32 rounding).
"""

import numpy as np
import pytest
import torch

from oracle import polar_oracle as po

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_14884_b200 as pb  # noqa: E402
from paper_2505_14884_b200.engine import DecodeEngine, SparsityPolicy  # noqa: E402
from paper_2505_14884_b200.model import DeviceModel, TransformerConfig  # noqa: E402


def _engine(kv_heads, mode, record=False, **kw):
    cfg = TransformerConfig(2, 256, 1024, 8, kv_heads, 512, 288, "relu")
    host = po.random_model(2, 256, 1024, 8, kv_heads, 512, 288, seed=21)
    model = DeviceModel.from_host(cfg, host)
    polar = mode == "polar"
    policy = SparsityPolicy(mode=mode, mlp_k_table={0: 128, 1: 128} if polar else None,
                            head_density=0.5 if polar else 1.0)
    hr = [pb.HeadRouter(256, kv_heads, seed=40 + ell) for ell in range(2)]
    mr = [pb.MlpRouter(256, 1024, seed=30 + ell) for ell in range(2)]
    eng = DecodeEngine(model, 8, 288, policy, head_routers=hr, mlp_routers=mr, **kw)
    rng = np.random.default_rng(22)  # reference bench.py:70-100 draw order
    for c in eng.caches:
        c.fill_random(rng, 256)
    tokens = rng.integers(0, 512, 8, dtype=np.int64)
    if record:
        eng.record = {}
    return eng, tokens


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("tag,kv_heads", [("mha", 8), ("gqa", 2)])
def test_dense_step_matches_reference(golden, tag, kv_heads):
    eng, tokens = _engine(kv_heads, "dense")
    assert np.array_equal(tokens, golden[f"dec_{tag}_dense_tokens"])
    logits = eng.step(tokens).cpu().numpy()
    ref = golden[f"dec_{tag}_dense_logits"]
    assert _rel(logits, ref) <= 2e-2
    assert np.abs(logits - ref).max() <= 2e-2 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("tag,kv_heads", [("mha", 8), ("gqa", 2)])
def test_polar_step_selection_and_logits(golden, tag, kv_heads):
    eng, tokens = _engine(kv_heads, "polar", record=True)
    logits = eng.step(tokens).cpu().numpy()
    rec = eng.record
    # layer 0 dense (layer0_dense_attention), layer 1 routed: bit-exact given logits
    assert len(rec["heads"]) == 1
    hl = rec["head_logits"][0].cpu().numpy()
    assert np.array_equal(rec["heads"][0].cpu().numpy(), po.topk_indices_rows(hl, 4 if kv_heads == 8 else 1))
    for ell in range(2):
        ml = rec["mlp_logits"][ell].cpu().numpy()
        ref_union = po.union_neuron_indices(list(po.topk_indices_rows(ml, 128)))
        assert np.array_equal(rec["union"][ell].cpu().numpy(), ref_union)
    # logits vs the oracle decode step run with the device's (checked) selections
    host = po.random_model(2, 256, 1024, 8, kv_heads, 512, 288, seed=21)
    rng = np.random.default_rng(22)
    caches = []
    for _ in range(2):
        c = po.KVCache(8, kv_heads, 288, 32)
        c.fill_random(rng, 256)
        caches.append(c)
    forced = {"heads": {1: rec["heads"][0].cpu().numpy()},
              "union": {e: rec["union"][e].cpu().numpy() for e in range(2)}}
    ref = po.decode_step(host, caches, tokens, mode="polar", head_density=0.5, k_table={0: 128, 1: 128},
                         head_routers=[None, None], mlp_routers=[po.init_mlp_router(256, 1024, seed=30 + e)
                                                                 for e in range(2)],
                         forced=forced)
    assert _rel(logits, ref) <= 2e-2
    # when the bf16 routers pick the reference's exact sets, match its golden logits too
    if np.array_equal(rec["heads"][0].cpu().numpy(), golden[f"dec_{tag}_polar_heads_1"]) and all(
            np.array_equal(rec["union"][e].cpu().numpy(), golden[f"dec_{tag}_polar_union_{e}"]) for e in range(2)):
        assert _rel(logits, golden[f"dec_{tag}_polar_logits"]) <= 2e-2


@pytest.mark.parametrize("mode,concurrent", [("dense", False), ("polar", False), ("polar", True)])
def test_graph_replay_equals_eager(mode, concurrent):
    """Graph replay == eager; with concurrent=True the head router runs on a
    side stream (a parallel branch of the captured graph)."""
    eng_a, tokens = _engine(8, mode)
    eng_b, _ = _engine(8, mode, concurrent_router=concurrent)
    eng_b.capture()
    for _ in range(3):
        la = eng_a.step(tokens).clone()
        lb = eng_b.step(tokens).clone()
        # shared GEMM tiles are reduced with f32 atomics: equal up to f32 rounding
        assert torch.allclose(la, lb, rtol=1e-4, atol=1e-5)
    assert np.array_equal(eng_a.host_lengths, eng_b.host_lengths)
    assert eng_b.caches[1].lengths.cpu().tolist() == [259] * 8


def test_capacity_error():
    eng, tokens = _engine(8, "dense")
    for c in eng.caches:
        c.set_lengths([287] * 8)
    eng.step(tokens)
    with pytest.raises(pb.CapacityError):
        eng.step(tokens)


def test_missing_router_is_configuration_error():
    cfg = TransformerConfig(2, 256, 1024, 8, 8, 512, 288, "relu")
    model = DeviceModel.random(cfg)
    with pytest.raises(pb.ConfigurationError):
        DecodeEngine(model, 2, 64, SparsityPolicy(mode="polar", head_density=0.5))
    with pytest.raises(pb.ConfigurationError):
        DecodeEngine(model, 2, 64, SparsityPolicy(mode="dejavu_mlp"))


@pytest.mark.parametrize("B", [1, 3])
def test_small_batch_polar_step_vs_oracle(B):
    """B <= 4 decodes through the gathered-GEMV UP projection: selections
    bit-exact given the device logits, logits within tolerance of the oracle
    forced to the same selections, eager and graph replay agree."""
    cfg = TransformerConfig(2, 256, 1024, 8, 8, 512, 288, "relu")
    host = po.random_model(2, 256, 1024, 8, 8, 512, 288, seed=21)
    model = DeviceModel.from_host(cfg, host)
    policy = SparsityPolicy(mode="polar", mlp_k_table={0: 128, 1: 128}, head_density=0.5)
    hr = [pb.HeadRouter(256, 8, seed=40 + ell) for ell in range(2)]
    mr = [pb.MlpRouter(256, 1024, seed=30 + ell) for ell in range(2)]
    eng = DecodeEngine(model, B, 288, policy, head_routers=hr, mlp_routers=mr)
    rng = np.random.default_rng(5)
    for c in eng.caches:
        c.fill_random(rng, 200)
    tokens = rng.integers(0, 512, B, dtype=np.int64)
    eng.record = {}
    logits = eng.step(tokens).cpu().numpy()
    rec = eng.record
    hl = rec["head_logits"][0].cpu().numpy()
    assert np.array_equal(rec["heads"][0].cpu().numpy(), po.topk_indices_rows(hl, 4))
    for ell in range(2):
        ml = rec["mlp_logits"][ell].cpu().numpy()
        assert np.array_equal(rec["union"][ell].cpu().numpy(),
                              po.union_neuron_indices(list(po.topk_indices_rows(ml, 128))))
    rng = np.random.default_rng(5)
    caches = []
    for _ in range(2):
        c = po.KVCache(B, 8, 288, 32)
        c.fill_random(rng, 200)
        caches.append(c)
    forced = {"heads": {1: rec["heads"][0].cpu().numpy()},
              "union": {e: rec["union"][e].cpu().numpy() for e in range(2)}}
    ref = po.decode_step(host, caches, tokens, mode="polar", head_density=0.5, k_table={0: 128, 1: 128},
                         head_routers=[None, None],
                         mlp_routers=[po.init_mlp_router(256, 1024, seed=30 + e) for e in range(2)], forced=forced)
    assert _rel(logits, ref) <= 2e-2
    # graph replay of the next step == an eager step from the same state
    eng.record = None
    eng2 = DecodeEngine(model, B, 288, policy, head_routers=hr, mlp_routers=mr)
    rng = np.random.default_rng(5)
    for c in eng2.caches:
        c.fill_random(rng, 200)
    eng2.step(tokens)
    eng2.capture()
    a = eng.step(tokens).clone()
    b = eng2.step(tokens).clone()
    assert torch.allclose(a, b, rtol=1e-4, atol=1e-5)
