"""Pin the CPU oracle against the reference's own outputs (CPU only).

``tests/golden/golden.npz`` was produced by the unmodified reference
(``tests/golden/make_golden.py``).  Selection results must match bit for
bit; floating-point results of this numpy restatement follow the same
float64 arithmetic, so they must match to ~1 ulp of float32.
"""

import math

import numpy as np
import pytest

from oracle import polar_oracle as po

from conftest import bf16_bits_to_f32


def test_topk_rows_bit_exact(golden):
    for i in range(int(golden["topk_n"])):
        s = golden[f"topk_scores_{i}"]
        k = int(golden[f"topk_k_{i}"])
        got = po.topk_indices_rows(s, k)
        assert np.array_equal(got, golden[f"topk_out_{i}"]), f"case {i}"


def test_topk_hand_kats():
    # tensors tie rules (reference tests/test_tensors.py:119-123,153-156)
    assert po.topk_indices(np.array([0.5, 0.5, 0.5]), 2).tolist() == [0, 1]
    assert po.topk_indices_rows(np.array([[0.5, 0.5, 0.1], [0.0, 1.0, 2.0]]), 2).tolist() == [[0, 1], [1, 2]]
    # SURVEY.md §7 hard parts: -0.0 ties +0.0; NaN ranks below -inf
    assert po.topk_indices(np.array([-0.0, 0.0, 0.5]), 2).tolist() == [0, 2]
    assert po.topk_indices(np.array([np.nan, 1, 2, np.nan, 0.5]), 4).tolist() == [0, 1, 2, 4]
    with pytest.raises(ValueError):
        po.topk_indices(np.array([1.0, 2.0]), 3)


def test_union_bit_exact(golden):
    for i in range(int(golden["union_n"])):
        got = po.union_neuron_indices(list(golden[f"union_rows_{i}"]))
        assert np.array_equal(got, golden[f"union_out_{i}"]), f"case {i}"
    assert po.union_neuron_indices([[1, 3], [3, 5]]).tolist() == [1, 3, 5]


def test_threshold_union(golden):
    assert np.array_equal(po.threshold_union(golden["thr_logits"], 0.0), golden["thr_union"])


def _cache_from(golden, i):
    keys = bf16_bits_to_f32(golden[f"attn_keys_{i}"])
    vals = bf16_bits_to_f32(golden[f"attn_values_{i}"])
    c = po.KVCache(*keys.shape)
    c.keys[:] = keys
    c.values[:] = vals
    c.lengths[:] = golden[f"attn_lengths_{i}"]
    return c


def test_attention_matches_reference(golden):
    for i in range(int(golden["attn_n"])):
        c = _cache_from(golden, i)
        q = golden[f"attn_q_{i}"]
        sel = golden[f"attn_sel_{i}"]
        got = po.gqa_selective_attention_decode(q, c, sel)
        ref = golden[f"attn_out_{i}"]
        assert np.abs(got - ref).max() <= 1e-6, f"case {i}"
        # independent two-pass check (reference tests/oracles.py:73-96 style)
        G = q.shape[1] // c.kv_heads
        naive = po.naive_attention_reference(q, c.keys, c.values, c.lengths, sel, G)
        assert np.abs(got - naive).max() <= 1e-5
        # non-selected heads are exactly zero
        for b in range(q.shape[0]):
            for g in range(c.kv_heads):
                if g not in sel[b]:
                    assert np.all(got[b, g * G:(g + 1) * G] == 0.0)


def test_attention_block_size_invariance(golden):
    c = _cache_from(golden, 0)
    q, sel = golden["attn_q_0"], golden["attn_sel_0"]
    base = po.gqa_selective_attention_decode(q, c, sel, block_size=37)
    for bc in (1, 2, 3, 8, 64, 100):
        out = po.gqa_selective_attention_decode(q, c, sel, block_size=bc)
        assert np.abs(out - base).max() <= 1e-5
    dfr = po.gqa_selective_attention_decode(q, c, sel, variant="deferred")
    assert np.abs(dfr - base).max() <= 1e-6


def test_attention_errors(golden):
    c = _cache_from(golden, 0)
    q, sel = golden["attn_q_0"], golden["attn_sel_0"]
    with pytest.raises(IndexError):
        po.gqa_selective_attention_decode(q, c, sel + c.kv_heads)
    with pytest.raises(ValueError):
        po.gqa_selective_attention_decode(q, c, np.zeros_like(sel))  # duplicate ids
    with pytest.raises(ValueError):
        po.gqa_selective_attention_decode(q, c, sel, scale=-1.0)
    c.lengths[1] = 0
    with pytest.raises(po.EmptyCache, match="1"):
        po.gqa_selective_attention_decode(q, c, sel)


def test_mlp_matches_reference(golden):
    g = golden
    x, w1, b1, w2, b2, idx = (g["mlp_x"], g["mlp_w1"], g["mlp_b1"], g["mlp_w2"],
                              g["mlp_b2"], g["mlp_idx"])
    assert np.array_equal(po.sparse_mlp_forward(x, w1, b1, w2, b2, idx), g["mlp_sparse"])
    assert np.array_equal(po.dense_mlp_forward(x, w1, b1, w2, b2), g["mlp_dense"])
    assert np.array_equal(po.selective_gemm(x[:, 0], w1, idx, "relu", b1), g["mlp_sgemm_relu"])
    assert np.array_equal(po.selective_gemm_t(g["mlp_h"], w2, idx, b2), g["mlp_sgemm_t"])
    assert np.abs(po.swiglu_mlp_forward(x, w1, g["mlp_w3"], w2, b2) - g["mlp_swiglu"]).max() <= 1e-6
    assert float(g["mlp_kat"].ravel()[0]) == 20.0


def test_routers_match_reference(golden):
    mr = po.init_mlp_router(64, 512, seed=5)
    hr = po.init_head_router(64, 8, seed=6)
    assert mr["w_in"].sum() == golden["router_mlp_w_in_sum"]
    assert mr["w_out"].sum() == golden["router_mlp_w_out_sum"]
    assert hr["w"].sum() == golden["router_head_w_sum"]
    x = golden["router_x"]
    assert np.array_equal(po.mlp_router_forward(mr["w_in"], mr["b_in"], mr["w_out"], mr["b_out"], x),
                          golden["router_mlp_logits"])
    assert np.array_equal(po.head_router_forward(hr["w"], hr["b"], x), golden["router_head_logits"])


def _model_checksum(m):
    tot = float(np.abs(m["embed"].astype(np.float64)).sum()
                + np.abs(m["pos_embed"].astype(np.float64)).sum()
                + np.abs(m["unembed"].astype(np.float64)).sum())
    for lw in m["layers"]:
        for k in ("ln1_g", "ln1_b", "w_q", "b_q", "w_k", "b_k", "w_v", "b_v", "w_o", "b_o",
                  "ln2_g", "ln2_b", "mlp_w1", "mlp_b1", "mlp_w2", "mlp_b2", "mlp_w3"):
            if lw[k] is not None:
                tot += float(np.abs(lw[k].astype(np.float64)).sum())
    return tot


@pytest.mark.parametrize("tag,kv_heads", [("mha", 8), ("gqa", 2)])
@pytest.mark.parametrize("mode", ["dense", "polar"])
def test_decode_step_matches_reference(golden, tag, kv_heads, mode):
    """BASELINE.json configs[0] end to end: one decode step, bit-exact
    selections and logits equal to the reference's."""
    m = po.random_model(2, 256, 1024, 8, kv_heads, 512, 288, seed=21)
    assert math.isclose(_model_checksum(m), float(golden[f"dec_{tag}_checksum"]), rel_tol=1e-12)
    rng = np.random.default_rng(22)  # bench.py:70-100 synthetic_session draw order
    caches = []
    for _ in range(2):
        c = po.KVCache(8, kv_heads, 288, 32)
        c.fill_random(rng, 256)
        caches.append(c)
    tokens = rng.integers(0, 512, 8, dtype=np.int64)
    assert np.array_equal(tokens, golden[f"dec_{tag}_{mode}_tokens"])
    mlp_r = [po.init_mlp_router(256, 1024, seed=30 + ell) for ell in range(2)]
    head_r = [po.init_head_router(256, kv_heads, seed=40 + ell) for ell in range(2)]
    rec = {}
    logits = po.decode_step(m, caches, tokens, mode=mode,
                            head_density=0.5 if mode == "polar" else 1.0,
                            k_table={0: 128, 1: 128} if mode == "polar" else None,
                            head_routers=head_r, mlp_routers=mlp_r, record=rec)
    for ell in range(2):
        assert np.array_equal(rec["heads"][ell], golden[f"dec_{tag}_{mode}_heads_{ell}"])
        if mode == "polar":
            assert np.array_equal(rec["union"][ell], golden[f"dec_{tag}_{mode}_union_{ell}"])
    assert np.array_equal(logits, golden[f"dec_{tag}_{mode}_logits"])


def test_single_unit_references(golden):
    """kernels.py:138-210 (OnlineSoftmaxState / online_softmax_attention) and
    tensors.py:83-113 (naive_softmax_attention_single_head), both variants."""
    for i in range(int(golden["unit_n"])):
        q, k, v = golden[f"unit_q_{i}"], golden[f"unit_k_{i}"], golden[f"unit_v_{i}"]
        scale = 1.0 / math.sqrt(q.shape[0])
        bs = int(golden[f"unit_bs_{i}"])
        np.testing.assert_allclose(po.naive_softmax_attention_single_head(q, k, v, scale),
                                   golden[f"unit_naive_{i}"], rtol=1e-6, atol=1e-7)
        for variant in ("running", "deferred"):
            out, st = po.online_softmax_attention(q, k, v, scale, bs, variant)
            np.testing.assert_allclose(out, golden[f"unit_online_{variant}_{i}"], rtol=1e-6, atol=1e-7)
            np.testing.assert_allclose([st.l_acc, st.m_acc], golden[f"unit_state_{variant}_{i}"], rtol=1e-12)
    np.testing.assert_allclose(po.matmul(golden["matmul_a"], golden["matmul_b"]), golden["matmul_out"],
                               rtol=1e-6, atol=1e-6)
