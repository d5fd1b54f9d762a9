"""Generate the golden fixtures that pin the CPU oracle (and the GPU path).

Runs ONLY in the build container, where the reference package is importable
from ``/root/reference/pkg/src``.  Every expected value below is produced by
the UNMODIFIED reference (``sparsedecode``); inputs are bf16-representable so
the device path can consume them without rounding.  The resulting
``golden.npz`` is committed; nothing on the GPU box reads /root/reference.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import sparsedecode as sd  # noqa: E402
from sparsedecode import bench as sd_bench  # noqa: E402
from sparsedecode import engine as sd_engine  # noqa: E402
from sparsedecode import kernels as sd_k  # noqa: E402
from sparsedecode import tensors as sd_t  # noqa: E402

from oracle.polar_oracle import round_bf16  # noqa: E402

OUT = {}


def put(name, arr):
    arr = np.asarray(arr)
    if arr.dtype == np.int64 and arr.ndim:
        arr = arr.astype(np.int32)  # index arrays: halve the fixture size
    OUT[name] = arr


def bf16_bits(a):
    """bf16-representable f32 -> its uint16 bf16 bit pattern (lossless)."""
    return (np.ascontiguousarray(a, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def rnd(rng, *shape, std=1.0):
    return round_bf16(rng.normal(0.0, std, shape).astype(np.float32))


def topk_cases():
    rng = np.random.default_rng(100)
    cases = [
        (np.array([[0.5, 0.5, 0.1], [0.0, 2.0, 1.0]], np.float32), 2),
        (np.array([[-0.0, 0.0, 0.5]], np.float32), 2),
        (np.array([[np.nan, 1.0, 2.0, np.nan, 0.5]], np.float32), 4),
        (np.array([[np.nan, -np.inf, np.inf, 0.0, -0.0, np.nan]], np.float32), 5),
        (np.array([[0.5, 0.5, 0.5, 0.5]], np.float32), 3),
    ]
    # random, with heavy ties (rounded) and specials sprinkled in
    for rows, cols, k in [(8, 8, 4), (64, 32, 16), (16, 72, 22), (16, 1024, 1),
                          (16, 1024, 128), (8, 1024, 1024), (4, 16384, 1638),
                          (3, 5000, 777)]:
        s = rng.normal(size=(rows, cols)).astype(np.float32)
        s[: rows // 2] = np.round(s[: rows // 2] * 2) / 2  # force ties
        m = rng.random((rows, cols))
        s[m < 0.01] = np.nan
        s[(m >= 0.01) & (m < 0.015)] = -0.0
        s[(m >= 0.015) & (m < 0.02)] = np.inf
        s[(m >= 0.02) & (m < 0.025)] = -np.inf
        cases.append((s, k))
    put("topk_n", len(cases))
    for i, (s, k) in enumerate(cases):
        put(f"topk_scores_{i}", s)
        put(f"topk_k_{i}", k)
        put(f"topk_out_{i}", sd_t.topk_indices_rows(s, k))


def union_cases():
    rng = np.random.default_rng(101)
    specs = [(2, 2, 8), (8, 128, 1024), (64, 100, 1024), (64, 1638, 16384), (1, 5, 64)]
    put("union_n", len(specs))
    for i, (b, k, width) in enumerate(specs):
        logits = rng.normal(size=(b, width)).astype(np.float32)
        rows = sd_t.topk_indices_rows(logits, k)
        put(f"union_rows_{i}", rows)
        put(f"union_width_{i}", width)
        put(f"union_out_{i}", sd_k.union_neuron_indices(list(rows)).indices)
    # threshold selection (routers.py predict: logit > 0)
    logits = rng.normal(size=(16, 512)).astype(np.float32) - 1.5
    put("thr_logits", logits)
    mask = logits > 0.0
    put("thr_union", np.flatnonzero(mask.any(axis=0)))


def attention_cases():
    rng = np.random.default_rng(102)
    specs = [
        # B, H, H_kv, d_h, cap, lengths, top_k
        (3, 4, 4, 32, 64, [37, 32, 11], 2),
        (2, 8, 2, 64, 96, [90, 17], 1),
        (2, 16, 16, 128, 208, [200, 129], 8),
        (4, 32, 8, 128, 72, [70, 1, 64, 65], 4),
        (2, 8, 8, 16, 40, [33, 40], 3),
        (3, 4, 4, 8, 16, [9, 14, 1], 4),
        (1, 32, 4, 128, 1032, [1030], 3),
    ]
    put("attn_n", len(specs))
    for i, (B, H, H_kv, d_h, cap, lens, k) in enumerate(specs):
        cache = sd_t.KVCache(B, H_kv, cap, d_h)
        for b, n in enumerate(lens):
            cache.append_tokens(b, rnd(rng, n, H_kv, d_h), rnd(rng, n, H_kv, d_h))
        q = rnd(rng, B, H, 1, d_h)
        sel = np.stack([np.sort(rng.choice(H_kv, size=k, replace=False)) for _ in range(B)])
        bhi = sd_k.BatchHeadIndex(sel.astype(np.int64))
        out = sd_k.gqa_selective_attention_decode(q, cache, bhi)
        put(f"attn_q_{i}", q)
        put(f"attn_keys_{i}", bf16_bits(cache.keys))
        put(f"attn_values_{i}", bf16_bits(cache.values))
        put(f"attn_lengths_{i}", cache.lengths)
        put(f"attn_sel_{i}", sel)
        put(f"attn_out_{i}", out)


def mlp_cases():
    rng = np.random.default_rng(103)
    B, d, D = 4, 64, 512
    x = rnd(rng, B, 1, d)
    w1 = rnd(rng, d, D, std=0.1)
    b1 = rnd(rng, D, std=0.1)
    w2 = rnd(rng, d, D, std=0.1)
    b2 = rnd(rng, d, std=0.1)
    idx = np.sort(rng.choice(D, size=200, replace=False)).astype(np.int64)
    put("mlp_x", x); put("mlp_w1", w1); put("mlp_b1", b1)
    put("mlp_w2", w2); put("mlp_b2", b2); put("mlp_idx", idx)
    put("mlp_sparse", sd_k.sparse_mlp_forward(x, w1, b1, w2, b2, idx))
    put("mlp_dense", sd_k.dense_mlp_forward(x, w1, b1, w2, b2))
    put("mlp_sgemm_relu", sd_k.selective_gemm(x[:, 0], w1, idx, "relu", b1))
    h = rnd(rng, B, idx.size)
    put("mlp_h", h)
    put("mlp_sgemm_t", sd_k.selective_gemm_t(h, w2, idx, b2))
    w3 = rnd(rng, d, D, std=0.1)
    put("mlp_w3", w3)
    put("mlp_swiglu", sd_k.swiglu_mlp_forward(x, w1, w3, w2, b2))
    # hand KAT (test_kernels_gemm.py:132-139): relu(2*3-1)*4 = 20
    put("mlp_kat", sd_k.dense_mlp_forward(np.array([[[2.0]]], np.float32),
                                          np.array([[3.0]], np.float32),
                                          np.array([-1.0], np.float32),
                                          np.array([[4.0]], np.float32),
                                          np.array([0.0], np.float32)))


def router_cases():
    rng = np.random.default_rng(104)
    mr = sd.MlpRouter(64, 512, seed=5)
    hr = sd.HeadRouter(64, 8, seed=6)
    x = rnd(rng, 6, 64)
    put("router_x", x)
    put("router_mlp_logits", mr.decision_function(x))
    put("router_head_logits", hr.decision_function(x))
    put("router_mlp_w_in_sum", mr.w_in_.sum())
    put("router_mlp_w_out_sum", mr.w_out_.sum())
    put("router_head_w_sum", hr.w_.sum())


def decode_cases():
    """BASELINE.json configs[0]: tiny OPT-style decoder, B=8, ctx 256."""
    for tag, kv_heads in (("mha", 8), ("gqa", 2)):
        cfg = sd.TransformerConfig(layers=2, model_dim=256, ffn_dim=1024, heads=8,
                                   kv_heads=kv_heads, vocab=512, max_seq=288,
                                   activation="relu")
        model = sd.random_model(cfg, seed=21)
        put(f"dec_{tag}_checksum", model.checksum())
        ktab = sd.LayerKTable(rows=tuple((ell, 128, 0.99) for ell in range(cfg.layers)))
        mlp_r = [sd.MlpRouter(cfg.model_dim, cfg.ffn_dim, seed=30 + ell) for ell in range(2)]
        head_r = [sd.HeadRouter(cfg.model_dim, cfg.kv_heads, seed=40 + ell) for ell in range(2)]
        for mode, rho in (("dense", 1.0), ("polar", 0.5)):
            policy = sd_engine.SparsityPolicy(mode=mode, mlp_k_table=ktab if mode != "dense" else None,
                                              head_density=rho)
            sess = sd_bench.synthetic_session(model, 8, 256, policy=policy,
                                              mlp_routers=mlp_r, head_routers=head_r, seed=22)
            seen = {"heads": [], "union": []}
            orig_attn = sd_engine.gqa_selective_attention_decode
            orig_mlp = sd_engine.sparse_mlp_forward

            def spy_attn(q, cache, bhi, *a, **kw):
                seen["heads"].append(bhi.entries.copy())
                return orig_attn(q, cache, bhi, *a, **kw)

            def spy_mlp(x, w1, b1, w2, b2, active):
                seen["union"].append(active.indices.copy())
                return orig_mlp(x, w1, b1, w2, b2, active)

            sd_engine.gqa_selective_attention_decode = spy_attn
            sd_engine.sparse_mlp_forward = spy_mlp
            try:
                tokens = sess.next_tokens.copy()
                logits = sd_engine.decode_step(sess, model, tokens)
            finally:
                sd_engine.gqa_selective_attention_decode = orig_attn
                sd_engine.sparse_mlp_forward = orig_mlp
            put(f"dec_{tag}_{mode}_tokens", tokens)
            put(f"dec_{tag}_{mode}_logits", logits)
            for ell, h in enumerate(seen["heads"]):
                put(f"dec_{tag}_{mode}_heads_{ell}", h)
            for ell, u in enumerate(seen["union"]):
                put(f"dec_{tag}_{mode}_union_{ell}", u)


def unit_cases():
    """Single-unit references (kernels.py:138-210, tensors.py:83-113)."""
    rng = np.random.default_rng(600)
    cases = [(1, 32, 1), (7, 32, 3), (300, 128, 64), (257, 64, 8), (50, 16, 50)]
    put("unit_n", len(cases))
    for i, (n, d_h, bs) in enumerate(cases):
        q, k, v = rnd(rng, d_h), rnd(rng, n, d_h), rnd(rng, n, d_h)
        scale = 1.0 / math.sqrt(d_h)
        put(f"unit_q_{i}", q)
        put(f"unit_k_{i}", k)
        put(f"unit_v_{i}", v)
        put(f"unit_bs_{i}", bs)
        put(f"unit_naive_{i}", sd_t.naive_softmax_attention_single_head(q, k, v, scale))
        for variant in ("running", "deferred"):
            out, st = sd_k.online_softmax_attention(q, k, v, scale, sd_k.FlashBlockParams(bs), variant)
            put(f"unit_online_{variant}_{i}", out)
            put(f"unit_state_{variant}_{i}", np.array([st.l_acc, st.m_acc]))
    a, b = rnd(rng, 5, 300), rnd(rng, 300, 700)
    put("matmul_a", a)
    put("matmul_b", b)
    put("matmul_out", sd_t.matmul(a, b))


def main():
    topk_cases()
    union_cases()
    attention_cases()
    mlp_cases()
    router_cases()
    decode_cases()
    unit_cases()
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **OUT)
    print(f"wrote {path}: {len(OUT)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
