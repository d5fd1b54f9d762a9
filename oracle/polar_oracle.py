"""CPU oracle for the Polar Sparsity batched-decode hot path.

TEST INFRASTRUCTURE ONLY.  This module restates, in plain numpy, the
algorithm of the reference package ``sparsedecode`` (``/root/reference/pkg``)
for the functions on the decode hot path.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
it -- always as the checker / reported CPU baseline, never as the thing
measured or shipped.  The product path (``paper_2505_14884_b200``) never
imports this file and fails loudly when its CUDA library is missing.

Parity is PINNED: ``tests/golden/make_golden.py`` imports the real reference
from ``/root/reference/pkg/src`` in the build container and records its
outputs (top-k rows, unions, attention, MLPs, routers, one full polar decode
step) into ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks
this restatement against every fixture.

Numerics follow the reference: float32 storage, float64 accumulation,
float32 results.  Every function cites the reference file:line it restates
(paths relative to ``/root/reference/pkg/src/sparsedecode``).
"""

from __future__ import annotations

import math

import numpy as np

F32 = np.float32
# tensors.py:24-26 -- shared output-column tile of matmul / selective GEMM.
TILE = 256
# model.py:20
LN_EPS = 1e-5


class EmptyCache(ValueError):
    """exceptions.py:4-5 (EmptyCacheError is a ValueError)."""


class Capacity(RuntimeError):
    """exceptions.py:8-9 (CapacityError is a RuntimeError)."""


# ---------------------------------------------------------------------------
# bf16 helpers (synthetic inputs are generated bf16-representable so the
# device path sees exactly the values the oracle sees)
# ---------------------------------------------------------------------------

def round_bf16(x) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even), keep f32."""
    a = np.ascontiguousarray(np.asarray(x, dtype=F32))
    u = a.view(np.uint32).astype(np.uint64)
    nan = np.isnan(a)
    bias = ((u >> 16) & 1) + 0x7FFF
    r = ((u + bias) >> 16) << 16
    out = r.astype(np.uint32).view(F32).reshape(a.shape)
    out = np.where(nan, np.float32(np.nan), out)
    return out.astype(F32)


# ---------------------------------------------------------------------------
# selection: top-k, union, threshold
# ---------------------------------------------------------------------------

def topk_indices(scores, k: int) -> np.ndarray:
    """tensors.py:54-62 -- k largest, ascending, ties to the lower index."""
    s = np.asarray(scores)
    if s.ndim != 1:
        raise ValueError("scores must be 1-dimensional")
    if not 1 <= k <= s.size:
        raise ValueError(f"k must be in [1, {s.size}], got {k}")
    return np.sort(np.argsort(-s, kind="stable")[:k]).astype(np.int64)


def topk_indices_rows(scores, k: int) -> np.ndarray:
    """tensors.py:65-73 -- row-wise top-k with the same tie rule.

    Note the ordering this inherits from numpy's stable argsort of
    ``-scores``: -0.0 ties with +0.0 and NaN sorts after every number
    (so NaN ranks below -inf), NaNs tied among themselves by index.
    """
    s = np.asarray(scores)
    if s.ndim != 2:
        raise ValueError("scores must be 2-dimensional")
    if not 1 <= k <= s.shape[1]:
        raise ValueError(f"k must be in [1, {s.shape[1]}], got {k}")
    order = np.argsort(-s, axis=1, kind="stable")[:, :k]
    return np.sort(order, axis=1).astype(np.int64)


def union_neuron_indices(per_sequence_sets) -> np.ndarray:
    """kernels.py:376-383 -- sorted, de-duplicated union (np.unique)."""
    parts = [np.asarray(s, dtype=np.int64).reshape(-1) for s in per_sequence_sets]
    if not parts:
        return np.empty(0, dtype=np.int64)
    return np.unique(np.concatenate(parts)).astype(np.int64)


def threshold_rows(logits, threshold: float = 0.0) -> np.ndarray:
    """routers.py:188-190 -- ``predict``: active iff logit > threshold (0 =
    sigmoid(logit) > 0.5).  Returns a boolean (rows, width) mask."""
    return np.asarray(logits, dtype=F32) > np.float32(threshold)


def threshold_union(logits, threshold: float = 0.0) -> np.ndarray:
    """Union over the batch of the threshold-selected neurons, ascending."""
    return np.flatnonzero(threshold_rows(logits, threshold).any(axis=0)).astype(np.int64)


def head_budget(density: float, n_route: int) -> int:
    """engine.py:64-65 -- per-layer head (KV-group) budget."""
    return max(1, math.ceil(density * n_route - 1e-9))


# ---------------------------------------------------------------------------
# routers (forward only)
# ---------------------------------------------------------------------------

def head_router_forward(w, b, x) -> np.ndarray:
    """routers.py:324-325 + 178-186 -- f64 affine, cast to f32."""
    x64 = np.atleast_2d(np.asarray(x, dtype=np.float64))
    return (x64 @ np.asarray(w, np.float64) + np.asarray(b, np.float64)).astype(F32)


def mlp_router_forward(w_in, b_in, w_out, b_out, x) -> np.ndarray:
    """routers.py:286-288 + 178-186 -- relu MLP in f64, cast to f32."""
    x64 = np.atleast_2d(np.asarray(x, dtype=np.float64))
    h = np.maximum(x64 @ np.asarray(w_in, np.float64) + np.asarray(b_in, np.float64), 0.0)
    return (h @ np.asarray(w_out, np.float64) + np.asarray(b_out, np.float64)).astype(F32)


def init_mlp_router(d_model: int, ffn_dim: int, hidden_dim=None, seed: int = 0):
    """routers.py:272-284 -- same RNG draw order as ``MlpRouter.__init__``."""
    h = hidden_dim if hidden_dim is not None else min(1024, 4 * d_model)
    rng = np.random.default_rng(seed)
    w_in = rng.normal(0.0, math.sqrt(2.0 / d_model), (d_model, h))
    w_out = rng.normal(0.0, math.sqrt(2.0 / h), (h, ffn_dim))
    return {"w_in": w_in, "b_in": np.zeros(h), "w_out": w_out, "b_out": np.zeros(ffn_dim)}


def init_head_router(d_model: int, n_heads: int, seed: int = 0):
    """routers.py:313-322 -- same RNG draw order as ``HeadRouter.__init__``."""
    rng = np.random.default_rng(seed)
    return {"w": rng.normal(0.0, 1.0 / math.sqrt(d_model), (d_model, n_heads)),
            "b": np.zeros(n_heads)}


# ---------------------------------------------------------------------------
# dense substrate
# ---------------------------------------------------------------------------

def matmul64(a, b) -> np.ndarray:
    """tensors.py:42-51 -- f64 product computed in 256-column tiles."""
    a64 = np.asarray(a, dtype=np.float64)
    b = np.asarray(b)
    out = np.empty((a64.shape[0], b.shape[1]))
    for c0 in range(0, b.shape[1], TILE):
        c1 = min(c0 + TILE, b.shape[1])
        out[:, c0:c1] = a64 @ np.ascontiguousarray(b[:, c0:c1], dtype=np.float64)
    return out


def matmul(a, b) -> np.ndarray:
    """tensors.py:29-39."""
    return matmul64(np.asarray(a, F32), np.asarray(b, F32)).astype(F32)


def naive_softmax_attention_single_head(q, keys, values, scale) -> np.ndarray:
    """tensors.py:83-113 -- two-pass max-subtract softmax, f64 inside."""
    q = np.asarray(q, F32)
    keys = np.asarray(keys, F32)
    values = np.asarray(values, F32)
    if keys.shape[0] == 0:
        raise EmptyCache("attention over an empty key/value history")
    s = scale * (keys.astype(np.float64) @ q.astype(np.float64))
    s -= s.max()
    p = np.exp(s)
    return ((p @ values.astype(np.float64)) / p.sum()).astype(F32)


class OnlineSoftmaxState:
    """kernels.py:138-180 -- (o, l, m) of the one-pass softmax, f64."""

    def __init__(self, head_dim):
        self.o_acc = np.zeros(head_dim, np.float64)
        self.l_acc = 0.0
        self.m_acc = -math.inf

    def update(self, scores, v_block, variant="running"):
        scores = np.asarray(scores, np.float64)
        v_block = np.asarray(v_block, np.float64)
        m_tilde = scores.max()
        p = np.exp(scores - m_tilde)
        l_tilde = p.sum()
        m_new = max(self.m_acc, m_tilde)
        alpha = math.exp(self.m_acc - m_new)
        beta = math.exp(m_tilde - m_new)
        l_new = alpha * self.l_acc + beta * l_tilde
        pv = p @ v_block
        if variant == "running":
            self.o_acc = (alpha * self.l_acc * self.o_acc + beta * pv) / l_new
        else:
            self.o_acc = alpha * self.o_acc + beta * pv
        self.l_acc, self.m_acc = l_new, m_new

    def output(self, variant="running"):
        return self.o_acc / self.l_acc if variant == "deferred" else self.o_acc


def online_softmax_attention(q, keys, values, scale, block_size=64, variant="running"):
    """kernels.py:183-210 -- single-unit blocked attention; (out f32, state)."""
    q64 = np.asarray(q, F32).astype(np.float64)
    keys = np.asarray(keys, F32)
    values = np.asarray(values, F32)
    if keys.shape[0] == 0:
        raise EmptyCache("attention over an empty key/value history")
    n = keys.shape[0]
    st = OnlineSoftmaxState(q64.shape[0])
    for j in range(-(-n // block_size)):
        k0, k1 = j * block_size, min((j + 1) * block_size, n)
        st.update(scale * (keys[k0:k1].astype(np.float64) @ q64), values[k0:k1], variant)
    return st.output(variant).astype(F32), st


def layernorm(x, g, b) -> np.ndarray:
    """model.py:168-175 -- f64 inside, f32 out, eps 1e-5."""
    x64 = np.asarray(x, dtype=np.float64)
    mu = x64.mean(axis=-1, keepdims=True)
    var = x64.var(axis=-1, keepdims=True)
    y = (x64 - mu) / np.sqrt(var + LN_EPS)
    return (y * np.asarray(g, np.float64) + np.asarray(b, np.float64)).astype(F32)


# ---------------------------------------------------------------------------
# selective GEMM / MLP
# ---------------------------------------------------------------------------

def _cols64(b: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """kernels.py:213-220 -- gathered columns of b as f64 (slice when the
    run is contiguous; values are identical either way)."""
    return np.take(b, idx, axis=1).astype(np.float64)


def _up64(a, b, idx, activation, bias) -> np.ndarray:
    """kernels.py:223-240 -- act(a @ b[:, idx] + bias[idx]) tile by tile."""
    a64 = np.asarray(a, F32).astype(np.float64)
    out = np.empty((a64.shape[0], idx.size))
    for t0 in range(0, idx.size, TILE):
        sel = idx[t0:t0 + TILE]
        out[:, t0:t0 + sel.size] = a64 @ _cols64(b, sel)
    if bias is not None:
        out += np.asarray(bias, F32).astype(np.float64)[idx]
    if activation == "relu":
        np.maximum(out, 0.0, out=out)
    return out


def _down64(h64, b, idx, bias) -> np.ndarray:
    """kernels.py:243-256 -- h @ b[:, idx].T + bias, accumulated per tile."""
    out = np.zeros((h64.shape[0], b.shape[0]))
    for t0 in range(0, idx.size, TILE):
        sel = idx[t0:t0 + TILE]
        out += h64[:, t0:t0 + sel.size] @ _cols64(b, sel).T
    if bias is not None:
        out += np.asarray(bias, F32).astype(np.float64)
    return out


def _idx(indices, upper: int) -> np.ndarray:
    """kernels.py:259-265 + validation.py:58-70."""
    idx = np.asarray(indices)
    if idx.ndim != 1:
        raise ValueError("indices must be 1-dimensional")
    idx = idx.astype(np.int64)
    if idx.size == 0:
        raise ValueError("indices must select at least one column")
    if idx.min() < 0:
        raise IndexError("negative index")
    if idx.max() >= upper:
        raise IndexError(f"index >= {upper}")
    return idx


def selective_gemm(a, b, indices, activation="none", bias=None) -> np.ndarray:
    """kernels.py:268-291."""
    b = np.asarray(b, F32)
    a = np.asarray(a, F32)
    if a.shape[1] != b.shape[0]:
        raise ValueError("inner dimension mismatch")
    return _up64(a, b, _idx(indices, b.shape[1]), activation, bias).astype(F32)


def selective_gemm_t(a, b, indices, bias=None) -> np.ndarray:
    """kernels.py:294-310."""
    b = np.asarray(b, F32)
    idx = _idx(indices, b.shape[1])
    a = np.asarray(a, F32)
    if a.shape[1] != idx.size:
        raise ValueError("a must have len(indices) columns")
    return _down64(a.astype(np.float64), b, idx, bias).astype(F32)


def sparse_mlp_forward(x, w1, b1, w2, b2, active) -> np.ndarray:
    """kernels.py:353-373 -- hidden stays f64 between the projections."""
    x = np.asarray(x, F32)
    w1 = np.asarray(w1, F32)
    w2 = np.asarray(w2, F32)
    batch, _, d = x.shape
    idx = _idx(active, w1.shape[1])
    h = _up64(x[:, 0, :], w1, idx, "relu", b1)
    return _down64(h, w2, idx, b2).astype(F32).reshape(batch, 1, d)


def dense_mlp_forward(x, w1, b1, w2, b2) -> np.ndarray:
    """kernels.py:313-332 -- the selective path over every neuron."""
    return sparse_mlp_forward(x, w1, b1, w2, b2, np.arange(np.asarray(w1).shape[1]))


def swiglu_mlp_forward(x, w1, w3, w2, b2) -> np.ndarray:
    """kernels.py:335-350 -- dense gated MLP."""
    x = np.asarray(x, F32)
    batch, _, d = x.shape
    x64 = x[:, 0, :].astype(np.float64)
    gate = x64 @ np.asarray(w1, np.float64)
    gate *= 1.0 / (1.0 + np.exp(-gate))
    up = x64 @ np.asarray(w3, np.float64)
    y = (gate * up) @ np.asarray(w2, np.float64).T + np.asarray(b2, np.float64)
    return y.astype(F32).reshape(batch, 1, d)


# ---------------------------------------------------------------------------
# KV cache + Select-Head Attention
# ---------------------------------------------------------------------------

class KVCache:
    """tensors.py:116-213 -- (B, H_kv, cap, d_h) f32 history + lengths."""

    def __init__(self, batch, kv_heads, capacity, head_dim):
        self.keys = np.zeros((batch, kv_heads, capacity, head_dim), F32)
        self.values = np.zeros_like(self.keys)
        self.lengths = np.zeros(batch, np.int64)

    @property
    def batch(self):
        return self.keys.shape[0]

    @property
    def kv_heads(self):
        return self.keys.shape[1]

    @property
    def capacity(self):
        return self.keys.shape[2]

    @property
    def head_dim(self):
        return self.keys.shape[3]

    def append_step(self, k_new, v_new):
        """tensors.py:150-170."""
        if (self.lengths >= self.capacity).any():
            raise Capacity(f"KV cache capacity {self.capacity} exhausted")
        rows = np.arange(self.batch)
        self.keys[rows, :, self.lengths, :] = np.asarray(k_new, F32)
        self.values[rows, :, self.lengths, :] = np.asarray(v_new, F32)
        self.lengths += 1

    def append_tokens(self, b, k_tokens, v_tokens):
        """tensors.py:172-192."""
        k_tokens = np.asarray(k_tokens, F32)
        t = k_tokens.shape[0]
        s = int(self.lengths[b])
        if s + t > self.capacity:
            raise Capacity("capacity exceeded")
        self.keys[b, :, s:s + t] = k_tokens.transpose(1, 0, 2)
        self.values[b, :, s:s + t] = np.asarray(v_tokens, F32).transpose(1, 0, 2)
        self.lengths[b] = s + t

    def fill_random(self, rng, length):
        """tensors.py:201-213 -- same draw order (keys then values)."""
        shape = (self.batch, self.kv_heads, length, self.head_dim)
        self.keys[:, :, :length] = rng.standard_normal(shape, dtype=F32)
        self.values[:, :, :length] = rng.standard_normal(shape, dtype=F32)
        self.lengths[:] = length


def _attend_units(q4, keys, values, lengths, b_idx, q_heads, kv_heads,
                  block_size, scale, deferred=False) -> np.ndarray:
    """kernels.py:386-444 -- blocked online softmax over (b, head) units.

    Units are grouped by cache length; each walks its K/V rows in blocks of
    ``block_size`` with the running-normalised recurrence (Alg. 3).  The
    output starts at zero, so non-selected heads stay exactly 0.0 and their
    cache rows are never touched.
    """
    out = np.zeros_like(q4)
    if b_idx.size == 0:
        return out
    lens = lengths[b_idx]
    q64 = q4[b_idx, q_heads, 0, :].astype(np.float64)
    d_h = q4.shape[3]
    for n in np.unique(lens):
        n = int(n)
        grp = np.nonzero(lens == n)[0]
        bu, ku, qg = b_idx[grp], kv_heads[grp], q64[grp]
        m = np.full(grp.size, -np.inf)
        l = np.zeros(grp.size)
        o = np.zeros((grp.size, d_h))
        for k0 in range(0, n, block_size):
            k1 = min(k0 + block_size, n)
            kb = keys[bu, ku, k0:k1, :]
            vb = values[bu, ku, k0:k1, :]
            s = scale * np.einsum("ud,ukd->uk", qg, kb, dtype=np.float64)
            mt = s.max(axis=1)
            p = np.exp(s - mt[:, None])
            lt = p.sum(axis=1)
            pv = np.einsum("uk,ukd->ud", p, vb, dtype=np.float64)
            mn = np.maximum(m, mt)
            al = np.exp(m - mn)
            be = np.exp(mt - mn)
            ln = al * l + be * lt
            if deferred:
                o = al[:, None] * o + be[:, None] * pv
            else:
                o = ((al * l)[:, None] * o + be[:, None] * pv) / ln[:, None]
            l, m = ln, mn
        if deferred:
            o = o / l[:, None]
        out[bu, q_heads[grp], 0, :] = o.astype(F32)
    return out


def _check_rows(sel):
    """kernels.py:80-92 -- BatchHeadIndex invariants."""
    sel = np.asarray(sel)
    if sel.ndim != 2 or sel.size == 0:
        raise ValueError("selection must be a non-empty 2-D array")
    sel = sel.astype(np.int64)
    if sel.min() < 0:
        raise IndexError("head ids must be non-negative")
    for row in sel:
        if np.unique(row).size != row.size:
            raise ValueError("head ids must be unique within a row")
    return sel


def gqa_selective_attention_decode(q, cache: KVCache, selection, block_size=64,
                                   scale=None, variant="running") -> np.ndarray:
    """kernels.py:513-548 (+ _check_attention_args 447-461).

    Selecting KV group g activates query heads g*G .. g*G+G-1.  With
    G == 1 this is ``selective_head_flash_attention_decode`` (464-510).
    """
    q4 = np.asarray(q, F32)
    if q4.ndim != 4 or q4.shape[2] != 1:
        raise ValueError("q must be (B, H, 1, d_h)")
    batch, n_heads, _, d_h = q4.shape
    if scale is None:
        scale = 1.0 / math.sqrt(d_h)
    sel = _check_rows(selection)
    if cache.batch != batch or cache.head_dim != d_h:
        raise ValueError("cache inconsistent with query")
    if sel.shape[0] != batch:
        raise ValueError("selection batch mismatch")
    if (cache.lengths < 1).any():
        raise EmptyCache(f"sequences {np.nonzero(cache.lengths < 1)[0].tolist()} have empty caches")
    if not scale > 0:
        raise ValueError("scale must be positive")
    n_groups = cache.kv_heads
    if n_heads % n_groups:
        raise ValueError("heads not divisible by groups")
    G = n_heads // n_groups
    if sel.max() >= n_groups:
        raise IndexError(f"group ids must be < {n_groups}")
    k = sel.shape[1]
    b_idx = np.repeat(np.arange(batch, dtype=np.int64), k * G)
    groups = np.repeat(sel.reshape(-1), G)
    q_heads = groups * G + np.tile(np.arange(G, dtype=np.int64), batch * k)
    return _attend_units(q4, cache.keys, cache.values, cache.lengths, b_idx,
                         q_heads, groups, int(block_size), float(scale),
                         deferred=(variant == "deferred"))


def selective_head_flash_attention_decode(q, cache, selection, block_size=64,
                                          scale=None, variant="running"):
    """kernels.py:464-510 -- MHA entry; requires cache.kv_heads == H."""
    if cache.kv_heads != np.asarray(q).shape[1]:
        raise ValueError("use gqa_selective_attention_decode for grouped KV")
    return gqa_selective_attention_decode(q, cache, selection, block_size, scale, variant)


def naive_attention_reference(q4, keys, values, lengths, rows, group_size=1, scale=None):
    """Two-pass softmax per unit (an independent check, like the reference
    tests' ``selective_attention_reference``, tests/oracles.py:73-96)."""
    q4 = np.asarray(q4, np.float64)
    batch, n_heads, _, d_h = q4.shape
    scale = 1.0 / math.sqrt(d_h) if scale is None else scale
    out = np.zeros((batch, n_heads, 1, d_h))
    for b in range(batch):
        n = int(lengths[b])
        for g in rows[b]:
            kk = np.asarray(keys[b, int(g), :n], np.float64)
            vv = np.asarray(values[b, int(g), :n], np.float64)
            for off in range(group_size):
                h = int(g) * group_size + off
                s = scale * (kk @ q4[b, h, 0])
                w = np.exp(s - s.max())
                out[b, h, 0] = (w / w.sum()) @ vv
    return out


# ---------------------------------------------------------------------------
# model + decode step (the caller of the hot path)
# ---------------------------------------------------------------------------

def random_model(layers, model_dim, ffn_dim, heads, kv_heads, vocab, max_seq,
                 activation="relu", seed=0, scale=0.02) -> dict:
    """model.py:178-210 -- identical RNG draw order, f32 weights."""
    rng = np.random.default_rng(seed)
    d, dk = model_dim, (model_dim // heads) * kv_heads

    def g(*shape):
        return rng.normal(0.0, scale, shape).astype(F32)

    def z(n):
        return np.zeros(n, F32)

    blocks = []
    for _ in range(layers):
        lw = {"ln1_g": np.ones(d, F32), "ln1_b": z(d)}
        lw["w_q"] = g(d, d); lw["b_q"] = z(d)
        lw["w_k"] = g(d, dk); lw["b_k"] = z(dk)
        lw["w_v"] = g(d, dk); lw["b_v"] = z(dk)
        lw["w_o"] = g(d, d); lw["b_o"] = z(d)
        lw["ln2_g"] = np.ones(d, F32); lw["ln2_b"] = z(d)
        lw["mlp_w1"] = g(d, ffn_dim); lw["mlp_b1"] = g(ffn_dim)
        lw["mlp_w2"] = g(d, ffn_dim); lw["mlp_b2"] = z(d)
        lw["mlp_w3"] = g(d, ffn_dim) if activation == "swiglu" else None
        blocks.append(lw)
    embed = g(vocab, d)
    pos = g(max_seq, d)
    unembed = g(d, vocab)
    return {"config": dict(layers=layers, model_dim=d, ffn_dim=ffn_dim, heads=heads,
                           kv_heads=kv_heads, vocab=vocab, max_seq=max_seq,
                           activation=activation),
            "layers": blocks, "embed": embed, "pos_embed": pos, "unembed": unembed,
            "lnf_g": np.ones(d, F32), "lnf_b": z(d)}


def decode_step(model: dict, caches, tokens, *, mode="dense", head_density=1.0,
                layer0_dense=True, k_table=None, head_routers=None,
                mlp_routers=None, block_size=64, record=None, forced=None) -> np.ndarray:
    """engine.py:314-392 -- one batched decode step, returns (B, vocab) f32.

    ``k_table`` maps layer -> neuron budget (calibration.py:64-68); routers
    are dicts from ``init_*_router``.  ``record`` (optional dict) receives
    the per-layer selections so tests can compare them bit-exactly.
    ``forced`` (optional dict with per-layer "heads" / "union" lists, keyed
    by layer) replaces the router selections -- used to check a device step
    against this oracle given the device's own (bit-exactly checked) picks.
    """
    cfg = model["config"]
    d, H, H_kv = cfg["model_dim"], cfg["heads"], cfg["kv_heads"]
    d_h = d // H
    tokens = np.asarray(tokens, np.int64)
    batch = tokens.size
    pos = caches[0].lengths.copy()
    if (pos >= cfg["max_seq"]).any():
        raise Capacity("position table exhausted (max_seq reached)")
    scale = 1.0 / math.sqrt(d_h)
    sparse_mlp = mode != "dense" and cfg["activation"] == "relu" and k_table is not None
    x = model["embed"][tokens] + model["pos_embed"][pos]
    for ell, lw in enumerate(model["layers"]):
        cache = caches[ell]
        h1 = layernorm(x, lw["ln1_g"], lw["ln1_b"])
        q4 = (matmul(h1, lw["w_q"]) + lw["b_q"]).reshape(batch, H, d_h)[:, :, None, :]
        kk = (matmul(h1, lw["w_k"]) + lw["b_k"]).reshape(batch, H_kv, d_h)
        vv = (matmul(h1, lw["w_v"]) + lw["b_v"]).reshape(batch, H_kv, d_h)
        cache.append_step(kk, vv)
        sparse_heads = (mode == "polar" and not (ell == 0 and layer0_dense)
                        and head_density < 1.0)
        if sparse_heads:
            if forced is not None and ell in forced.get("heads", {}):
                sel = np.asarray(forced["heads"][ell], np.int64)
            else:
                r = head_routers[ell]
                logits = head_router_forward(r["w"], r["b"], h1)
                sel = topk_indices_rows(logits, head_budget(head_density, H_kv))
        else:
            sel = np.tile(np.arange(H_kv, dtype=np.int64), (batch, 1))
        if record is not None:
            record.setdefault("heads", []).append(sel)
        attn = gqa_selective_attention_decode(q4, cache, sel, block_size, scale)
        x = x + (matmul(attn[:, :, 0, :].reshape(batch, d), lw["w_o"]) + lw["b_o"])
        h2 = layernorm(x, lw["ln2_g"], lw["ln2_b"])
        if sparse_mlp:
            k_ell = min(int(k_table[ell]), cfg["ffn_dim"])
            r = mlp_routers[ell]
            logits = mlp_router_forward(r["w_in"], r["b_in"], r["w_out"], r["b_out"], h2)
            rows = topk_indices_rows(logits, k_ell)
            union = union_neuron_indices(list(rows))
            if forced is not None and ell in forced.get("union", {}):
                union = np.asarray(forced["union"][ell], np.int64)
            if record is not None:
                record.setdefault("union", []).append(union)
            mlp = sparse_mlp_forward(h2[:, None, :], lw["mlp_w1"], lw["mlp_b1"],
                                     lw["mlp_w2"], lw["mlp_b2"], union)[:, 0, :]
        elif cfg["activation"] == "swiglu":
            mlp = swiglu_mlp_forward(h2[:, None, :], lw["mlp_w1"], lw["mlp_w3"],
                                     lw["mlp_w2"], lw["mlp_b2"])[:, 0, :]
        else:
            mlp = dense_mlp_forward(h2[:, None, :], lw["mlp_w1"], lw["mlp_b1"],
                                    lw["mlp_w2"], lw["mlp_b2"])[:, 0, :]
        x = x + mlp
    xf = layernorm(x, model["lnf_g"], model["lnf_b"])
    return matmul(xf, model["unembed"])
