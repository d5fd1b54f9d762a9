"""Router forward passes on B200 -- drop-in for ``sparsedecode.routers``
forward API (routers.py:154-341).

Training (BCE + AdamW, supervision collection) stays in the reference: it is
offline CPU work.  A router trained there is moved here
with ``from_reference(router)``; a router built here with the same seed
draws the reference's exact initial weights (routers.py:280-284, 320-322).
Weights are stored bf16 on the device; logits are f32.

* :class:`HeadRouter` -- ``logits = x W + b`` fused with the per-row top-k
  (one launch, ``select``), routers.py:306-331.
* :class:`MlpRouter` -- ``relu(x W_in + b_in) W_out + b_out`` as two tcgen05
  GEMM launches, routers.py:256-303; ``select_topk`` / ``select_threshold``
  write the batch union straight into a device bitmap.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib, _ws
from .kernels import BatchHeadIndex, NeuronIndexTensor, ROW_PAD, _round_up, gather_gemm_into
from .validation import as_device_tensor, check_count, default_device


def _as_batch(x, d, device):
    t = as_device_tensor(x, "x", device=device)
    single = t.ndim == 1
    if single:
        t = t[None, :]
    if t.ndim != 2:
        raise ValueError(f"expected vector or batch of vectors, got {tuple(t.shape)}")
    if t.shape[1] != d:
        raise ValueError(f"expected {d} features, got {t.shape[1]}")
    return t.to(torch.bfloat16).contiguous(), single


class HeadRouter:
    """Single linear layer scoring heads / KV groups (routers.py:306-331)."""

    def __init__(self, d_model: int, n_heads: int, seed: int = 0, device=None, _weights=None):
        check_count(d_model, "d_model")
        check_count(n_heads, "n_heads")
        self.d_model, self.n_heads, self.seed = d_model, n_heads, seed
        if _weights is None:
            rng = np.random.default_rng(seed)
            w = rng.normal(0.0, 1.0 / math.sqrt(d_model), (d_model, n_heads))
            b = np.zeros(n_heads)
        else:
            w, b = _weights
        dev = device or default_device()
        self.w_t = torch.as_tensor(np.ascontiguousarray(np.asarray(w, np.float64).T), dtype=torch.float32).to(
            dev, torch.bfloat16).contiguous()
        self.b = torch.as_tensor(np.asarray(b, np.float64), dtype=torch.float32).to(dev)
        self._scratch = None

    @classmethod
    def from_reference(cls, router, device=None) -> "HeadRouter":
        return cls(router.w_.shape[0], router.w_.shape[1], getattr(router, "seed", 0), device,
                   _weights=(router.w_, router.b_))

    @classmethod
    def from_weights(cls, w, b, device=None) -> "HeadRouter":
        w = np.asarray(w)
        return cls(w.shape[0], w.shape[1], 0, device, _weights=(w, b))

    def select_into(self, x2d: torch.Tensor, k: int, sel_out: torch.Tensor, logits_out=None) -> None:
        B, d = x2d.shape
        _lib.call("ps_head_router_topk", _lib.ptr(x2d), x2d.stride(0), _lib.ptr(self.w_t), _lib.ptr(self.b),
                  B, d, self.n_heads, int(k), _lib.ptr(logits_out), _lib.ptr(sel_out), _lib.stream_ptr())

    def select_append_into(self, x2d: torch.Tensor, k: int, sel_out: torch.Tensor, cache, k_new, v_new,
                           src_ld: int, logits_out=None) -> None:
        """select_into fused with the step's KV append into ``cache``
        (tensors.py:150-170 semantics; one launch instead of two)."""
        B, d = x2d.shape
        if hasattr(cache, "block_table"):  # PagedKVCache
            _lib.call("ps_head_router_topk_append_paged", _lib.ptr(x2d), x2d.stride(0), _lib.ptr(self.w_t),
                      _lib.ptr(self.b), B, d, self.n_heads, int(k), _lib.ptr(logits_out), _lib.ptr(sel_out),
                      _lib.ptr(cache.k_pool), _lib.ptr(cache.v_pool), cache.page_rows, _lib.ptr(cache.block_table),
                      cache.max_pages, _lib.ptr(cache.lengths), _lib.ptr(k_new), _lib.ptr(v_new), int(src_ld),
                      cache.kv_heads, cache.head_dim, _lib.ptr(cache._err), _lib.stream_ptr())
            return
        _lib.call("ps_head_router_topk_append", _lib.ptr(x2d), x2d.stride(0), _lib.ptr(self.w_t), _lib.ptr(self.b),
                  B, d, self.n_heads, int(k), _lib.ptr(logits_out), _lib.ptr(sel_out), _lib.ptr(cache.keys),
                  _lib.ptr(cache.values), _lib.ptr(cache.lengths), _lib.ptr(k_new), _lib.ptr(v_new), int(src_ld),
                  cache.kv_heads, cache.capacity, cache.head_dim, _lib.ptr(cache._err), _lib.stream_ptr())

    def decision_function(self, x) -> torch.Tensor:
        """routers.py:178-186: per-head logits (f32), vector or batch."""
        xb, single = _as_batch(x, self.d_model, self.w_t.device)
        B = xb.shape[0]
        logits = torch.empty((B, self.n_heads), dtype=torch.float32, device=xb.device)
        sel = torch.empty((B, 1), dtype=torch.int32, device=xb.device)
        self.select_into(xb, 1, sel, logits)
        return logits[0] if single else logits

    def predict(self, x) -> torch.Tensor:
        return self.decision_function(x) > 0.0

    def select(self, x, k: int) -> BatchHeadIndex:
        """Fused router + top-k -> BatchHeadIndex (engine.py:352-357)."""
        xb, _ = _as_batch(x, self.d_model, self.w_t.device)
        if not 1 <= k <= self.n_heads:
            raise ValueError(f"k must be in [1, {self.n_heads}], got {k}")
        sel = torch.empty((xb.shape[0], k), dtype=torch.int32, device=xb.device)
        self.select_into(xb, k, sel)
        return BatchHeadIndex(sel, validate=False, n_max=self.n_heads)


class MlpRouter:
    """Two-layer ReLU neuron-activity predictor (routers.py:256-303)."""

    def __init__(self, d_model: int, ffn_dim: int, hidden_dim: int | None = None, seed: int = 0,
                 device=None, _weights=None):
        check_count(d_model, "d_model")
        check_count(ffn_dim, "ffn_dim")
        h = hidden_dim if hidden_dim is not None else min(1024, 4 * d_model)
        check_count(h, "hidden_dim")
        self.d_model, self.ffn_dim, self.hidden_dim_, self.seed = d_model, ffn_dim, h, seed
        if _weights is None:
            rng = np.random.default_rng(seed)
            w_in = rng.normal(0.0, math.sqrt(2.0 / d_model), (d_model, h))
            w_out = rng.normal(0.0, math.sqrt(2.0 / h), (h, ffn_dim))
            b_in, b_out = np.zeros(h), np.zeros(ffn_dim)
        else:
            w_in, b_in, w_out, b_out = _weights
        dev = device or default_device()
        f32 = lambda a: torch.as_tensor(np.asarray(a, np.float64), dtype=torch.float32)  # noqa: E731
        self.w_in_t = f32(np.asarray(w_in).T).to(dev, torch.bfloat16).contiguous()    # (h, d)
        self.b_in = f32(b_in).to(dev)
        self.w_out_t = f32(np.asarray(w_out).T).to(dev, torch.bfloat16).contiguous()  # (D, h)
        self.b_out = f32(b_out).to(dev)

    @classmethod
    def random_device(cls, d_model: int, ffn_dim: int, hidden_dim: int | None = None, seed: int = 0,
                      device=None, hot=None, hot_bias: float = 20.0, center: bool = False) -> "MlpRouter":
        """Router drawn on the device with the reference's distribution
        (N(0, sqrt(2/d)), N(0, sqrt(2/h)), zero biases) -- for production
        shapes where host-side init is slow.  ``hot`` (neuron ids) adds
        ``hot_bias`` to their output bias: the controlled "hot neuron" union
        density of SURVEY.md §7 / analysis.py:124-140 (every token's top-k
        then covers the hot set, so |S|/D is set by the caller)."""
        obj = cls.__new__(cls)
        h = hidden_dim if hidden_dim is not None else min(1024, 4 * d_model)
        obj.d_model, obj.ffn_dim, obj.hidden_dim_, obj.seed = d_model, ffn_dim, h, seed
        dev = torch.device(device or default_device())
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        obj.w_in_t = (torch.randn(h, d_model, device=dev, generator=gen) * math.sqrt(2.0 / d_model)).to(
            torch.bfloat16)
        obj.w_out_t = (torch.randn(ffn_dim, h, device=dev, generator=gen) * math.sqrt(2.0 / h)).to(torch.bfloat16)
        obj.b_in = torch.zeros(h, device=dev)
        obj.b_out = torch.zeros(ffn_dim, device=dev)
        if center:
            # remove the token-independent part of the logits: for unit-variance
            # inputs the hidden pre-activations are N(0, 2), so E[relu] = 1/sqrt(pi)
            # and every logit carries the constant offset E[relu] * sum_i W_out[i, j];
            # subtracting it leaves per-token (not per-neuron) variation, so the
            # non-hot picks differ from token to token
            obj.b_out -= obj.w_out_t.float().sum(dim=1) / math.sqrt(math.pi)
        if hot is not None:
            obj.b_out[torch.as_tensor(np.asarray(hot), device=dev, dtype=torch.long)] += hot_bias
        return obj

    @classmethod
    def from_reference(cls, router, device=None) -> "MlpRouter":
        return cls(router.w_in_.shape[0], router.w_out_.shape[1], router.w_in_.shape[1],
                   getattr(router, "seed", 0), device,
                   _weights=(router.w_in_, router.b_in_, router.w_out_, router.b_out_))

    @classmethod
    def from_weights(cls, w_in, b_in, w_out, b_out, device=None) -> "MlpRouter":
        w_in = np.asarray(w_in)
        return cls(w_in.shape[0], np.asarray(w_out).shape[1], w_in.shape[1], 0, device,
                   _weights=(w_in, b_in, w_out, b_out))

    def fused_bytes(self, batch: int) -> int:
        """Workspace bytes of the one-launch router (0: shape unsupported)."""
        return int(_lib.load().ps_router_mlp_fused_workspace_bytes(batch, self.d_model, self.hidden_dim_,
                                                                   self.ffn_dim))

    def fused_into(self, x2d: torch.Tensor, hid: torch.Tensor, logits: torch.Tensor, with_bias: bool = True,
                   tag: str = "router_fused") -> bool:
        """Both router layers in ONE persistent launch with a device grid
        barrier between them (ps_router_mlp_fused; static weights prefetched
        ahead of the dependency wait).  Returns False (nothing launched) for
        shapes the kernel does not cover."""
        B, d = x2d.shape
        nb = self.fused_bytes(B)
        if not nb:
            return False
        lib = _lib.load()
        ws = _ws.get(tag, nb, x2d.device)
        st = lib.ps_router_mlp_fused(_lib.ptr(self.w_in_t), _lib.ptr(self.b_in), _lib.ptr(self.w_out_t),
                                     _lib.ptr(self.b_out) if with_bias else None, d, self.hidden_dim_, self.ffn_dim,
                                     _lib.ptr(x2d), x2d.stride(0), B, _lib.ptr(hid), hid.stride(0),
                                     _lib.ptr(logits), logits.stride(0), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        if st == 5:  # PS_ERR_UNSUPPORTED
            return False
        _lib.check(st, "ps_router_mlp_fused")
        return True

    def logits_into(self, x2d: torch.Tensor, hid: torch.Tensor, logits: torch.Tensor, with_bias: bool = True,
                    fused: bool = False) -> None:
        """hid = relu(x W_in + b_in) (bf16), logits = hid W_out (+ b_out) (f32).
        ``fused``: both layers in ONE chained launch (ps_router_mlp; B <= 256;
        measured slower than the two launches, kept as an option);
        else two tcgen05 launches (ps_gather_gemm).  ``with_bias=False`` leaves
        b_out to the consumer (ps_select_union adds it while ranking)."""
        B, d = x2d.shape
        h = self.hidden_dim_
        if fused and B <= 256:
            lib = _lib.load()
            ws = _ws.get("router_chain", lib.ps_router_mlp_workspace_bytes(B, h, self.ffn_dim), x2d.device)
            _lib.call("ps_router_mlp", _lib.ptr(self.w_in_t), _lib.ptr(self.b_in), _lib.ptr(self.w_out_t),
                      _lib.ptr(self.b_out) if with_bias else None, d, h, self.ffn_dim, _lib.ptr(x2d),
                      x2d.stride(0), B, _lib.ptr(hid), hid.stride(0), _lib.ptr(logits), logits.stride(0),
                      _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
            return
        gather_gemm_into(self.w_in_t, None, None, x2d, x2d.stride(0), self.b_in, B, h, d, _lib.PS_ACT_RELU,
                         hid, hid.stride(0), tag="gg_router")
        gather_gemm_into(self.w_out_t, None, None, hid, hid.stride(0), self.b_out if with_bias else None, B,
                         self.ffn_dim, h, _lib.PS_ACT_NONE, logits, logits.stride(0), tag="gg_router")

    def decision_function(self, x) -> torch.Tensor:
        xb, single = _as_batch(x, self.d_model, self.w_in_t.device)
        B = xb.shape[0]
        if self.hidden_dim_ % 8:
            raise ValueError("router hidden width must be a multiple of 8 on the GPU path")
        hid = torch.empty((B, self.hidden_dim_), dtype=torch.bfloat16, device=xb.device)
        logits = torch.empty((B, self.ffn_dim), dtype=torch.float32, device=xb.device)
        self.logits_into(xb, hid, logits)
        return logits[0] if single else logits

    def predict(self, x) -> torch.Tensor:
        """routers.py:188-190: sigmoid(logit) > 0.5, i.e. logit > 0."""
        return self.decision_function(x) > 0.0

    def select_topk(self, x, k: int, layer: int = 0) -> NeuronIndexTensor:
        """Per-row top-k of the logits, unioned over the batch (engine.py:371-376)."""
        logits = self.decision_function(x)
        if logits.ndim == 1:
            logits = logits[None, :]
        return union_from_logits(logits, k=k, layer=layer)

    def select_threshold(self, x, threshold: float = 0.0, layer: int = 0) -> NeuronIndexTensor:
        logits = self.decision_function(x)
        if logits.ndim == 1:
            logits = logits[None, :]
        return union_from_logits(logits, threshold=threshold, layer=layer)


def union_from_logits(logits: torch.Tensor, k: int | None = None, threshold: float | None = None,
                      layer: int = 0) -> NeuronIndexTensor:
    """Top-k (or threshold) selection per row, ORed into a bitmap and
    compacted into the ascending batch union -- all on the device."""
    rows, width = logits.shape
    logits = logits.contiguous().float()
    dev = logits.device
    if k is not None and not 1 <= k <= width:
        raise ValueError(f"k must be in [1, {width}], got {k}")
    nbytes = int(_lib.load().ps_select_union_workspace_bytes(rows, width))
    ws = _ws.get(f"select_union_{rows}_{width}", nbytes, dev)
    buf = torch.empty(_round_up(width, ROW_PAD), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("ps_select_union", _lib.ptr(logits), None, rows, width, width, int(k) if k is not None else 0,
              float(threshold or 0.0), _lib.ptr(ws), nbytes, 0, width, ROW_PAD, _lib.ptr(buf),
              _lib.ptr(cnt), _lib.stream_ptr())
    return NeuronIndexTensor(layer, buf, cnt)


def mlp_router_forward(router: MlpRouter, x) -> torch.Tensor:
    """routers.py:334-336."""
    return router.decision_function(x)


def head_router_forward(router: HeadRouter, x) -> torch.Tensor:
    """routers.py:339-341."""
    return router.decision_function(x)
