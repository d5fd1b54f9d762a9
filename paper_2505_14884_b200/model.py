"""Model shapes and device-resident weights for the decode step.

``TransformerConfig`` mirrors sparsedecode/model.py:23-67 (pre-norm decoder,
learned positions, LayerNorm, ReLU or SwiGLU MLP, GQA via kv_heads).
``DeviceModel`` holds one model in HBM laid out for the kernels:

* attention projections packed neuron-major: ``w_qkv_t`` (d + 2*kv_dim, d)
  so Q, K and V come out of ONE GEMM launch (cuBLAS by default, the
  tcgen05 gathered-GEMM kernel with identity ids under
  ``dense_backend="native"``); ``w_o_t`` (d, d);
* MLP blocks as :class:`~paper_2505_14884_b200.kernels.PackedMLP`
  (W1^T / W2^T rows = one neuron each, the gather unit);
* embeddings bf16, LayerNorm parameters and biases f32.

Weights come either from a reference-layout host model (numpy arrays in the
reference's (d_in, d_out) convention -- the oracle's ``random_model`` or a
``sparsedecode.Model``; model.py:178-210 draw order) or are drawn directly
on the device (N(0, 0.02), LayerNorm 1/0, zero biases except b1) for the
production shapes, where host-side init would dominate start-up.
"""

from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np
import torch

from .kernels import PackedMLP
from .validation import check_choice, check_count

_ACTIVATIONS = ("relu", "swiglu")


@dataclass(frozen=True)
class TransformerConfig:
    layers: int
    model_dim: int
    ffn_dim: int
    heads: int
    kv_heads: int
    vocab: int
    max_seq: int
    activation: str = "relu"

    def __post_init__(self):
        for name in ("layers", "model_dim", "ffn_dim", "heads", "kv_heads", "vocab", "max_seq"):
            check_count(getattr(self, name), name)
        check_choice(self.activation, _ACTIVATIONS, "activation")
        if self.model_dim % self.heads:
            raise ValueError(f"model_dim {self.model_dim} not divisible by heads {self.heads}")
        if self.heads % self.kv_heads:
            raise ValueError(f"heads {self.heads} not divisible by kv_heads {self.kv_heads}")

    @property
    def head_dim(self) -> int:
        return self.model_dim // self.heads

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.head_dim

    @property
    def group_size(self) -> int:
        return self.heads // self.kv_heads

    def to_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}


# BASELINE.json configs (shapes only; OPT-style blocks as in the reference)
SHAPES = {
    "tiny": TransformerConfig(2, 256, 1024, 8, 8, 512, 288, "relu"),
    "opt-6.7b": TransformerConfig(32, 4096, 16384, 32, 32, 50272, 2048, "relu"),
    "llama-3.1-8b": TransformerConfig(32, 4096, 14336, 32, 8, 128256, 8192, "swiglu"),
    "opt-66b": TransformerConfig(64, 9216, 36864, 72, 72, 50272, 2048, "relu"),
    "llama-3.1-70b": TransformerConfig(80, 8192, 28672, 64, 8, 128256, 8448, "swiglu"),
}


class DeviceLayer:
    __slots__ = ("ln1_g", "ln1_b", "w_qkv_t", "b_qkv", "w_o_t", "b_o", "ln2_g", "ln2_b", "mlp")


class DeviceModel:
    def __init__(self, config: TransformerConfig, layers, embed, pos_embed, lnf_g, lnf_b, unembed_t):
        self.config = config
        self.layers = layers
        self.embed = embed
        self.pos_embed = pos_embed
        self.lnf_g = lnf_g
        self.lnf_b = lnf_b
        self.unembed_t = unembed_t

    @property
    def device(self):
        return self.embed.device

    # ------------------------------------------------------------------ builders
    @classmethod
    def from_host(cls, config: TransformerConfig, host, device="cuda") -> "DeviceModel":
        """Upload a reference-layout model: a dict like the oracle's
        ``random_model`` output, or a ``sparsedecode.Model``."""
        dev = torch.device(device)

        def get(obj, name):
            return obj[name] if isinstance(obj, dict) else getattr(obj, name)

        def f32(a):
            return torch.as_tensor(np.asarray(a, np.float32)).to(dev)

        def bf(a):
            return torch.as_tensor(np.asarray(a, np.float32)).to(dev, torch.bfloat16)

        layers = []
        for lw in get(host, "layers"):
            L = DeviceLayer()
            L.ln1_g, L.ln1_b = f32(get(lw, "ln1_g")), f32(get(lw, "ln1_b"))
            wqkv = np.concatenate([get(lw, "w_q"), get(lw, "w_k"), get(lw, "w_v")], axis=1)
            L.w_qkv_t = bf(wqkv.T.copy()).contiguous()
            L.b_qkv = f32(np.concatenate([get(lw, "b_q"), get(lw, "b_k"), get(lw, "b_v")]))
            L.w_o_t = bf(np.asarray(get(lw, "w_o")).T.copy()).contiguous()
            L.b_o = f32(get(lw, "b_o"))
            L.ln2_g, L.ln2_b = f32(get(lw, "ln2_g")), f32(get(lw, "ln2_b"))
            w3 = get(lw, "mlp_w3")
            L.mlp = PackedMLP.from_reference(f32(get(lw, "mlp_w1")), f32(get(lw, "mlp_b1")),
                                             f32(get(lw, "mlp_w2")), f32(get(lw, "mlp_b2")),
                                             None if w3 is None else f32(w3), device=dev)
            layers.append(L)
        return cls(config, layers, bf(get(host, "embed")), bf(get(host, "pos_embed")),
                   f32(get(host, "lnf_g")), f32(get(host, "lnf_b")),
                   bf(np.asarray(get(host, "unembed")).T.copy()).contiguous())

    @classmethod
    def random(cls, config: TransformerConfig, seed: int = 0, scale: float = 0.02, device="cuda",
               distinct_layers: int | None = None) -> "DeviceModel":
        """On-device random init with the reference's distribution
        (model.py:178-210).  ``distinct_layers`` < layers aliases weight
        storage round-robin (every layer still reads its full weights from
        HBM; only capacity is saved) -- used for shapes that exceed one GPU."""
        dev = torch.device(device)
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        d, D, dk = config.model_dim, config.ffn_dim, config.kv_dim

        def g(*shape):
            return (torch.randn(*shape, device=dev, generator=gen) * scale).to(torch.bfloat16)

        def ones(n):
            return torch.ones(n, device=dev)

        def zeros(n):
            return torch.zeros(n, device=dev)

        n_distinct = config.layers if distinct_layers is None else max(1, min(distinct_layers, config.layers))
        uniq = []
        for _ in range(n_distinct):
            L = DeviceLayer()
            L.ln1_g, L.ln1_b = ones(d), zeros(d)
            L.w_qkv_t = g(d + 2 * dk, d)
            L.b_qkv = zeros(d + 2 * dk)
            L.w_o_t = g(d, d)
            L.b_o = zeros(d)
            L.ln2_g, L.ln2_b = ones(d), zeros(d)
            w1t = g(D, d)
            b1 = (torch.randn(D, device=dev, generator=gen) * scale)
            w2t = g(D, d)
            w3t = g(D, d) if config.activation == "swiglu" else None
            L.mlp = PackedMLP(w1t, b1, w2t, zeros(d), w3t)
            uniq.append(L)
        layers = [uniq[i % n_distinct] for i in range(config.layers)]
        return cls(config, layers, g(config.vocab, d), g(config.max_seq, d), ones(d), zeros(d),
                   g(config.vocab, d))

    def weight_bytes(self) -> int:
        seen, total = set(), 0
        for L in self.layers:
            for t in (L.w_qkv_t, L.w_o_t, L.mlp.w1t, L.mlp.w2t, L.mlp.w3t):
                if t is not None and t.data_ptr() not in seen:
                    seen.add(t.data_ptr())
                    total += t.numel() * t.element_size()
        return total + sum(t.numel() * t.element_size() for t in (self.embed, self.pos_embed, self.unembed_t))
