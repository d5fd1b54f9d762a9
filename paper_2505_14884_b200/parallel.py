"""Tensor parallelism for the 66B / 70B shapes.

One process per GPU (torchrun), NCCL over NVLink 5 / NVSwitch.

* Attention: contiguous KV-group shards.  Rank r owns groups
  [r*H_kv/T, (r+1)*H_kv/T) and their G query heads each: the q/k/v rows of
  the packed QKV weight, the matching input columns of W_o, and its slice of
  every KV cache.
* MLP: contiguous neuron shards [r*D/T, (r+1)*D/T) of W1^T / W2^T (neuron
  rows) and b1.
* Routers are REPLICATED (head router d x H_kv, MLP router d x h_r + h_r x D),
  so every rank computes bit-identical logits and the identical global
  top-k / union without any communication; each rank then attends over
  ``sel ∩ own groups`` (ps_sha_decode's group_base) and runs the selective
  MLP over ``S ∩ own neurons`` (ps_select_union's [lo, hi) compaction).
* Collectives: the O-projection and the down-projection produce partial sums
  of the residual update; one all-reduce (sum) after each, exactly where the
  row-parallel GEMMs need it.  b_o / b2 are added by rank 0 only.

``TPPlan`` is pure host logic (tested on CPU with gloo, world_size 2);
``TensorParallel`` holds the device hooks the decode engine calls.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .kernels import PackedMLP, ROW_PAD, _round_up, gather_gemm_into, mlp_into
from .model import DeviceLayer, DeviceModel, TransformerConfig


@dataclass(frozen=True)
class TPPlan:
    world: int
    rank: int
    heads: int
    kv_heads: int
    head_dim: int
    model_dim: int
    ffn_dim: int

    @classmethod
    def make(cls, cfg: TransformerConfig, world: int, rank: int) -> "TPPlan":
        if world < 1 or not 0 <= rank < world:
            raise ValueError(f"bad TP rank {rank} of {world}")
        if cfg.kv_heads % world:
            raise ValueError(f"kv_heads {cfg.kv_heads} not divisible by TP degree {world}")
        if cfg.ffn_dim % (32 * world):
            raise ValueError(f"ffn_dim {cfg.ffn_dim} must split into 32-aligned shards over {world} ranks")
        return cls(world, rank, cfg.heads, cfg.kv_heads, cfg.head_dim, cfg.model_dim, cfg.ffn_dim)

    # ---- attention shard
    @property
    def group_size(self) -> int:
        return self.heads // self.kv_heads

    @property
    def kv_heads_local(self) -> int:
        return self.kv_heads // self.world

    @property
    def heads_local(self) -> int:
        return self.kv_heads_local * self.group_size

    @property
    def group_base(self) -> int:
        return self.rank * self.kv_heads_local

    @property
    def q_cols(self) -> tuple:
        """Columns of q / attn (and input rows of W_o) owned by this rank."""
        lo = self.group_base * self.group_size * self.head_dim
        return lo, lo + self.heads_local * self.head_dim

    @property
    def kv_cols(self) -> tuple:
        lo = self.group_base * self.head_dim
        return lo, lo + self.kv_heads_local * self.head_dim

    def qkv_rows(self) -> list:
        """Row ranges of the packed [W_q; W_k; W_v]^T owned by this rank."""
        d, dk = self.model_dim, self.kv_heads * self.head_dim
        (q0, q1), (k0, k1) = self.q_cols, self.kv_cols
        return [(q0, q1), (d + k0, d + k1), (d + dk + k0, d + dk + k1)]

    def groups_of(self, sel_row) -> list:
        """Selected global group ids that this rank computes."""
        lo, hi = self.group_base, self.group_base + self.kv_heads_local
        return [int(g) for g in sel_row if lo <= int(g) < hi]

    # ---- MLP shard
    @property
    def ffn_local(self) -> int:
        return self.ffn_dim // self.world

    @property
    def ffn_range(self) -> tuple:
        return self.rank * self.ffn_local, (self.rank + 1) * self.ffn_local

    def union_local(self, union_ids):
        """Global union ids -> this rank's shard, rebased (what the device's
        [lo, hi) compaction produces)."""
        lo, hi = self.ffn_range
        return [int(i) - lo for i in union_ids if lo <= int(i) < hi]


def shard_model(model: DeviceModel, plan: TPPlan) -> DeviceModel:
    """This rank's weights (copies) of a full device model."""
    q0, q1 = plan.q_cols
    f0, f1 = plan.ffn_range
    layers = []
    cache = {}
    for lw in model.layers:
        key = id(lw)
        if key in cache:
            layers.append(cache[key])
            continue
        L = DeviceLayer()
        L.ln1_g, L.ln1_b, L.ln2_g, L.ln2_b = lw.ln1_g, lw.ln1_b, lw.ln2_g, lw.ln2_b
        rows = plan.qkv_rows()
        L.w_qkv_t = torch.cat([lw.w_qkv_t[a:b] for a, b in rows], 0).contiguous()
        L.b_qkv = torch.cat([lw.b_qkv[a:b] for a, b in rows], 0).contiguous()
        L.w_o_t = lw.w_o_t[:, q0:q1].contiguous()
        L.b_o = lw.b_o if plan.rank == 0 else torch.zeros_like(lw.b_o)
        mk = lw.mlp
        L.mlp = PackedMLP(mk.w1t[f0:f1].contiguous(), None if mk.b1 is None else mk.b1[f0:f1].contiguous(),
                          mk.w2t[f0:f1].contiguous(),
                          mk.b2 if plan.rank == 0 or mk.b2 is None else torch.zeros_like(mk.b2),
                          None if mk.w3t is None else mk.w3t[f0:f1].contiguous())
        cache[key] = L
        layers.append(L)
    return DeviceModel(model.config, layers, model.embed, model.pos_embed, model.lnf_g, model.lnf_b, model.unembed_t)


def random_shard(cfg: TransformerConfig, plan: TPPlan, seed: int = 0, scale: float = 0.02, device="cuda",
                 distinct_layers: int | None = None) -> DeviceModel:
    """Draw only this rank's shard on the device (benchmark-scale models)."""
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed * 131 + plan.rank)
    d, dk = cfg.model_dim, plan.kv_heads_local * cfg.head_dim
    dq = plan.heads_local * cfg.head_dim
    Dl = plan.ffn_local

    def g(*shape):
        return (torch.randn(*shape, device=dev, generator=gen) * scale).to(torch.bfloat16)

    n_distinct = cfg.layers if distinct_layers is None else max(1, min(distinct_layers, cfg.layers))
    uniq = []
    for _ in range(n_distinct):
        L = DeviceLayer()
        L.ln1_g = L.ln2_g = torch.ones(d, device=dev)
        L.ln1_b = L.ln2_b = torch.zeros(d, device=dev)
        L.w_qkv_t = g(dq + 2 * dk, d)
        L.b_qkv = torch.zeros(dq + 2 * dk, device=dev)
        L.w_o_t = g(d, dq)
        L.b_o = torch.zeros(d, device=dev)
        L.mlp = PackedMLP(g(Dl, d), torch.randn(Dl, device=dev, generator=gen) * scale, g(Dl, d),
                          torch.zeros(d, device=dev), g(Dl, d) if cfg.activation == "swiglu" else None)
        uniq.append(L)
    layers = [uniq[i % n_distinct] for i in range(cfg.layers)]
    return DeviceModel(cfg, layers, g(cfg.vocab, d), g(cfg.max_seq, d), torch.ones(d, device=dev),
                       torch.zeros(d, device=dev), g(cfg.vocab, d))


class TensorParallel:
    """Device hooks used by DecodeEngine(tp=...)."""

    def __init__(self, plan: TPPlan, group=None, collective: str = "nccl"):
        """``collective``: "nccl" (torch.distributed all-reduce, then x += sum)
        or "p2p" (collective.P2PAllReduce: one peer-memory kernel that waits
        for every rank's bf16 partial and adds the sum into x; its IPC handles
        travel over ``group``, which may be gloo)."""
        if collective not in ("nccl", "p2p"):
            raise ValueError(f"collective must be 'nccl' or 'p2p', got {collective!r}")
        self.plan = plan
        self.group = group
        self.collective = collective
        self._p2p = None
        self.heads_local = plan.heads_local
        self.kv_heads_local = plan.kv_heads_local
        self.group_base = plan.group_base
        self.ffn_local = plan.ffn_local
        self.ffn_range = plan.ffn_range
        self._tmp = {}

    def all_reduce(self, t: torch.Tensor) -> None:
        if self.plan.world > 1:
            import torch.distributed as dist

            if t.dtype == torch.bfloat16 and dist.get_backend(self.group) == "gloo":
                f = t.float()  # CPU-test transport (gloo): no bf16 reduction
                dist.all_reduce(f, op=dist.ReduceOp.SUM, group=self.group)
                t.copy_(f)
                return
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def _p2p_engine(self, eng):
        if self._p2p is None:
            from .collective import P2PAllReduce

            self._p2p = P2PAllReduce(self.group, self.plan.rank, self.plan.world, eng.x.numel(), eng.x.device)
        return self._p2p

    def reduce_into(self, eng, part) -> None:
        """eng.x += sum over ranks of ``part`` (this rank's bf16 partial)."""
        if self.collective == "p2p":
            self._p2p_engine(eng).add_into(eng.x)
            return
        self.all_reduce(part)
        eng.x.add_(part)

    def _partial(self, eng, name):
        """bf16 (B, d) buffer for a rank's partial residual update: the
        all-reduce moves half the bytes of f32 partials (SURVEY.md §8(e)
        budgets bf16); the sum is added into the f32 residual stream.  With
        the p2p collective it is the peer-mapped buffer of the next call."""
        if self.collective == "p2p":
            return self._p2p_engine(eng).next_buffer(eng.x.shape)
        t = self._tmp.get(name)
        if t is None:
            t = torch.zeros(eng.x.shape, dtype=torch.bfloat16, device=eng.x.device)
            self._tmp[name] = t
        return t

    def o_proj(self, eng, lw) -> int:
        """x += all_reduce(attn_local @ W_o[local rows] (+ b_o on rank 0))."""
        part = self._partial(eng, "o")
        n = eng._linear_bf16(eng.attn, lw.w_o_t, lw.b_o, part, tag="gg_o")
        self.reduce_into(eng, part)
        return n

    def mlp(self, eng, lw, idx, cnt, ell: int = 0) -> int:
        """x += all_reduce(MLP over this rank's neurons (+ b2 on rank 0))."""
        part = self._partial(eng, "mlp")
        mk = lw.mlp
        n = 0
        if idx is not None:
            mlp_into(mk, eng.h, idx, cnt, eng.hidden, part, residual=None, expected=eng.union_est[ell])
            n += 2
        elif eng.cfg.activation == "swiglu":
            torch.mm(eng.h, mk.gate_up().t(), out=eng.gu)
            _lib.call("ps_swiglu", _lib.ptr(eng.gu), eng.gu.stride(0), eng.B, mk.D, _lib.ptr(eng.hidden),
                      eng.hidden.stride(0), _lib.stream_ptr())
            n += 1
            if mk.b2 is not None:
                torch.addmm(eng._bf(mk.b2), eng.hidden[:, :mk.D], mk.w2t, out=part)
            else:
                torch.mm(eng.hidden[:, :mk.D], mk.w2t, out=part)
        else:
            hid = eng._scratch("hid_tp", (eng.B, mk.D), torch.bfloat16)
            n += eng._linear_bf16(eng.h, mk.w1t, mk.b1, hid, act_relu=True)
            if mk.b2 is not None:
                torch.addmm(eng._bf(mk.b2), hid, mk.w2t, out=part)
            else:
                torch.mm(hid, mk.w2t, out=part)
        self.reduce_into(eng, part)
        return n
