"""Batched decode step on B200 -- the caller of the hot path.

Restates ``sparsedecode.engine.decode_step`` (engine.py:314-392) with the
same policy semantics (``SparsityPolicy``: modes dense / dejavu_mlp / polar,
head budget ceil(rho*H_kv - 1e-9), layer 0 dense by default, sparse MLP only
for ReLU models with a k table) and the same per-layer order:

    LN1 -> QKV -> KV append -> [head router -> top-k] -> SHA -> O-proj(+res)
        -> LN2 -> [MLP router -> per-row top-k -> union] -> selective MLP(+res)

Every launch is a libpolar_b200 kernel on static buffers, so the whole step
is captured once into a CUDA graph and replayed (the paper measured with
CUDA graphs).  The host only keeps the length mirror used for
capacity checks.  Tensor parallelism (heads + neurons sharded, routers
replicated, all-reduce after the O- and down-projections) lives in
``parallel.py`` and reuses :meth:`DecodeEngine.step_launches`.
"""

from __future__ import annotations

import copy
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, _ws
from .exceptions import CapacityError, ConfigurationError
from .kernels import (ROW_PAD, _round_up, gather_gemm_into, mlp_into, mlp_into_bitmap, sha_decode_into,
                      sparse_mlp_into, swiglu_into)
from .model import DeviceModel, TransformerConfig
from .tensors import KVCache, PagedKVCache
from .validation import check_choice, check_count

_MODES = ("dense", "dejavu_mlp", "polar")


@dataclass(frozen=True)
class SparsityPolicy:
    """engine.py:42-77 (router ranking only; the oracle-norm ranking is a
    study tool that computes every head and gives no speedup)."""

    mode: str = "dense"
    mlp_k_table: object = None
    head_density: float = 1.0
    layer0_dense_attention: bool = True

    def __post_init__(self):
        check_choice(self.mode, _MODES, "mode")
        if not 0.0 < float(self.head_density) <= 1.0:
            raise ValueError(f"head_density must be in (0, 1], got {self.head_density}")

    def head_budget(self, n_route: int) -> int:
        return max(1, math.ceil(self.head_density * n_route - 1e-9))

    def wants_sparse_mlp(self, config: TransformerConfig) -> bool:
        if self.mode == "dense" or config.activation != "relu":
            return False
        return self.mlp_k_table is not None

    def wants_sparse_heads(self, layer: int) -> bool:
        if self.mode != "polar":
            return False
        if layer == 0 and self.layer0_dense_attention:
            return False
        return self.head_density < 1.0

    def k_for(self, layer: int) -> int:
        t = self.mlp_k_table
        if hasattr(t, "k_for"):
            return int(t.k_for(layer))  # calibration.LayerKTable (calibration.py:64-68)
        try:
            return int(t[layer])
        except (KeyError, IndexError, TypeError) as exc:
            raise ConfigurationError(f"no calibrated k for layer {layer}") from exc


class DecodeEngine:
    """Decode session + step for one GPU (or one tensor-parallel rank).

    ``kv_ring``: number of distinct per-layer K/V storage buffers.  Default =
    layers.  A smaller ring aliases K/V STORAGE round-robin for shapes whose
    full cache exceeds HBM; every layer keeps its own lengths and reads its
    full (selected) history, so bytes moved and kernel work are unchanged --
    only capacity is saved (SURVEY.md §7 hard parts; reported in bench.py).
    """

    def __init__(self, model: DeviceModel, batch: int, capacity: int, policy: SparsityPolicy,
                 head_routers=None, mlp_routers=None, kv_ring: int | None = None, tp=None,
                 caches=None, dense_backend: str = "cublas", router_backend: str | None = None,
                 concurrent_router: bool | None = None, kv_page_rows: int = 0, kv_reserve: str = "full",
                 mlp_backend: str = "split", o_backend: str | None = None, union_handoff: bool | None = None):
        cfg = model.config
        check_count(batch, "batch")
        check_count(capacity, "capacity")
        self.model, self.cfg, self.B, self.policy = model, cfg, batch, policy
        self.dense_backend = check_choice(dense_backend, ("cublas", "native"), "dense_backend")
        # the MLP router's two layers: tcgen05 kernels with their static weights
        # streamed ahead of the previous launch (PDL), or cuBLAS
        # "fused": both layers in one persistent launch (ps_router_mlp_fused),
        # falling back to cuBLAS for shapes it does not cover.  Default: fused
        # for B <= 16 (OPT-6.7B per step: B=1 3.564 -> 3.507 ms, B=8 4.309 ->
        # 4.292, B=16 5.122 -> 5.112), cuBLAS above (B=64: 1.5 % faster than fused)
        if router_backend is None and dense_backend == "cublas" and batch <= 16:
            router_backend = "fused"
        self.router_backend = check_choice(router_backend or dense_backend,
                                           ("fused", "cublas", "native", "native_in"), "router_backend")
        # head router on a side stream, concurrent with the QKV GEMM (a
        # parallel branch of the captured graph) + a separate KV append; False
        # = fused with the append after the QKV GEMM.  Default: concurrent for
        # B <= 8 without TP (OPT-6.7B per step, same box: B=1 3.478 -> 3.341 ms,
        # B=2 3.548 -> 3.438, B=4 3.819 -> 3.714, B=8 4.302 -> 4.190; B=16
        # 5.052 -> 5.138 and B=64 slower: the cluster competes with the GEMM)
        if concurrent_router is None:
            concurrent_router = batch <= 8 and tp is None
        self.concurrent_router = bool(concurrent_router)
        # selective MLP: "split" = UP and DOWN as two tcgen05 launches
        # (ps_gather_gemm / _t); "chain" = both in one persistent launch
        # (ps_sparse_mlp, batch <= 256)
        self.mlp_backend = check_choice(mlp_backend, ("split", "chain"), "mlp_backend")
        # attention output projection (+ residual): cuBLAS, or the tcgen05
        # dense kernel, whose static W_o streams ahead of the SHA tail (PDL) and
        # which hands LayerNorm a PDL edge.  Default: native for B <= 8 without
        # TP (OPT-6.7B per step, same box: B=1 3.347 -> 3.301 ms, B=4 3.745 ->
        # 3.67-3.72, B=8 4.192 -> 4.167; B=16 5.059 -> 5.14, B=64 +0.8 %)
        if o_backend is None:
            o_backend = "native" if batch <= 8 and tp is None else dense_backend
        self.o_backend = check_choice(o_backend, ("cublas", "native"), "o_backend")
        self.side = torch.cuda.Stream(device=model.device) if self.concurrent_router else None
        self._cache = {}
        self.head_routers, self.mlp_routers = head_routers, mlp_routers
        self.tp = tp
        dev = model.device
        self.device = dev
        d, dk, H, H_kv, d_h = cfg.model_dim, cfg.kv_dim, cfg.heads, cfg.kv_heads, cfg.head_dim
        # TP: local head / group / neuron counts (parallel.py fills tp)
        self.H_loc = H if tp is None else tp.heads_local
        self.Hkv_loc = H_kv if tp is None else tp.kv_heads_local
        self.group_base = 0 if tp is None else tp.group_base
        self.d_loc = self.H_loc * d_h
        self.dk_loc = self.Hkv_loc * d_h
        self.sparse_mlp = policy.wants_sparse_mlp(cfg)
        if policy.mode == "dejavu_mlp" and not self.sparse_mlp:
            raise ConfigurationError("dejavu_mlp mode requires a ReLU model and a calibrated k table")
        # per-layer selection budgets (validated up front: ConfigurationError like engine.py:294-301)
        self.k_heads = []
        self.k_mlp = []
        for ell in range(cfg.layers):
            if policy.wants_sparse_heads(ell):
                if head_routers is None or len(head_routers) <= ell or head_routers[ell] is None:
                    raise ConfigurationError(f"no head router available for layer {ell}")
                self.k_heads.append(policy.head_budget(H_kv))
            else:
                self.k_heads.append(0)
            if self.sparse_mlp:
                if mlp_routers is None or len(mlp_routers) <= ell or mlp_routers[ell] is None:
                    raise ConfigurationError(f"no neuron router available for layer {ell}")
                self.k_mlp.append(min(policy.k_for(ell), cfg.ffn_dim))
            else:
                self.k_mlp.append(0)
        # KV caches (optionally aliased storage)
        ring = cfg.layers if kv_ring is None else max(1, min(kv_ring, cfg.layers))
        self.kv_ring = ring
        self.caches = []
        if caches is not None:  # share another engine's caches (e.g. dense vs polar bench)
            if len(caches) != cfg.layers:
                raise ValueError("caches must hold one KVCache per layer")
            self.caches = list(caches)
            ring = 0
        # kv_page_rows > 0: paged caches (block table per sequence, pages
        # reserved for the whole capacity in a scattered order)
        self.kv_page_rows = int(kv_page_rows)
        # "full": every page of the capacity mapped up front; "on_demand": a
        # page is mapped (host allocator + one table-row copy) just before the
        # step whose append enters it -- pool memory follows the actual lengths
        self.kv_reserve = check_choice(kv_reserve, ("full", "on_demand"), "kv_reserve")
        if self.kv_page_rows and tp is not None:
            raise ValueError("paged KV caches are not wired into tensor parallelism")

        def new_cache(i):
            if self.kv_page_rows:
                pc = PagedKVCache(batch, self.Hkv_loc, capacity, d_h, page_rows=self.kv_page_rows, device=dev,
                                  seed=1000 + i)
                if self.kv_reserve == "full":
                    pc.reserve_all()
                return pc
            return KVCache(batch, self.Hkv_loc, capacity, d_h, device=dev)

        base = [new_cache(i) for i in range(ring)]
        for ell in range(cfg.layers if ring else 0):
            c = base[ell % ring]
            if ell >= ring:  # shares the storage (and page table), own lengths
                alias = copy.copy(c)
                alias.lengths = torch.zeros(batch, dtype=torch.int32, device=dev)
                alias.host_lengths = np.zeros(batch, dtype=np.int64)
                alias._err = torch.zeros(1, dtype=torch.int32, device=dev)
                c = alias
            self.caches.append(c)
        self.paged = isinstance(self.caches[0], PagedKVCache)
        # static activation buffers (graph-capturable)
        f32, bf = torch.float32, torch.bfloat16
        D = cfg.ffn_dim
        self.D_loc = D if tp is None else tp.ffn_local
        self.x = torch.zeros(batch, d, dtype=f32, device=dev)
        self.h = torch.zeros(batch, d, dtype=bf, device=dev)
        qkv_w = self.d_loc + 2 * self.dk_loc
        self.qkv = torch.zeros(batch, qkv_w, dtype=bf, device=dev)
        self.attn = torch.zeros(batch, self.d_loc, dtype=bf, device=dev)
        self.hidden = torch.zeros(batch, _round_up(self.D_loc, ROW_PAD), dtype=bf, device=dev)
        self.gu = torch.zeros(batch, 2 * self.D_loc, dtype=bf, device=dev) if cfg.activation == "swiglu" else None
        self.tokens = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.logits = torch.zeros(batch, cfg.vocab, dtype=f32, device=dev)
        self.next_tokens = torch.zeros(batch, dtype=torch.int64, device=dev)
        self.sel_full = torch.arange(H_kv, dtype=torch.int32, device=dev).repeat(batch, 1).contiguous()
        kmax = max(self.k_heads + [1])
        self.sel = torch.zeros(batch, kmax, dtype=torch.int32, device=dev)
        if self.sparse_mlp:
            h_r = mlp_routers[0].hidden_dim_
            self.r_hid = torch.zeros(batch, h_r, dtype=bf, device=dev)
            self.r_logits = torch.zeros(batch, D, dtype=f32, device=dev)
            self.su_bytes = int(_lib.load().ps_select_union_workspace_bytes(batch, D))
            self.su_ws = torch.zeros(self.su_bytes, dtype=torch.uint8, device=dev)
            self.union_idx = torch.zeros(_round_up(D, ROW_PAD), dtype=torch.int32, device=dev)
            # per-layer device union sizes (the count each layer's MLP reads)
            self.union_counts = torch.zeros(cfg.layers, dtype=torch.int32, device=dev)
        # union hand-off: the selection kernel only ORs the rows' sets into a
        # bitmap (two buffers alternating over the layers) and the UP / DOWN
        # GEMMs derive the ids from it, so no compaction sits between top-k and
        # the MLP.  Opt-in (default off): measured ~3 % slower per step at B=16
        # and B=64 (DOWN's id expansion costs more than the compaction it
        # removes).  Needs the tensor-core UP path (B > 4),
        # no TP, split MLP launches, an even number of layers (every layer of a
        # sparse-MLP engine selects; layer ell uses buffer ell % 2, so a
        # replayed step starts on the buffer the previous step's last layer
        # cleared), D <= 32768.
        can = (self.sparse_mlp and tp is None and self.mlp_backend == "split" and cfg.layers % 2 == 0
               and cfg.ffn_dim <= 32768)
        if union_handoff is None:
            union_handoff = False
        if union_handoff and not (can and batch > 4):
            raise ConfigurationError("union_handoff needs a sparse MLP, batch > 4, no TP, mlp_backend='split', an "
                                     "even number of layers and ffn_dim <= 32768")
        self.union_handoff = bool(union_handoff)
        if self.union_handoff:
            self.union_bm = torch.zeros(2, (cfg.ffn_dim + 31) // 32, dtype=torch.int32, device=dev)
        # expected union size per layer: sizes the selective-MLP grids (0 =
        # the maximum).  Set from the device counts of the warm-up step that
        # precedes every capture, so it follows the actual |S| (not k)
        self.union_est = [0] * cfg.layers
        # this engine's own workspaces (tickets / partials; never shared with
        # another engine, never freed while a captured graph may use them)
        self.ws = _ws.Pool()
        self._pending = False  # next_tokens holds a decoded token (after the first step)
        self._captured_len = 0
        self.scale = 1.0 / math.sqrt(d_h)
        self.graph = None
        self.launches_per_step = None
        self.record = None  # eager-only debug capture of selections (parity tests)
        self.trace = None   # device copies of every layer's selections, captured with the graph (tests)

    def enable_trace(self) -> None:
        """Keep a device copy of every layer's head selection and neuron union
        (two D2D copies per layer, recorded into the captured graph too), so a
        replayed step's own selections can be read back: ``trace["heads"][l]``
        (B, k_h), ``trace["union"][l][:union_counts[l]]``.  Call before
        ``capture()``; for parity tests, not for timing."""
        L, dev = self.cfg.layers, self.device
        self.trace = {"heads": [torch.zeros(self.B, max(1, k), dtype=torch.int32, device=dev) for k in self.k_heads],
                      "union": [torch.zeros_like(self.union_idx) if self.sparse_mlp else None for _ in range(L)]}

    # ------------------------------------------------------------------ state
    @property
    def host_lengths(self) -> np.ndarray:
        return self.caches[0].host_lengths

    def fill_random(self, length: int, seed: int = 0) -> None:
        """bench.py:70-100 synthetic_session: N(0,1) history of ``length``."""
        gen = torch.Generator(device=self.device)
        gen.manual_seed(seed)
        for ell, c in enumerate(self.caches):
            if ell < self.kv_ring:
                c.fill_random(gen, length)
            else:
                c.host_lengths[:] = length
                c.lengths.fill_(length)

    def _check_capacity(self) -> None:
        if (self.host_lengths >= self.cfg.max_seq).any():
            raise CapacityError("position table exhausted (max_seq reached)")
        for c in self.caches:
            if (c.host_lengths >= c.capacity).any():
                raise CapacityError(f"KV cache capacity {c.capacity} exhausted")
            if (c.host_lengths < 0).any():
                raise ValueError("negative cache length")

    # ------------------------------------------------------------------ launches
    def _allreduce(self, t: torch.Tensor) -> None:
        if self.tp is not None:
            self.tp.all_reduce(t)

    # ------------------------------------------------------------------ dense glue
    # Plain dense projections (QKV, O, router layers, dense MLP, LM head) run
    # on cuBLAS by default ("plain library GEMMs", identical in dense and
    # polar modes); dense_backend="native" routes them through the tcgen05
    # gathered-GEMM kernel with identity indices instead.
    def _bf(self, t: torch.Tensor) -> torch.Tensor:
        key = ("bf", t.data_ptr())
        c = self._cache.get(key)
        if c is None:
            c = t.to(torch.bfloat16)
            self._cache[key] = c
        return c

    def _scratch(self, name, shape, dtype):
        key = ("scr", name)
        t = self._cache.get(key)
        if t is None or tuple(t.shape) != tuple(shape):
            t = torch.empty(shape, dtype=dtype, device=self.device)
            self._cache[key] = t
        return t

    def _linear_bf16(self, x2d, w_t, bias, out, act_relu=False, tag="gg"):
        """out (bf16) = act(x w^T + bias)."""
        if self.dense_backend == "cublas":
            if bias is not None and act_relu:  # cublasLt RELU_BIAS epilogue
                torch._addmm_activation(self._bf(bias), x2d, w_t.t(), out=out)
            elif bias is not None:
                torch.addmm(self._bf(bias), x2d, w_t.t(), out=out)
            else:
                torch.mm(x2d, w_t.t(), out=out)
                if act_relu:
                    out.relu_()
            return 0
        gather_gemm_into(w_t, None, None, x2d, x2d.stride(0), bias, x2d.shape[0], w_t.shape[0], x2d.shape[1],
                         _lib.PS_ACT_RELU if act_relu else _lib.PS_ACT_NONE, out, out.stride(0), tag=tag)
        return 1

    def _linear_f32(self, x2d, w_t, bias, out, residual=False, tag="gg", defer_bias=False):
        """out (f32) = x w^T + bias (+ out if residual).  cuBLAS accumulates
        the residual in its epilogue (beta = 1).  With ``defer_bias`` the
        bias is NOT added here: the caller hands it to the next
        ps_add_layernorm as the pending bias (returned as the 2nd value)."""
        if self.dense_backend == "cublas" and not (tag == "gg_o" and self.o_backend == "native"):
            if residual:
                torch.addmm(out, x2d, w_t.t(), out_dtype=torch.float32, out=out)
            elif bias is not None and not defer_bias:  # bias in the GEMM epilogue
                torch.addmm(bias, x2d, w_t.t(), out_dtype=torch.float32, out=out)
                bias = None
            else:
                torch.mm(x2d, w_t.t(), out_dtype=torch.float32, out=out)
            if bias is not None and not defer_bias:
                out.add_(bias)
            return (0, bias) if defer_bias else 0
        gather_gemm_into(w_t, None, None, x2d, x2d.stride(0), bias, x2d.shape[0], w_t.shape[0], x2d.shape[1],
                         _lib.PS_ACT_NONE, out, out.stride(0), residual=out if residual else None,
                         res_ld=out.stride(0), tag=tag)
        return (1, None) if defer_bias else 1

    def _ln(self, g, b, pending) -> int:
        """h = layernorm(x (+= pending bias)) -- ps_add_layernorm."""
        d = self.cfg.model_dim
        _lib.check(_lib.load().ps_add_layernorm(_lib.ptr(self.x), d, _lib.ptr(pending) if pending is not None else None,
                                                _lib.ptr(g), _lib.ptr(b), self.B, d, _lib.ptr(self.h), d,
                                                _lib.stream_ptr()), "ps_add_layernorm")
        return 1

    def step_launches(self) -> int:
        """Enqueue one decode step on the current stream; returns the number
        of libpolar_b200 kernel launches enqueued."""
        with _ws.using(self.ws):
            return self._step_launches()

    def _step_launches(self) -> int:
        cfg, m, B = self.cfg, self.model, self.B
        d = cfg.model_dim
        n = 0
        st = _lib.stream_ptr()
        L = _lib.load()
        _lib.check(L.ps_embed(_lib.ptr(self.tokens), _lib.ptr(self.caches[0].lengths), _lib.ptr(m.embed),
                              _lib.ptr(m.pos_embed), B, d, _lib.ptr(self.x), st), "ps_embed")
        n += 1
        qkv_w = self.qkv.shape[1]
        pending = None  # bias of the last residual GEMM, folded into the next LN
        for ell, lw in enumerate(m.layers):
            c = self.caches[ell]
            n += self._ln(lw.ln1_g, lw.ln1_b, pending)
            pending = None
            k_h = self.k_heads[ell]
            if k_h and self.concurrent_router:
                # the head router depends only on h1: run it on a side stream
                # (a parallel graph branch) concurrently with the QKV GEMM
                main = torch.cuda.current_stream()
                self.side.wait_stream(main)
                with torch.cuda.stream(self.side):
                    sel = self._head_select(ell, k_h)
                n += 1
            n += self._linear_bf16(self.h, lw.w_qkv_t, lw.b_qkv, self.qkv, tag="gg_qkv")
            kq = self.qkv[:, self.d_loc:]
            vq = self.qkv[:, self.d_loc + self.dk_loc:]
            if not k_h or self.concurrent_router:
                st = _lib.stream_ptr()
                if self.paged:
                    _lib.check(L.ps_kv_append_paged(_lib.ptr(c.k_pool), _lib.ptr(c.v_pool), c.page_rows,
                                                    _lib.ptr(c.block_table), c.max_pages, _lib.ptr(c.lengths),
                                                    _lib.ptr(kq), _lib.ptr(vq), qkv_w, B, self.Hkv_loc, cfg.head_dim,
                                                    _lib.ptr(c._err), st), "ps_kv_append_paged")
                else:
                    _lib.check(L.ps_kv_append(_lib.ptr(c.keys), _lib.ptr(c.values), _lib.ptr(c.lengths),
                                              _lib.ptr(kq), _lib.ptr(vq), qkv_w, B, self.Hkv_loc, c.capacity,
                                              cfg.head_dim, _lib.ptr(c._err), st), "ps_kv_append")
                n += 1
            if k_h and self.concurrent_router:
                torch.cuda.current_stream().wait_stream(self.side)
            elif k_h:
                # head router + top-k fused with the KV append (one launch)
                sel = self._head_select(ell, k_h, append=(c, kq, vq, qkv_w))
                n += 1
            else:
                sel = self.sel_full
            if self.trace is not None and k_h:
                self.trace["heads"][ell].copy_(sel)
            # the hint only sizes the grid: the kernel reads the tile count from
            # the device lengths, so a captured graph stays exact as they grow
            sha_decode_into(self.qkv, qkv_w, c, sel, self.H_loc, self.scale, self.attn, self.d_loc,
                            group_base=self.group_base, max_len_hint=int(c.host_lengths.max()) + 1)
            n += 1
            if self.tp is None:
                k, pending = self._linear_f32(self.attn, lw.w_o_t, lw.b_o, self.x, residual=True, tag="gg_o",
                                              defer_bias=True)
                n += k
            else:
                n += self.tp.o_proj(self, lw)
            n += self._ln(lw.ln2_g, lw.ln2_b, pending)
            pending = None
            if self.sparse_mlp:
                r = self.mlp_routers[ell]
                cnt = self.union_counts[ell:ell + 1]
                out_bias = None  # the router's output bias is added inside ps_select_union
                if self.router_backend == "fused" and r.fused_into(self.h, self.r_hid, self.r_logits,
                                                                  with_bias=False):
                    out_bias = r.b_out
                    n += 1
                elif self.router_backend in ("cublas", "native_in", "fused"):
                    if self.router_backend == "native_in":  # tcgen05 kernel, static weights prefetched (PDL)
                        gather_gemm_into(r.w_in_t, None, None, self.h, self.h.stride(0), r.b_in, B, r.hidden_dim_,
                                         d, _lib.PS_ACT_RELU, self.r_hid, self.r_hid.stride(0), tag="gg_router")
                        n += 1
                    else:
                        n += self._linear_bf16(self.h, r.w_in_t, r.b_in, self.r_hid, act_relu=True)
                    torch.mm(self.r_hid, r.w_out_t.t(), out_dtype=torch.float32, out=self.r_logits)
                    out_bias = r.b_out
                else:
                    r.logits_into(self.h, self.r_hid, self.r_logits)
                    n += 2
                lo, hi = (0, cfg.ffn_dim) if self.tp is None else self.tp.ffn_range
                if self.union_handoff and self.trace is None and self.record is None:
                    par = ell % 2
                    bm, other = self.union_bm[par], self.union_bm[1 - par]
                    _lib.check(L.ps_select_union_bitmap(_lib.ptr(self.r_logits), _lib.ptr(out_bias), B, cfg.ffn_dim,
                                                        cfg.ffn_dim, self.k_mlp[ell], 0.0, _lib.ptr(bm),
                                                        _lib.ptr(other), st), "ps_select_union_bitmap")
                    mlp_into_bitmap(lw.mlp, self.h, bm, cnt, self.hidden, self.x, residual=self.x,
                                    expected=self.union_est[ell])
                    n += 3
                    continue
                _lib.check(L.ps_select_union(_lib.ptr(self.r_logits), _lib.ptr(out_bias), B, cfg.ffn_dim, cfg.ffn_dim,
                                             self.k_mlp[ell], 0.0, _lib.ptr(self.su_ws), self.su_bytes,
                                             lo, hi, ROW_PAD, _lib.ptr(self.union_idx),
                                             _lib.ptr(cnt), st), "ps_select_union")
                n += 1
                if self.trace is not None:
                    self.trace["union"][ell].copy_(self.union_idx)
                if self.record is not None:
                    lg = self.r_logits.clone()
                    if out_bias is not None:
                        lg += out_bias
                    self.record.setdefault("mlp_logits", []).append(lg)
                    self.record.setdefault("union", []).append(
                        self.union_idx[: int(cnt.item())].clone())
                if self.tp is None and self.mlp_backend == "chain" and B <= 256:
                    sparse_mlp_into(lw.mlp, self.h, self.union_idx, cnt, self.hidden, self.x, residual=self.x)
                    n += 1
                elif self.tp is None:
                    mlp_into(lw.mlp, self.h, self.union_idx, cnt, self.hidden, self.x,
                             residual=self.x, expected=self.union_est[ell])
                    n += 2
                else:
                    n += self.tp.mlp(self, lw, self.union_idx, cnt, ell)
            elif self.tp is not None:
                n += self.tp.mlp(self, lw, None, None, ell)
            elif cfg.activation == "swiglu":
                mk = lw.mlp
                if self.dense_backend == "cublas":
                    torch.mm(self.h, mk.gate_up().t(), out=self.gu)
                    _lib.call("ps_swiglu", _lib.ptr(self.gu), self.gu.stride(0), B, mk.D, _lib.ptr(self.hidden),
                              self.hidden.stride(0), st)
                    n += 1
                    pending = self._dense_down(mk, self.hidden[:, :mk.D])
                else:
                    swiglu_into(mk, self.h, self.gu, self.hidden, self.x, residual=self.x)
                    n += 3
            else:
                mk = lw.mlp
                if self.dense_backend == "cublas":
                    hid = self._scratch("hid", (B, mk.D), torch.bfloat16)
                    n += self._linear_bf16(self.h, mk.w1t, mk.b1, hid, act_relu=True)
                    pending = self._dense_down(mk, hid)
                else:
                    mlp_into(mk, self.h, None, None, self.hidden, self.x, residual=self.x)
                    n += 2
        n += self._ln(m.lnf_g, m.lnf_b, pending)
        n += self._linear_f32(self.h, m.unembed_t, None, self.logits, tag="gg_lm")
        torch.argmax(self.logits, dim=1, out=self.next_tokens)
        return n

    def _head_select(self, ell: int, k_h: int, append=None) -> torch.Tensor:
        """Head router + per-row top-k into the selection buffer (optionally
        fused with the KV append)."""
        B = self.B
        sel = self.sel[:, :k_h]
        if k_h != self.sel.shape[1]:
            sel = self.sel_bufs(k_h)
        hl = None
        if self.record is not None:
            hl = torch.empty(B, self.cfg.kv_heads, dtype=torch.float32, device=self.device)
        if append is None:
            self.head_routers[ell].select_into(self.h, k_h, sel, hl)
        else:
            c, kq, vq, ld = append
            self.head_routers[ell].select_append_into(self.h, k_h, sel, c, kq, vq, ld, hl)
        if self.record is not None:
            self.record.setdefault("head_logits", []).append(hl)
            self.record.setdefault("heads", []).append(sel.clone())
        return sel

    def _dense_down(self, mk, hid):
        """x += hid @ W2 with W2^T stored neuron-major (D, d): a plain
        (B, D) x (D, d) cuBLAS GEMM on the packed rows accumulating into x
        (beta = 1).  Returns b2 as the pending bias of the next LN."""
        torch.addmm(self.x, hid, mk.w2t, out_dtype=torch.float32, out=self.x)
        return mk.b2

    def sel_bufs(self, k: int) -> torch.Tensor:
        key = f"_sel_{k}"
        buf = getattr(self, key, None)
        if buf is None:
            buf = torch.zeros(self.B, k, dtype=torch.int32, device=self.device)
            setattr(self, key, buf)
        return buf

    def _advance(self) -> None:
        for c in self.caches:
            c.host_lengths += 1

    # ------------------------------------------------------------------ public
    def step(self, tokens=None) -> torch.Tensor:
        """engine.py:314-392: advance every sequence by one token; returns the
        (B, vocab) f32 logits (device).  Uses the captured graph if any.
        ``tokens=None`` decodes the previous step's argmax tokens (like the
        reference's pending tokens; ValueError before the first step)."""
        self._check_capacity()
        if tokens is None and not self._pending:
            raise ValueError("no pending tokens: pass the first step's tokens explicitly")
        if tokens is not None:
            tk = torch.as_tensor(np.asarray(tokens) if not isinstance(tokens, torch.Tensor) else tokens)
            if tuple(tk.shape) != (self.B,):
                raise ValueError(f"tokens must have shape ({self.B},), got {tuple(tk.shape)}")
            if tk.dtype.is_floating_point or tk.dtype == torch.bool:
                raise ValueError("tokens must hold integer ids")
            lo, hi = int(tk.min()), int(tk.max())
            if lo < 0 or hi >= self.cfg.vocab:
                raise IndexError(f"tokens must be in [0, {self.cfg.vocab}), got values in [{lo}, {hi}]")
        if self.graph is not None and self._regrow():
            self.capture()  # the sequences outgrew the captured grid size (perf only; see _regrow)
        if self.paged and self.kv_reserve == "on_demand":
            self._map_next_pages()
        if tokens is not None:
            self.tokens.copy_(tk.to(torch.int32), non_blocking=True)
        else:
            self.tokens.copy_(self.next_tokens.to(torch.int32))
        if self.graph is not None:
            self.graph.replay()
        else:
            self.launches_per_step = self.step_launches()
        self._advance()
        self._pending = True
        return self.logits

    def _regrow(self) -> bool:
        """True when the longest sequence has doubled (+256 rows) since the
        capture.  Correctness never needs a re-capture (the SHA kernel reads
        the tile count from the device lengths); the captured SHA grid was
        sized for the capture-time length, so a much longer history is
        re-captured to get a grid sized for it."""
        return int(self.host_lengths.max()) + 1 > 2 * self._captured_len + 256

    def _map_next_pages(self) -> None:
        """Map the page this step's append enters, for every storage buffer
        (aliased layers share their base cache's table)."""
        c0 = self.caches[0]
        if not (c0.host_lengths % c0.page_rows == 0).any():
            return  # no append opens a page this step (every layer advances in lock step)
        seen = set()
        for c in self.caches:
            key = id(c.block_table)
            if key in seen:
                continue
            seen.add(key)
            nxt = c.host_lengths // c.page_rows
            for b in np.nonzero(c.host_table[np.arange(c.batch), nxt] < 0)[0]:
                c.reserve(int(b), int(c.host_lengths[b]) + 1)

    def capture(self, warmup: int = 1) -> None:
        """Capture one step into a CUDA graph (workspaces sized by a warm-up
        step first; the warm-up's KV writes are undone via the lengths).
        The warm-up's union sizes become the expected |S| per layer that
        sizes the captured selective-MLP grids."""
        self.graph = None
        if self.paged and self.kv_reserve == "on_demand":
            self._map_next_pages()  # the warm-up step appends too
        saved = [c.host_lengths.copy() for c in self.caches]
        saved_tokens, saved_next = self.tokens.clone(), self.next_tokens.clone()
        saved_logits = self.logits.clone()
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.launches_per_step = self.step_launches()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        if self.sparse_mlp:
            counts = self.union_counts.cpu().numpy()
            D = self.D_loc if self.tp is not None else self.cfg.ffn_dim
            # 1/16 headroom over the warm-up's union (steps vary); the tile
            # loop still covers any larger union at run time
            self.union_est = [int(min(D, int(c) + int(c) // 16 + ROW_PAD)) if c > 0 else 0 for c in counts]
        for c, hl in zip(self.caches, saved):
            c.host_lengths[:] = hl
            c.lengths.copy_(torch.from_numpy(hl.astype(np.int32)))
        self.tokens.copy_(saved_tokens)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.step_launches()
        torch.cuda.synchronize()
        self.next_tokens.copy_(saved_next)  # the pending tokens of the last real step
        self.logits.copy_(saved_logits)
        self.graph = g
        self._captured_len = int(self.host_lengths.max()) + 1
