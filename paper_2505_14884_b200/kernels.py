"""Sparsity-aware decode kernels -- the drop-in surface of
``sparsedecode.kernels`` (kernels.py:44-548), executed by libpolar_b200.so.

Same names, argument order and error types as the reference; inputs are
torch CUDA tensors (numpy inputs are uploaded), storage is bf16, accumulation
f32.  Differences a caller can observe, all stated in DESIGN.md:

* results are float32 torch tensors on the device, computed from bf16
  operands (tolerance documented in tests/test_gpu_parity.py);
* ``FlashBlockParams.block_size`` and ``variant`` are accepted and validated
  but do not change the GPU schedule (the reference guarantees output
  invariance to both, kernels.py:137-180, tests: block-size invariance);
* MLP weights in the reference layout (d, D) are transposed to neuron-major
  (D, d) on the fly; hot callers pre-pack once with :class:`PackedMLP`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, _ws
from .exceptions import EmptyCacheError
from .tensors import KVCache, PagedKVCache, _rows_topk
from .validation import as_device_tensor, as_index_tensor, check_choice, check_count

_ACTIVATIONS = ("none", "relu")
_VARIANTS = ("running", "deferred")
ROW_PAD = 128  # gathered-GEMM tile rows


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


# ---------------------------------------------------------------------------
# index containers
# ---------------------------------------------------------------------------

class NeuronIndexTensor:
    """Union set of active neurons for one layer and step (kernels.py:44-64).

    Backed by a device int32 buffer whose first ``count`` entries are the
    strictly ascending ids; ``count`` lives on the device (produced by the
    union kernel without a host sync).  ``.indices`` / ``.size`` read it back.
    """

    def __init__(self, layer: int, indices, count=None, validate: bool = True):
        self.layer = int(layer)
        if count is None:
            idx = as_index_tensor(indices, "indices", validate=validate)
            if validate and idx.numel() > 1:
                if bool((idx[1:] <= idx[:-1]).any()):
                    raise ValueError("neuron indices must be strictly ascending")
            n = idx.numel()
            buf = torch.empty(max(_round_up(n, ROW_PAD), ROW_PAD), dtype=torch.int32, device=idx.device)
            buf[:n] = idx
            if n:
                buf[n:] = idx[-1]
            else:
                buf.zero_()
            self.buffer = buf
            self.count = torch.tensor([n], dtype=torch.int32, device=idx.device)
            self._n = n
        else:
            self.buffer = indices
            self.count = count
            self._n = None

    @property
    def size(self) -> int:
        if self._n is None:
            self._n = int(self.count.item())
        return self._n

    @property
    def indices(self) -> torch.Tensor:
        return self.buffer[: self.size]

    def __len__(self) -> int:
        return self.size


class BatchHeadIndex:
    """Active head / KV-group ids per sequence, (batch, top_k) (kernels.py:67-112).

    ``entries`` is a device int32 tensor.  Host-supplied entries are
    validated like the reference (2-D, integer, non-empty, >= 0, rows
    duplicate-free); device-produced ones (``from_logits``, ``full``) are
    correct by construction and skip the sync.
    """

    def __init__(self, entries, validate: bool = True, n_max: int | None = None):
        if validate:
            arr = entries.detach().cpu().numpy() if isinstance(entries, torch.Tensor) else np.asarray(entries)
            if arr.ndim != 2:
                raise ValueError(f"entries must be 2-dimensional, got {arr.shape}")
            if not np.issubdtype(arr.dtype, np.integer):
                raise ValueError("entries must hold integers")
            if arr.size == 0:
                raise ValueError("entries must not be empty")
            if arr.min() < 0:
                raise IndexError("head ids must be non-negative")
            srt = np.sort(arr, axis=1)
            if (srt[:, 1:] == srt[:, :-1]).any():
                raise ValueError("head ids must be unique within a row")
            n_max = int(arr.max()) + 1
        self.entries = as_device_tensor(entries, "entries").to(torch.int32).contiguous()
        self._n_max = n_max  # exclusive upper bound of the ids, when known

    @property
    def batch(self) -> int:
        return self.entries.shape[0]

    @property
    def top_k(self) -> int:
        return self.entries.shape[1]

    @classmethod
    def full(cls, batch: int, n_heads: int, device=None) -> "BatchHeadIndex":
        e = torch.arange(n_heads, dtype=torch.int32, device=device or "cuda").repeat(batch, 1)
        return cls(e, validate=False, n_max=n_heads)

    @classmethod
    def from_logits(cls, logits, top_k: int) -> "BatchHeadIndex":
        """Per-row top-k of router logits; ties go to the lower head id."""
        s = as_device_tensor(logits, "logits")
        if s.ndim == 1:
            s = s[None, :]
        if not 1 <= top_k <= s.shape[1]:
            raise ValueError(f"k must be in [1, {s.shape[1]}], got {top_k}")
        return cls(_rows_topk(s, int(top_k)), validate=False, n_max=s.shape[1])


@dataclass(frozen=True)
class FlashBlockParams:
    """Key-block size (kernels.py:115-135).  Accepted for API parity; the
    GPU tile is fixed by the hardware mapping (8 KB K + 8 KB V per stage)
    and the output is invariant to it, as the reference guarantees."""

    block_size: int = 64

    def __post_init__(self):
        check_count(self.block_size, "block_size")

    def num_blocks(self, n_kv: int) -> int:
        return -(-int(n_kv) // self.block_size)

    @classmethod
    def from_byte_budget(cls, budget_bytes: int, model_dim: int) -> "FlashBlockParams":
        return cls(max(1, int(budget_bytes) // (4 * int(model_dim))))


class OnlineSoftmaxState:
    """Running (accumulator, normalizer, max) of the one-pass softmax
    (kernels.py:138-180), held on the device in float64.

    The SHA kernel runs the same recurrence per warp in f32 registers (its
    ``(m, l, o)`` partials merge like :meth:`update`); this object is the
    single-unit reference path that exposes the state for inspection.
    """

    def __init__(self, o_acc: torch.Tensor, l_acc: float = 0.0, m_acc: float = -math.inf):
        self.o_acc = o_acc
        self.l_acc = float(l_acc)
        self.m_acc = float(m_acc)

    @classmethod
    def fresh(cls, head_dim: int, device=None) -> "OnlineSoftmaxState":
        from .validation import default_device
        return cls(torch.zeros(int(head_dim), dtype=torch.float64, device=device or default_device()))

    def update(self, scores, v_block, variant: str = "running") -> None:
        """Fold one key block (already-scaled scores, matching value rows)."""
        check_choice(variant, _VARIANTS, "variant")
        s = as_device_tensor(scores, "scores", device=self.o_acc.device).to(torch.float64)
        v = as_device_tensor(v_block, "v_block", device=self.o_acc.device).to(torch.float64)
        m_tilde = float(s.max())
        p = torch.exp(s - m_tilde)
        l_tilde = float(p.sum())
        m_new = max(self.m_acc, m_tilde)
        alpha = math.exp(self.m_acc - m_new)
        beta = math.exp(m_tilde - m_new)
        l_new = alpha * self.l_acc + beta * l_tilde
        pv = p @ v
        if variant == "running":
            self.o_acc = (alpha * self.l_acc * self.o_acc + beta * pv) / l_new
        else:
            self.o_acc = alpha * self.o_acc + beta * pv
        self.l_acc = l_new
        self.m_acc = m_new

    def output(self, variant: str = "running") -> torch.Tensor:
        if variant == "deferred":
            return self.o_acc / self.l_acc
        return self.o_acc


def online_softmax_attention(q, keys, values, scale: float, params: "FlashBlockParams" = None,
                             variant: str = "running"):
    """kernels.py:183-210: single-unit blocked attention over ``keys`` /
    ``values`` (N, d_h) in blocks of ``params.block_size``; returns
    (f32 output, final :class:`OnlineSoftmaxState`)."""
    params = params or FlashBlockParams()
    check_choice(variant, _VARIANTS, "variant")
    qv = as_device_tensor(q, "q", ndim=1)
    k = as_device_tensor(keys, "keys", device=qv.device, ndim=2)
    v = as_device_tensor(values, "values", device=qv.device, ndim=2)
    if k.shape[0] == 0:
        raise EmptyCacheError("attention over an empty key/value history")
    n_kv = k.shape[0]
    state = OnlineSoftmaxState.fresh(qv.shape[0], device=qv.device)
    q64 = qv.to(torch.float64)
    for j in range(params.num_blocks(n_kv)):
        k0, k1 = j * params.block_size, min((j + 1) * params.block_size, n_kv)
        state.update(scale * (k[k0:k1].to(torch.float64) @ q64), v[k0:k1], variant=variant)
    return state.output(variant).to(torch.float32), state


# ---------------------------------------------------------------------------
# Select-Head Attention
# ---------------------------------------------------------------------------

def sha_decode_into(q2d: torch.Tensor, q_ld: int, cache, sel: torch.Tensor, n_heads: int,
                    scale: float, out: torch.Tensor, out_ld: int, group_base: int = 0,
                    num_splits: int = 0, max_len_hint: int = 0) -> None:
    """Raw launch (no validation) used by the engine's captured step;
    ``cache`` is a KVCache or a PagedKVCache."""
    B, H_kv, cap, d_h = cache.batch, cache.kv_heads, cache.capacity, cache.head_dim
    k = sel.shape[1]
    lib = _lib.load()
    if num_splits == 0:
        num_splits = lib.ps_sha_auto_splits(B, H_kv, d_h, k, max_len_hint or cap)
    nbytes = lib.ps_sha_workspace_bytes(B, n_heads, H_kv, d_h, k, num_splits)
    ws = _ws.get("sha", nbytes, cache.device)
    dt = _lib.PS_DTYPE_BF16 if out.dtype == torch.bfloat16 else _lib.PS_DTYPE_F32
    if isinstance(cache, PagedKVCache):
        _lib.call("ps_sha_decode_paged", _lib.ptr(q2d), int(q_ld), _lib.ptr(cache.k_pool), _lib.ptr(cache.v_pool),
                  cache.pool_pages, cache.page_rows, _lib.ptr(cache.block_table), cache.max_pages,
                  _lib.ptr(cache.lengths), _lib.ptr(sel), int(group_base), B, n_heads, H_kv, d_h, k,
                  float(scale), int(num_splits), int(max_len_hint), _lib.ptr(out), int(out_ld), dt,
                  _lib.ptr(ws), ws.numel(), _lib.stream_ptr())
        return
    _lib.call("ps_sha_decode", _lib.ptr(q2d), int(q_ld), _lib.ptr(cache.keys), _lib.ptr(cache.values),
              _lib.ptr(cache.lengths), _lib.ptr(sel), int(group_base), B, n_heads, H_kv, cap, d_h, k,
              float(scale), int(num_splits), int(max_len_hint), _lib.ptr(out), int(out_ld), dt,
              _lib.ptr(ws), ws.numel(), _lib.stream_ptr())


def _check_attention_args(q, cache: KVCache, bhi: BatchHeadIndex, scale):
    """kernels.py:447-461."""
    q4 = as_device_tensor(q, "q", device=cache.device)
    if q4.ndim != 4 or q4.shape[2] != 1:
        raise ValueError(f"q must have a singleton query axis (B, H, 1, d_h), got {tuple(q4.shape)}")
    batch, _, _, d_h = q4.shape
    if cache.batch != batch or cache.head_dim != d_h:
        raise ValueError(f"cache shape {(cache.batch, cache.kv_heads, cache.capacity, cache.head_dim)} "
                         f"inconsistent with query {tuple(q4.shape)}")
    if bhi.batch != batch:
        raise ValueError(f"batch_head_index covers {bhi.batch} sequences, not {batch}")
    if (cache.host_lengths < 1).any():
        empty = np.nonzero(cache.host_lengths < 1)[0]
        raise EmptyCacheError(f"sequences {empty.tolist()} have empty caches")
    if not scale > 0:
        raise ValueError(f"scale must be positive, got {scale}")
    return q4


def gqa_selective_attention_decode(q, cache: KVCache, group_index: BatchHeadIndex,
                                   params: FlashBlockParams = FlashBlockParams(),
                                   scale: float | None = None, variant: str = "running",
                                   *, out_dtype=torch.float32, num_splits: int = 0) -> torch.Tensor:
    """kernels.py:513-548 on the SHA kernel.  Selecting group g activates the
    G = H/H_kv query heads sharing KV head g; non-selected heads are exact
    zeros and their cache rows are never read."""
    check_choice(variant, _VARIANTS, "variant")
    d_h = q.shape[-1]
    if scale is None:
        scale = 1.0 / math.sqrt(d_h)
    q4 = _check_attention_args(q, cache, group_index, scale)
    batch, n_heads = q4.shape[0], q4.shape[1]
    n_groups = cache.kv_heads
    if n_heads % n_groups != 0:
        raise ValueError(f"{n_heads} query heads not divisible by {n_groups} groups")
    nmax = group_index._n_max
    if nmax is None or nmax > n_groups:
        if int(group_index.entries.max()) >= n_groups:
            raise IndexError(f"group ids must be < {n_groups}")
    qb = q4.to(torch.bfloat16).reshape(batch, n_heads * d_h).contiguous()
    out = torch.empty((batch, n_heads * d_h), dtype=out_dtype, device=cache.device)
    sha_decode_into(qb, n_heads * d_h, cache, group_index.entries, n_heads, scale, out, n_heads * d_h,
                    num_splits=num_splits, max_len_hint=int(cache.host_lengths.max()))
    return out.view(batch, n_heads, 1, d_h)


def selective_head_flash_attention_decode(q, cache: KVCache, batch_head_index: BatchHeadIndex,
                                          params: FlashBlockParams = FlashBlockParams(),
                                          scale: float | None = None, variant: str = "running",
                                          **kw) -> torch.Tensor:
    """kernels.py:464-510: MHA entry point (one KV head per query head)."""
    check_choice(variant, _VARIANTS, "variant")
    n_heads = q.shape[1]
    if cache.kv_heads != n_heads:
        raise ValueError(
            f"cache has {cache.kv_heads} KV heads but query has {n_heads}; "
            "use gqa_selective_attention_decode for grouped KV")
    nmax = batch_head_index._n_max
    if (nmax is None or nmax > n_heads) and int(batch_head_index.entries.max()) >= n_heads:
        raise IndexError(f"head ids must be < {n_heads}")
    return gqa_selective_attention_decode(q, cache, batch_head_index, params, scale, variant, **kw)


# ---------------------------------------------------------------------------
# gathered GEMM / MLP
# ---------------------------------------------------------------------------

def gather_gemm_into(w_rows, idx, count, x, x_ld, bias, N, M, K, act, out, out_ld,
                     residual=None, res_ld=0, splits=0, tag="gg_up", flags=0):
    """Raw rows-form launch (see include/polar_b200.h ps_gather_gemm)."""
    lib = _lib.load()
    if splits <= 0:
        splits = lib.ps_gather_gemm_auto_splits(N, M, K)
    ws = _ws.get(tag, lib.ps_gather_gemm_workspace_bytes(N, M, K, splits), out.device)
    dt = _lib.PS_DTYPE_BF16 if out.dtype == torch.bfloat16 else _lib.PS_DTYPE_F32
    _lib.call("ps_gather_gemm", _lib.ptr(w_rows), w_rows.shape[0], _lib.ptr(idx), _lib.ptr(count), _lib.ptr(x),
              int(x_ld),
              _lib.ptr(bias), _lib.ptr(residual), int(res_ld), N, M, K, act, splits, flags, _lib.ptr(out),
              int(out_ld), dt, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())


def gather_gemm_t_into(w_rows, idx, count, h, h_ld, bias, N, M, K_max, out, out_ld,
                       residual=None, res_ld=0, splits=0, tag="gg_down", flags=0):
    """Raw contraction-form launch (ps_gather_gemm_t)."""
    lib = _lib.load()
    if splits <= 0:
        splits = lib.ps_gather_gemm_auto_splits(N, M, K_max)
    ws = _ws.get(tag, lib.ps_gather_gemm_workspace_bytes(N, M, K_max, splits), out.device)
    dt = _lib.PS_DTYPE_BF16 if out.dtype == torch.bfloat16 else _lib.PS_DTYPE_F32
    _lib.call("ps_gather_gemm_t", _lib.ptr(w_rows), w_rows.shape[0], _lib.ptr(idx), _lib.ptr(count), _lib.ptr(h),
              int(h_ld),
              _lib.ptr(bias), _lib.ptr(residual), int(res_ld), N, M, K_max, splits, flags, _lib.ptr(out),
              int(out_ld), dt, _lib.ptr(ws), ws.numel(), _lib.stream_ptr())


class PackedMLP:
    """Neuron-major bf16 copy of one MLP block (packed once at load).

    ``w1t``/``w2t`` (and ``w3t`` for SwiGLU) are (D, d): row j is neuron j's
    input / output weights, a contiguous 2*d-byte gather unit.  The
    reference stores both as (d, D) with the neuron axis innermost
    (model.py:1-8, 105-106); ``from_reference`` transposes.
    """

    def __init__(self, w1t, b1, w2t, b2, w3t=None):
        self.w1t, self.w2t, self.w3t = w1t, w2t, w3t
        self.b1, self.b2 = b1, b2
        self.D, self.d = w1t.shape
        self.D_pad = _round_up(self.D, ROW_PAD)
        self._gu = None

    @classmethod
    def from_reference(cls, w1, b1, w2, b2, w3=None, device=None) -> "PackedMLP":
        w1 = as_device_tensor(w1, "w1", device=device, ndim=2)
        w2 = as_device_tensor(w2, "w2", device=device, ndim=2)
        d, D = w1.shape
        if tuple(w2.shape) != (d, D):
            raise ValueError("MLP weight shapes inconsistent with input")
        b1t = None if b1 is None else as_device_tensor(b1, "b1", dtype=torch.float32, device=w1.device, ndim=1)
        b2t = None if b2 is None else as_device_tensor(b2, "b2", dtype=torch.float32, device=w1.device, ndim=1)
        w3t = None
        if w3 is not None:
            w3t = as_device_tensor(w3, "w3", device=w1.device, ndim=2).t().to(torch.bfloat16).contiguous()
        return cls(w1.t().to(torch.bfloat16).contiguous(), b1t, w2.t().to(torch.bfloat16).contiguous(),
                   b2t, w3t)

    def gate_up(self) -> torch.Tensor:
        """[W1^T; W3^T] stacked (2D, d) for the fused SwiGLU up-projection."""
        if self._gu is None:
            self._gu = torch.cat([self.w1t, self.w3t], 0).contiguous()
        return self._gu


def _hidden_in(x, name="x"):
    x = as_device_tensor(x, name)
    if x.ndim != 3 or x.shape[1] != 1:
        raise ValueError(f"{name} must have a singleton token axis (batch, 1, d), got {tuple(x.shape)}")
    return x


def _pad_cols(t: torch.Tensor, mult: int = 8) -> torch.Tensor:
    c = t.shape[-1]
    if c % mult == 0:
        return t.contiguous()
    return torch.nn.functional.pad(t, (0, mult - c % mult)).contiguous()


def _resolve(active, upper: int, device) -> NeuronIndexTensor:
    """kernels.py:259-265."""
    if isinstance(active, NeuronIndexTensor):
        if active._n is not None:
            if active._n == 0:
                raise ValueError("active must select at least one column")
            if int(active.indices.max()) >= upper:
                raise IndexError(f"active contains indices >= {upper}")
        return active
    idx = as_index_tensor(active, "active", upper=upper, device=device)
    if idx.numel() == 0:
        raise ValueError("active must select at least one column")
    return NeuronIndexTensor(0, idx, validate=False)


def _mlp_packed(x, w1, b1, w2, b2, w3=None) -> PackedMLP:
    if isinstance(w1, PackedMLP):
        return w1
    return PackedMLP.from_reference(w1, b1, w2, b2, w3, device=x.device)


def mlp_into(pk: PackedMLP, x2d: torch.Tensor, idx, count, hidden: torch.Tensor, out: torch.Tensor,
             residual=None, splits_up=0, splits_down=0, expected=0) -> None:
    """relu(x W1[:, S] + b1[S]) W2[:, S]^T + b2 (+ residual) into ``out``.

    ``idx``/``count`` = None runs the dense MLP through the same kernels.
    ``hidden`` is a bf16 (B, D_pad) scratch buffer.
    """
    B, d = x2d.shape
    gather_gemm_into(pk.w1t, idx, count, x2d, x2d.stride(0), pk.b1, B, pk.D if idx is None else pk.D_pad,
                     d, _lib.PS_ACT_RELU, hidden, hidden.stride(0), splits=splits_up or expected, tag="gg_up")
    gather_gemm_t_into(pk.w2t, idx, count, hidden, hidden.stride(0), pk.b2, B, d,
                       pk.D if idx is None else pk.D_pad, out, out.stride(0),
                       residual=residual, res_ld=0 if residual is None else residual.stride(0),
                       splits=splits_down or expected, tag="gg_down",
                       flags=_lib.PS_GG_A_READY)  # idx/count were written before the UP launch


def mlp_into_bitmap(pk: PackedMLP, x2d: torch.Tensor, bitmap: torch.Tensor, count, hidden: torch.Tensor,
                    out: torch.Tensor, residual=None, expected=0) -> None:
    """:func:`mlp_into` over the union given as a selection BITMAP (the
    union hand-off: ps_select_union_bitmap wrote it, PS_GG_BITMAP makes UP
    and DOWN derive the ids on the device).  ``count`` (int32 device scalar
    or None) receives the union size from UP."""
    B, d = x2d.shape
    gather_gemm_into(pk.w1t, bitmap, count, x2d, x2d.stride(0), pk.b1, B, pk.D_pad, d, _lib.PS_ACT_RELU, hidden,
                     hidden.stride(0), splits=expected, tag="gg_up", flags=_lib.PS_GG_BITMAP)
    gather_gemm_t_into(pk.w2t, bitmap, None, hidden, hidden.stride(0), pk.b2, B, d, pk.D_pad, out, out.stride(0),
                       residual=residual, res_ld=0 if residual is None else residual.stride(0), splits=expected,
                       tag="gg_down", flags=_lib.PS_GG_A_READY | _lib.PS_GG_BITMAP)


def sparse_mlp_into(pk: PackedMLP, x2d: torch.Tensor, idx, count, hidden: torch.Tensor, out: torch.Tensor,
                    residual=None, tag: str = "mlp_chain") -> None:
    """The whole selective MLP in ONE launch (ps_sparse_mlp): UP over the
    union rows, ReLU, DOWN over the same rows, + b2, ADDED into ``out``
    (f32).  ``residual``: ``out`` is set to it first (``out`` itself: in
    place; None: out = MLP only).  ``idx`` / ``count`` None = every neuron.
    Batch <= 256 (else :func:`mlp_into`)."""
    B, d = x2d.shape
    if out.dtype != torch.float32:
        raise ValueError("sparse_mlp_into accumulates into an f32 output")
    if residual is None:
        out.zero_()
    elif residual is not out:
        out.copy_(residual)
    lib = _lib.load()
    ws = _ws.get(tag, lib.ps_sparse_mlp_workspace_bytes(B, pk.D, d), x2d.device)
    _lib.call("ps_sparse_mlp", _lib.ptr(pk.w1t), _lib.ptr(pk.b1), _lib.ptr(pk.w2t), _lib.ptr(pk.b2), pk.D, d,
              _lib.ptr(idx), _lib.ptr(count), _lib.ptr(x2d), x2d.stride(0), B, _lib.ptr(hidden), hidden.stride(0),
              _lib.ptr(out), out.stride(0), _lib.ptr(ws), ws.numel(), _lib.stream_ptr())


def sparse_mlp_forward(x, w1, b1=None, w2=None, b2=None, active=None) -> torch.Tensor:
    """kernels.py:353-373: ReLU MLP restricted to the union set ``active``.

    ``w1`` may be a :class:`PackedMLP` (then b1/w2/b2 are ignored).  The
    hidden activations are rounded to bf16 between the projections.
    """
    x = _hidden_in(x)
    pk = _mlp_packed(x, w1, b1, w2, b2)
    batch, _, d = x.shape
    if d != pk.d:
        raise ValueError("MLP weight shapes inconsistent with input")
    nit = _resolve(active, pk.D, x.device)
    x2 = x[:, 0, :].to(torch.bfloat16).contiguous()
    if d % 8:
        raise ValueError("model_dim must be a multiple of 8 on the GPU path")
    hidden = torch.empty((batch, pk.D_pad), dtype=torch.bfloat16, device=x.device)
    out = torch.empty((batch, d), dtype=torch.float32, device=x.device)
    mlp_into(pk, x2, nit.buffer, nit.count, hidden, out)
    return out.view(batch, 1, d)


def dense_mlp_forward(x, w1, b1=None, w2=None, b2=None) -> torch.Tensor:
    """kernels.py:313-332: the same kernels with every neuron selected."""
    x = _hidden_in(x)
    pk = _mlp_packed(x, w1, b1, w2, b2)
    batch, _, d = x.shape
    if d != pk.d:
        raise ValueError("MLP weight shapes inconsistent with input")
    x2 = x[:, 0, :].to(torch.bfloat16).contiguous()
    hidden = torch.empty((batch, pk.D_pad), dtype=torch.bfloat16, device=x.device)
    out = torch.empty((batch, d), dtype=torch.float32, device=x.device)
    mlp_into(pk, x2, None, None, hidden, out)
    return out.view(batch, 1, d)


def swiglu_into(pk: PackedMLP, x2d, gu, hidden, out, residual=None) -> None:
    B, d = x2d.shape
    D = pk.D
    gather_gemm_into(pk.gate_up(), None, None, x2d, x2d.stride(0), None, B, 2 * D, d, _lib.PS_ACT_NONE,
                     gu, gu.stride(0), tag="gg_up")
    _lib.call("ps_swiglu", _lib.ptr(gu), gu.stride(0), B, D, _lib.ptr(hidden), hidden.stride(0),
              _lib.stream_ptr())
    gather_gemm_t_into(pk.w2t, None, None, hidden, hidden.stride(0), pk.b2, B, d, D, out, out.stride(0),
                       residual=residual, res_ld=0 if residual is None else residual.stride(0), tag="gg_down")


def swiglu_mlp_forward(x, w1, w3=None, w2=None, b2=None) -> torch.Tensor:
    """kernels.py:335-350: dense gated MLP (never sparsified)."""
    x = _hidden_in(x)
    pk = w1 if isinstance(w1, PackedMLP) else PackedMLP.from_reference(w1, None, w2, b2, w3, device=x.device)
    batch, _, d = x.shape
    x2 = x[:, 0, :].to(torch.bfloat16).contiguous()
    gu = torch.empty((batch, 2 * pk.D), dtype=torch.bfloat16, device=x.device)
    hidden = torch.empty((batch, _round_up(pk.D, 8)), dtype=torch.bfloat16, device=x.device)
    out = torch.empty((batch, d), dtype=torch.float32, device=x.device)
    swiglu_into(pk, x2, gu, hidden, out)
    return out.view(batch, 1, d)


def selective_gemm(a, b, indices, activation: str = "none", bias=None) -> torch.Tensor:
    """kernels.py:268-291: act(a @ b[:, indices] + bias[indices]), (M, |I|) f32."""
    check_choice(activation, _ACTIVATIONS, "activation")
    a = as_device_tensor(a, "a", ndim=2)
    b = as_device_tensor(b, "b", ndim=2, device=a.device)
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"selective_gemm shape mismatch: {tuple(a.shape)} x {tuple(b.shape)}")
    nit = _resolve(indices, b.shape[1], a.device)
    n = nit.size
    M_rows, K = a.shape
    a16 = _pad_cols(a.to(torch.bfloat16))
    bt = _pad_cols(b.t().to(torch.bfloat16))
    Kp = a16.shape[1]
    bias_t = None if bias is None else as_device_tensor(bias, "bias", dtype=torch.float32, device=a.device, ndim=1)
    out = torch.empty((M_rows, n), dtype=torch.float32, device=a.device)
    act = _lib.PS_ACT_RELU if activation == "relu" else _lib.PS_ACT_NONE
    gather_gemm_into(bt, nit.buffer, None, a16, Kp, bias_t, M_rows, n, Kp, act, out, n)
    return out


def selective_gemm_t(a, b, indices, bias=None) -> torch.Tensor:
    """kernels.py:294-310: a @ b[:, indices].T (+ bias), (M, K) f32."""
    a = as_device_tensor(a, "a", ndim=2)
    b = as_device_tensor(b, "b", ndim=2, device=a.device)
    nit = _resolve(indices, b.shape[1], a.device)
    n = nit.size
    if a.shape[1] != n:
        raise ValueError(f"a has {a.shape[1]} columns but {n} indices were selected")
    M_rows = a.shape[0]
    K_out = b.shape[0]
    h = _pad_cols(a.to(torch.bfloat16))
    wt = _pad_cols(b.t().to(torch.bfloat16))  # (N, K_out padded)
    Mp = wt.shape[1]
    bias_t = None
    if bias is not None:
        bias_t = torch.zeros(Mp, dtype=torch.float32, device=a.device)
        bias_t[:K_out] = as_device_tensor(bias, "bias", dtype=torch.float32, device=a.device, ndim=1)
    out = torch.empty((M_rows, Mp), dtype=torch.float32, device=a.device)
    gather_gemm_t_into(wt, nit.buffer, None, h, h.shape[1], bias_t, M_rows, Mp, n, out, Mp)
    return out[:, :K_out]


# ---------------------------------------------------------------------------
# union
# ---------------------------------------------------------------------------

def union_into(rows_idx: torch.Tensor, width: int, bitmap: torch.Tensor, idx_out: torch.Tensor,
               count_out: torch.Tensor, lo: int = 0, hi: int | None = None) -> None:
    """OR an id matrix into the bitmap and compact it (device only)."""
    r, k = rows_idx.shape
    _lib.call("ps_union_rows", _lib.ptr(rows_idx), r, k, width, _lib.ptr(bitmap), _lib.stream_ptr())
    _lib.call("ps_bitmap_compact", _lib.ptr(bitmap), width, lo, width if hi is None else hi, ROW_PAD,
              _lib.ptr(idx_out), _lib.ptr(count_out), _lib.stream_ptr())


def union_neuron_indices(per_sequence_sets, layer: int = 0, width: int | None = None) -> NeuronIndexTensor:
    """kernels.py:376-383: sorted, de-duplicated union (device bitmap + compaction)."""
    if isinstance(per_sequence_sets, torch.Tensor) and per_sequence_sets.ndim == 2:
        rows = per_sequence_sets.to(torch.int32).contiguous()
        if not rows.is_cuda:
            rows = as_device_tensor(rows, "per_sequence_sets")
    else:
        parts = [as_index_tensor(s, "per_sequence_sets").reshape(-1) for s in per_sequence_sets]
        if not parts or sum(p.numel() for p in parts) == 0:
            return NeuronIndexTensor(layer, np.empty(0, dtype=np.int64))
        rows = torch.cat(parts)[None, :].contiguous()
    if rows.numel() and int(rows.min()) < 0:
        raise IndexError("per_sequence_sets contains negative indices")
    if width is None:
        width = int(rows.max()) + 1 if rows.numel() else 1
    dev = rows.device
    bitmap = _ws.get("union_bitmap", ((width + 31) // 32) * 4, dev).view(torch.int32)
    buf = torch.empty(_round_up(width, ROW_PAD), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    union_into(rows, width, bitmap, buf, cnt)
    return NeuronIndexTensor(layer, buf, cnt)
