"""Device substrate: the KV cache and the bit-exact top-k.

Mirrors ``sparsedecode.tensors`` (tensors.py:24-213) on B200: the cache
keeps the reference's (B, H_kv, capacity, d_h) layout -- every selected
(sequence, KV group) history is one contiguous slab, which is what lets the
SHA kernel stage it with bulk async copies -- but stores bf16 K/V and int32
lengths in HBM.  A host mirror of ``lengths`` lets capacity / empty-cache
errors be raised before launch without a device sync.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .exceptions import CapacityError, EmptyCacheError
from .validation import as_device_tensor, check_count

MATMUL_TILE = 256  # tensors.py:24-26 (kept for API parity)


def _rows_topk(scores: torch.Tensor, k: int) -> torch.Tensor:
    scores = scores.contiguous()
    if scores.dtype != torch.float32:
        scores = scores.float()
    rows, cols = scores.shape
    out = torch.empty((rows, k), dtype=torch.int32, device=scores.device)
    _lib.call("ps_topk_rows", _lib.ptr(scores), rows, cols, cols, k, _lib.ptr(out), None,
              _lib.stream_ptr())
    return out


def topk_indices_rows(scores, k: int) -> torch.Tensor:
    """tensors.py:65-73: row-wise top-k, ascending ids, ties to the lower index.

    Bit-exact with the reference given identical f32 scores (-0.0 == +0.0,
    NaN ranks below -inf).  Returns int32 (rows, k) on the scores' device.
    """
    s = as_device_tensor(scores, "scores")
    if s.ndim != 2:
        raise ValueError(f"scores must be 2-dimensional, got shape {tuple(s.shape)}")
    if not 1 <= k <= s.shape[1]:
        raise ValueError(f"k must be in [1, {s.shape[1]}], got {k}")
    return _rows_topk(s, int(k))


def topk_indices(scores, k: int) -> torch.Tensor:
    """tensors.py:54-62: 1-D top-k with the same tie rule."""
    s = as_device_tensor(scores, "scores")
    if s.ndim != 1:
        raise ValueError(f"scores must be 1-dimensional, got shape {tuple(s.shape)}")
    if not 1 <= k <= s.shape[0]:
        raise ValueError(f"k must be in [1, {s.shape[0]}], got {k}")
    return _rows_topk(s[None, :], int(k))[0]


def _raise_append_error(cache) -> None:
    code = int(cache._err.item())
    if code:
        cache._err.zero_()
        if code == 2:
            raise ValueError("KV append into an unmapped page (reserve the page before the step)")
        raise CapacityError(f"KV cache capacity {cache.capacity} exhausted on the device")


def matmul64(a, b) -> torch.Tensor:
    """tensors.py:42-51: float64-accumulated product on the device (cuBLAS
    DGEMM; the reference's 256-column tiling does not change the result)."""
    a = as_device_tensor(a, "a", ndim=2)
    b = as_device_tensor(b, "b", ndim=2, device=a.device)
    return a.to(torch.float64) @ b.to(torch.float64)


def matmul(a, b) -> torch.Tensor:
    """tensors.py:29-39: dense float32 product with float64 accumulation."""
    a = as_device_tensor(a, "a", ndim=2)
    b = as_device_tensor(b, "b", ndim=2, device=a.device)
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"matmul shape mismatch: {tuple(a.shape)} x {tuple(b.shape)} (inner dims differ)")
    return matmul64(a, b).to(torch.float32)


def naive_softmax_attention_single_head(q, keys, values, scale: float) -> torch.Tensor:
    """tensors.py:83-113: two-pass (max-subtract) softmax attention for one
    head of one sequence, float64 on the device -- the stability reference
    the blocked SHA kernel is validated against."""
    q = as_device_tensor(q, "q", ndim=1)
    keys = as_device_tensor(keys, "keys", ndim=2, device=q.device)
    values = as_device_tensor(values, "values", ndim=2, device=q.device)
    if keys.shape[0] == 0:
        raise EmptyCacheError("attention over an empty key/value history")
    if tuple(keys.shape) != tuple(values.shape):
        raise ValueError(f"keys {tuple(keys.shape)} and values {tuple(values.shape)} differ")
    if keys.shape[1] != q.shape[0]:
        raise ValueError(f"q dim {q.shape[0]} != head dim {keys.shape[1]}")
    if not scale > 0:
        raise ValueError(f"scale must be positive, got {scale}")
    s = scale * (keys.to(torch.float64) @ q.to(torch.float64))
    p = torch.exp(s - s.max())
    return ((p @ values.to(torch.float64)) / p.sum()).to(torch.float32)


class KVCache:
    """Per-layer K/V history in HBM (tensors.py:116-213 semantics).

    ``keys``/``values``: bf16 (batch, kv_heads, capacity, head_dim);
    ``lengths``: int32 device vector; ``host_lengths``: int64 numpy mirror.
    """

    def __init__(self, batch: int, kv_heads: int, capacity: int, head_dim: int,
                 device="cuda", dtype=torch.bfloat16):
        check_count(batch, "batch")
        check_count(kv_heads, "kv_heads")
        check_count(capacity, "capacity")
        check_count(head_dim, "head_dim")
        if dtype != torch.bfloat16:
            raise ValueError("the B200 cache stores bf16 K/V")
        shape = (batch, kv_heads, capacity, head_dim)
        self.keys = torch.zeros(shape, dtype=dtype, device=device)
        self.values = torch.zeros(shape, dtype=dtype, device=device)
        self.lengths = torch.zeros(batch, dtype=torch.int32, device=device)
        self.host_lengths = np.zeros(batch, dtype=np.int64)
        self._err = torch.zeros(1, dtype=torch.int32, device=device)

    @classmethod
    def from_reference(cls, cache, device="cuda") -> "KVCache":
        """Device copy of a reference ``KVCache`` (tensors.py:116-148 fields
        ``keys``/``values`` f32 (B, H_kv, cap, d_h) and ``lengths``), rounded
        to bf16.  Used by the parity adapter only (a full H2D copy)."""
        keys = np.asarray(cache.keys)
        b, h, cap, d_h = keys.shape
        out = cls(b, h, cap, d_h, device=device)
        out.keys.copy_(torch.from_numpy(np.ascontiguousarray(keys, dtype=np.float32)))
        out.values.copy_(torch.from_numpy(np.ascontiguousarray(np.asarray(cache.values), dtype=np.float32)))
        out.host_lengths[:] = np.asarray(cache.lengths, dtype=np.int64)
        out._sync_lengths()
        return out

    @property
    def batch(self) -> int:
        return self.keys.shape[0]

    @property
    def kv_heads(self) -> int:
        return self.keys.shape[1]

    @property
    def capacity(self) -> int:
        return self.keys.shape[2]

    @property
    def head_dim(self) -> int:
        return self.keys.shape[3]

    @property
    def device(self):
        return self.keys.device

    def _sync_lengths(self) -> None:
        self.lengths.copy_(torch.from_numpy(self.host_lengths.astype(np.int32)))

    def append_step(self, k_new, v_new, src_ld=None) -> None:
        """tensors.py:150-170 -- one token for every sequence (device kernel).

        ``k_new``/``v_new``: (batch, kv_heads, head_dim) bf16 CUDA tensors, or
        row-strided views (``src_ld`` elements between sequences).
        """
        if (self.host_lengths >= self.capacity).any():
            raise CapacityError(f"KV cache capacity {self.capacity} exhausted")
        k_new = as_device_tensor(k_new, "k_new", dtype=torch.bfloat16)
        v_new = as_device_tensor(v_new, "v_new", dtype=torch.bfloat16)
        if src_ld is None:
            expect = (self.batch, self.kv_heads, self.head_dim)
            if tuple(k_new.shape) != expect or tuple(v_new.shape) != expect:
                raise ValueError(f"append_step expects shape {expect}")
            k_new, v_new = k_new.contiguous(), v_new.contiguous()
            src_ld = self.kv_heads * self.head_dim
        _lib.call("ps_kv_append", _lib.ptr(self.keys), _lib.ptr(self.values), _lib.ptr(self.lengths),
                  _lib.ptr(k_new), _lib.ptr(v_new), int(src_ld), self.batch, self.kv_heads,
                  self.capacity, self.head_dim, _lib.ptr(self._err), _lib.stream_ptr())
        self.host_lengths += 1

    def append_tokens(self, b: int, k_tokens, v_tokens) -> None:
        """tensors.py:172-192 -- a run of tokens for one sequence (prefill)."""
        k_tokens = as_device_tensor(k_tokens, "k_tokens", dtype=torch.bfloat16, device=self.device)
        v_tokens = as_device_tensor(v_tokens, "v_tokens", dtype=torch.bfloat16, device=self.device)
        t = k_tokens.shape[0]
        if tuple(k_tokens.shape[1:]) != (self.kv_heads, self.head_dim):
            raise ValueError("k_tokens shape mismatch with cache")
        start = int(self.host_lengths[b])
        if start + t > self.capacity:
            raise CapacityError(f"sequence {b}: {start}+{t} tokens exceed capacity {self.capacity}")
        self.keys[b, :, start:start + t] = k_tokens.transpose(0, 1)
        self.values[b, :, start:start + t] = v_tokens.transpose(0, 1)
        self.host_lengths[b] = start + t
        self._sync_lengths()

    def set_lengths(self, lengths) -> None:
        lengths = np.asarray(lengths, dtype=np.int64).reshape(self.batch)
        if (lengths < 0).any() or (lengths > self.capacity).any():
            raise ValueError("lengths out of range")
        self.host_lengths[:] = lengths
        self._sync_lengths()

    def fill_random(self, rng, length: int) -> None:
        """tensors.py:201-213 -- synthetic N(0,1) history.

        ``rng`` may be a numpy Generator (reproduces the reference's exact
        draws, host-side, for parity tests) or a torch.Generator / int seed
        (drawn on the device, for benchmark-sized caches).
        """
        if not 1 <= length <= self.capacity:
            raise ValueError(f"length must be in [1, {self.capacity}]")
        shape = (self.batch, self.kv_heads, length, self.head_dim)
        if isinstance(rng, np.random.Generator):
            k = rng.standard_normal(shape, dtype=np.float32)
            v = rng.standard_normal(shape, dtype=np.float32)
            self.keys[:, :, :length] = torch.from_numpy(k).to(self.device, torch.bfloat16)
            self.values[:, :, :length] = torch.from_numpy(v).to(self.device, torch.bfloat16)
        else:
            gen = rng if isinstance(rng, torch.Generator) else None
            if gen is None:
                gen = torch.Generator(device=self.device)
                gen.manual_seed(int(rng) if rng is not None else 0)
            self.keys[:, :, :length].normal_(generator=gen)
            self.values[:, :, :length].normal_(generator=gen)
        self.host_lengths[:] = length
        self._sync_lengths()

    def check_errors(self) -> None:
        """Raise for a refused device append (reads the error flag: one
        device sync, so eager / debug use)."""
        _raise_append_error(self)

    def keys_for(self, b: int, h: int) -> torch.Tensor:
        return self.keys[b, h, : int(self.host_lengths[b])]

    def values_for(self, b: int, h: int) -> torch.Tensor:
        return self.values[b, h, : int(self.host_lengths[b])]


class PagedKVCache:
    """Block-table KV cache with the ``KVCache`` API.

    The reference cache is one contiguous (B, H_kv, cap, d_h) array
    (tensors.py:116-213).  Here K/V live in page pools of layout
    (pages, H_kv, page_rows, d_h) bf16 and ``block_table`` (B, max_pages)
    int32 maps sequence b's logical rows [j*page_rows, (j+1)*page_rows) to
    a physical page -- the serving format (pages are allocated as sequences
    grow and returned by :meth:`release`).  The SHA kernel streams the same
    32-row tiles through the table (``ps_sha_decode_paged``); ``page_rows``
    must be a multiple of the tile (4096 / head_dim rows).
    """

    def __init__(self, batch: int, kv_heads: int, capacity: int, head_dim: int, page_rows: int = 64,
                 pool_pages: int | None = None, device="cuda", dtype=torch.bfloat16, seed: int | None = None):
        check_count(batch, "batch")
        check_count(kv_heads, "kv_heads")
        check_count(capacity, "capacity")
        check_count(head_dim, "head_dim")
        check_count(page_rows, "page_rows")
        if dtype != torch.bfloat16:
            raise ValueError("the B200 cache stores bf16 K/V")
        tile = max(1, 4096 // head_dim)
        if page_rows % tile:
            raise ValueError(f"page_rows must be a multiple of the SHA tile ({tile} rows at head_dim {head_dim})")
        self.page_rows = page_rows
        self.max_pages = -(-capacity // page_rows)
        pool = pool_pages if pool_pages is not None else batch * self.max_pages
        check_count(pool, "pool_pages")
        shape = (pool, kv_heads, page_rows, head_dim)
        self.k_pool = torch.zeros(shape, dtype=dtype, device=device)
        self.v_pool = torch.zeros(shape, dtype=dtype, device=device)
        self.block_table = torch.full((batch, self.max_pages), -1, dtype=torch.int32, device=device)
        self.host_table = np.full((batch, self.max_pages), -1, dtype=np.int64)
        self.lengths = torch.zeros(batch, dtype=torch.int32, device=device)
        self.host_lengths = np.zeros(batch, dtype=np.int64)
        self._err = torch.zeros(1, dtype=torch.int32, device=device)
        order = np.arange(pool)
        if seed is not None:  # scattered page placement (tests / benchmarks)
            np.random.default_rng(seed).shuffle(order)
        self._free = list(order[::-1])
        self._batch, self._kv_heads, self._head_dim = batch, kv_heads, head_dim

    # KVCache-compatible shape API
    @property
    def batch(self) -> int:
        return self._batch

    @property
    def kv_heads(self) -> int:
        return self._kv_heads

    @property
    def capacity(self) -> int:
        return self.max_pages * self.page_rows

    @property
    def head_dim(self) -> int:
        return self._head_dim

    @property
    def pool_pages(self) -> int:
        return self.k_pool.shape[0]

    @property
    def device(self):
        return self.k_pool.device

    def _sync_lengths(self) -> None:
        self.lengths.copy_(torch.from_numpy(self.host_lengths.astype(np.int32)))

    # ------------------------------------------------------------ page management
    def reserve(self, b: int, rows: int) -> None:
        """Map pages so sequence b can hold ``rows`` rows (host allocator,
        one H2D copy of the changed table row)."""
        need = -(-int(rows) // self.page_rows)
        if need > self.max_pages:
            raise CapacityError(f"sequence {b}: {rows} rows exceed capacity {self.capacity}")
        row = self.host_table[b]
        changed = False
        for j in range(need):
            if row[j] < 0:
                if not self._free:
                    raise CapacityError("KV page pool exhausted")
                row[j] = self._free.pop()
                changed = True
        if changed:  # unmapped pages stay -1 on the device (appends into them are refused)
            self.block_table[b].copy_(torch.from_numpy(row.astype(np.int32)))

    def reserve_all(self) -> None:
        for b in range(self.batch):
            self.reserve(b, self.capacity)

    def release(self, b: int) -> None:
        """Return sequence b's pages to the pool and empty it."""
        row = self.host_table[b]
        self._free.extend(int(p) for p in row[row >= 0][::-1])
        row[:] = -1
        self.block_table[b].fill_(-1)
        self.host_lengths[b] = 0
        self._sync_lengths()

    def _page_rows_of(self, b: int, start: int, stop: int):
        """(page, row-in-page, logical start, logical stop) runs covering [start, stop)."""
        P = self.page_rows
        r = start
        while r < stop:
            j, o = divmod(r, P)
            e = min(stop, (j + 1) * P)
            yield int(self.host_table[b, j]), o, r, e
            r = e

    # ------------------------------------------------------------ KVCache API
    def append_step(self, k_new, v_new, src_ld=None) -> None:
        """tensors.py:150-170 into the page holding each sequence's next row."""
        if (self.host_lengths >= self.capacity).any():
            raise CapacityError(f"KV cache capacity {self.capacity} exhausted")
        # only sequences whose next row opens a page that is not mapped yet
        nxt = self.host_lengths // self.page_rows
        for b in np.nonzero(self.host_table[np.arange(self.batch), nxt] < 0)[0]:
            self.reserve(int(b), int(self.host_lengths[b]) + 1)
        k_new = as_device_tensor(k_new, "k_new", dtype=torch.bfloat16)
        v_new = as_device_tensor(v_new, "v_new", dtype=torch.bfloat16)
        if src_ld is None:
            expect = (self.batch, self.kv_heads, self.head_dim)
            if tuple(k_new.shape) != expect or tuple(v_new.shape) != expect:
                raise ValueError(f"append_step expects shape {expect}")
            k_new, v_new = k_new.contiguous(), v_new.contiguous()
            src_ld = self.kv_heads * self.head_dim
        _lib.call("ps_kv_append_paged", _lib.ptr(self.k_pool), _lib.ptr(self.v_pool), self.page_rows,
                  _lib.ptr(self.block_table), self.max_pages, _lib.ptr(self.lengths), _lib.ptr(k_new),
                  _lib.ptr(v_new), int(src_ld), self.batch, self.kv_heads, self.head_dim, _lib.ptr(self._err),
                  _lib.stream_ptr())
        self.host_lengths += 1

    def append_tokens(self, b: int, k_tokens, v_tokens) -> None:
        """tensors.py:172-192 -- a run of tokens for one sequence (prefill)."""
        k_tokens = as_device_tensor(k_tokens, "k_tokens", dtype=torch.bfloat16, device=self.device)
        v_tokens = as_device_tensor(v_tokens, "v_tokens", dtype=torch.bfloat16, device=self.device)
        t = k_tokens.shape[0]
        if tuple(k_tokens.shape[1:]) != (self.kv_heads, self.head_dim):
            raise ValueError("k_tokens shape mismatch with cache")
        start = int(self.host_lengths[b])
        if start + t > self.capacity:
            raise CapacityError(f"sequence {b}: {start}+{t} tokens exceed capacity {self.capacity}")
        self.reserve(b, start + t)
        for pg, o, r0, r1 in self._page_rows_of(b, start, start + t):
            self.k_pool[pg, :, o:o + r1 - r0] = k_tokens[r0 - start:r1 - start].transpose(0, 1)
            self.v_pool[pg, :, o:o + r1 - r0] = v_tokens[r0 - start:r1 - start].transpose(0, 1)
        self.host_lengths[b] = start + t
        self._sync_lengths()

    def set_lengths(self, lengths) -> None:
        lengths = np.asarray(lengths, dtype=np.int64).reshape(self.batch)
        if (lengths < 0).any() or (lengths > self.capacity).any():
            raise ValueError("lengths out of range")
        for b in range(self.batch):
            self.reserve(b, int(lengths[b]))
        self.host_lengths[:] = lengths
        self._sync_lengths()

    def load_contiguous(self, keys, values, lengths) -> None:
        """Copy (B, H_kv, >= max length, d_h) K/V histories into pages."""
        lengths = np.asarray(lengths, dtype=np.int64).reshape(self.batch)
        for b in range(self.batch):
            n = int(lengths[b])
            if n > self.capacity:
                raise CapacityError(f"sequence {b}: {n} rows exceed capacity {self.capacity}")
            self.reserve(b, n)
            for pg, o, r0, r1 in self._page_rows_of(b, 0, n):
                self.k_pool[pg, :, o:o + r1 - r0] = keys[b, :, r0:r1]
                self.v_pool[pg, :, o:o + r1 - r0] = values[b, :, r0:r1]
        self.host_lengths[:] = lengths
        self._sync_lengths()

    @classmethod
    def from_contiguous(cls, cache: "KVCache", page_rows: int = 64, pool_pages: int | None = None,
                        seed: int | None = None) -> "PagedKVCache":
        out = cls(cache.batch, cache.kv_heads, cache.capacity, cache.head_dim, page_rows=page_rows,
                  pool_pages=pool_pages, device=cache.device, seed=seed)
        out.load_contiguous(cache.keys, cache.values, cache.host_lengths)
        return out

    def fill_random(self, rng, length: int) -> None:
        """tensors.py:201-213 -- same draws as ``KVCache.fill_random``."""
        if not 1 <= length <= self.capacity:
            raise ValueError(f"length must be in [1, {self.capacity}]")
        shape = (self.batch, self.kv_heads, length, self.head_dim)
        if isinstance(rng, np.random.Generator):
            k = torch.from_numpy(rng.standard_normal(shape, dtype=np.float32)).to(self.device, torch.bfloat16)
            v = torch.from_numpy(rng.standard_normal(shape, dtype=np.float32)).to(self.device, torch.bfloat16)
        else:
            gen = rng if isinstance(rng, torch.Generator) else None
            if gen is None:
                gen = torch.Generator(device=self.device)
                gen.manual_seed(int(rng) if rng is not None else 0)
            k = torch.empty(shape, dtype=torch.bfloat16, device=self.device).normal_(generator=gen)
            v = torch.empty(shape, dtype=torch.bfloat16, device=self.device).normal_(generator=gen)
        self.load_contiguous(k, v, np.full(self.batch, length))

    def check_errors(self) -> None:
        """Raise for a refused device append (reads the error flag: one
        device sync, so eager / debug use).  1 = capacity, 2 = unmapped page."""
        _raise_append_error(self)

    def keys_for(self, b: int, h: int) -> torch.Tensor:
        return torch.cat([self.k_pool[pg, h, o:o + r1 - r0]
                          for pg, o, r0, r1 in self._page_rows_of(b, 0, int(self.host_lengths[b]))])

    def values_for(self, b: int, h: int) -> torch.Tensor:
        return torch.cat([self.v_pool[pg, h, o:o + r1 - r0]
                          for pg, o, r0, r1 in self._page_rows_of(b, 0, int(self.host_lengths[b]))])


def l2_norm_per_head(attn_out) -> torch.Tensor:
    """tensors.py:76-80 (study helper; plain torch on device)."""
    a = as_device_tensor(attn_out, "attn_out")
    return torch.linalg.vector_norm(a[:, :, 0, :].double(), dim=-1).float()


def rsqrt_head_dim(d_h: int) -> float:
    return 1.0 / math.sqrt(d_h)
