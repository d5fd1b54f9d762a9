"""Device workspace pools.

The C ABI never allocates.  Kernels that merge split partials keep
self-resetting tickets in their workspace, so each workspace is zero-filled
once when created and then reused.  Allocate (and warm) before CUDA-graph
capture -- a capture never allocates here because the engine sizes
everything up front.

A CUDA graph keeps the raw pointers of the workspaces its kernels used, so
a pool never frees a buffer it has handed out: when a tag needs more bytes,
the old buffer is retired (kept alive for the pool's lifetime) and a larger
one takes its place.  Each :class:`~.engine.DecodeEngine` owns its own pool
(``with using(engine.ws): ...`` around its launches), so two engines never
share tickets or partials; eager public API calls use the module's default
pool.
"""

from __future__ import annotations

import contextlib

import torch


class Pool:
    """Tag -> zero-initialised uint8 device buffer; buffers only grow and
    are never released while the pool lives."""

    def __init__(self):
        self._bufs: dict = {}
        self._retired: list = []

    def get(self, tag: str, nbytes: int, device) -> torch.Tensor:
        dev = torch.device(device)
        key = (tag, dev)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError(f"workspace {tag!r} must be sized before CUDA-graph capture")
            if buf is not None:
                self._retired.append(buf)  # a captured graph may still point at it
            buf = torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
            self._bufs[key] = buf
        return buf

    def nbytes(self) -> int:
        return sum(b.numel() for b in self._bufs.values()) + sum(b.numel() for b in self._retired)


_DEFAULT = Pool()
_STACK: list = [_DEFAULT]


@contextlib.contextmanager
def using(pool: Pool):
    """Route every ``get`` inside the block to ``pool``."""
    _STACK.append(pool)
    try:
        yield pool
    finally:
        _STACK.pop()


def get(tag: str, nbytes: int, device) -> torch.Tensor:
    """Zero-initialised uint8 buffer of at least ``nbytes`` for ``tag`` from
    the current pool."""
    return _STACK[-1].get(tag, nbytes, device)


def default_pool() -> Pool:
    return _DEFAULT
