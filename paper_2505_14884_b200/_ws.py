"""Device workspace pool.

The C ABI never allocates.  Kernels that merge split partials keep
self-resetting tickets in their workspace, so each workspace is zero-filled
once when created and then reused; buffers only grow.  Allocate (and warm)
before CUDA-graph capture -- a capture never allocates here because the
engine sizes everything up front.
"""

from __future__ import annotations

import torch

_POOL: dict = {}


def get(tag: str, nbytes: int, device) -> torch.Tensor:
    """Zero-initialised uint8 buffer of at least ``nbytes`` for ``tag``."""
    dev = torch.device(device)
    key = (tag, dev)
    buf = _POOL.get(key)
    if buf is None or buf.numel() < nbytes:
        if torch.cuda.is_current_stream_capturing():
            raise RuntimeError(f"workspace {tag!r} must be sized before CUDA-graph capture")
        buf = torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
        _POOL[key] = buf
    return buf


def clear() -> None:
    _POOL.clear()
