"""Boundary validation (mirrors sparsedecode/validation.py:13-104).

Host-visible metadata is checked once at the public API; device-resident
index validation (ranges, duplicates) costs a device->host sync and is
opt-in (``validate=True``), used when ids come from the host.
"""

from __future__ import annotations

import numpy as np
import torch


def check_count(value: int, name: str, minimum: int = 1, upper: int | None = None) -> int:
    value = int(value)
    if value < minimum:
        raise ValueError(f"{name} must be >= {minimum}, got {value}")
    if upper is not None and value > upper:
        raise ValueError(f"{name} must be <= {upper}, got {value}")
    return value


def check_choice(value: str, options: tuple, name: str) -> str:
    if value not in options:
        raise ValueError(f"{name} must be one of {options}, got {value!r}")
    return value


def default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2505_14884_b200 needs a CUDA device (sm_100a); no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def as_device_tensor(x, name: str, dtype=None, device=None, ndim: int | None = None) -> torch.Tensor:
    """Return ``x`` as a CUDA tensor (numpy / lists are uploaded)."""
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.to(device or default_device())
    else:
        arr = np.asarray(x)
        if arr.dtype == np.float64:
            arr = arr.astype(np.float32)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(device or default_device())
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if ndim is not None and t.ndim != ndim:
        raise ValueError(f"{name} must be {ndim}-dimensional, got shape {tuple(t.shape)}")
    return t


def as_index_tensor(x, name: str, upper: int | None = None, device=None, validate: bool = True) -> torch.Tensor:
    """1-D int32 device index vector; bounds checked when ``validate``."""
    t = as_device_tensor(x, name, device=device)
    if t.ndim != 1:
        raise ValueError(f"{name} must be 1-dimensional, got shape {tuple(t.shape)}")
    if t.numel() and t.dtype.is_floating_point:
        raise ValueError(f"{name} must hold integers, got dtype {t.dtype}")
    t = t.to(torch.int32)
    if validate and t.numel():
        lo, hi = int(t.min()), int(t.max())
        if lo < 0:
            raise IndexError(f"{name} contains negative indices")
        if upper is not None and hi >= upper:
            raise IndexError(f"{name} contains indices >= {upper}")
    return t
