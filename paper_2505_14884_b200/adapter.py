"""Rebind a reference-shaped engine module onto the B200 kernels.

The reference's decode step (``sparsedecode.engine.decode_step``,
engine.py:314-392) looks its kernels up as module globals bound in
engine.py:25-35; rebinding them is the reference's own injection point
(tests/test_engine.py:55-64).  :func:`install` swaps those globals for
wrappers that run this package's CUDA path and hand numpy back, so the
unmodified reference engine decodes on the GPU.  Every call copies numpy <->
device: this is a PARITY adapter, never a timed path (the production path is
``engine.DecodeEngine``).
"""

from __future__ import annotations

import numpy as np

from . import kernels as _k
from . import tensors as _t

# names decode_step resolves at call time (engine.py:25-35)
NAMES = ("gqa_selective_attention_decode", "sparse_mlp_forward", "topk_indices_rows", "union_neuron_indices")


def _np(t):
    return t.float().cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


def gqa_selective_attention_decode(q, cache, group_index, params=None, scale=None, variant="running"):
    gc = cache if isinstance(cache, _t.KVCache) else _t.KVCache.from_reference(cache)
    rows = getattr(group_index, "entries", group_index)
    bhi = _k.BatchHeadIndex(np.asarray(_np(rows)).astype(np.int64))
    if not isinstance(params, _k.FlashBlockParams):  # a CPU block size: no meaning on the GPU kernel
        params = _k.FlashBlockParams()
    return _np(_k.gqa_selective_attention_decode(q, gc, bhi, params, scale, variant))


def sparse_mlp_forward(x, w1, b1, w2, b2, active):
    idx = getattr(active, "indices", active)
    return _np(_k.sparse_mlp_forward(x, w1, b1, w2, b2, np.asarray(_np(idx)).astype(np.int64)))


def topk_indices_rows(scores, k):
    return _t.topk_indices_rows(scores, k).cpu().numpy().astype(np.int64)


def union_neuron_indices(per_sequence_sets, layer=0):
    u = _k.union_neuron_indices([np.asarray(s) for s in per_sequence_sets], layer)
    return u.indices.cpu().numpy().astype(np.int64)


def install(engine_module) -> dict:
    """Rebind ``engine_module``'s kernel globals; returns the originals so
    :func:`uninstall` can restore them."""
    saved = {}
    for name in NAMES:
        if hasattr(engine_module, name):
            saved[name] = getattr(engine_module, name)
            setattr(engine_module, name, globals()[name])
    return saved


def uninstall(engine_module, saved: dict) -> None:
    for name, fn in saved.items():
        setattr(engine_module, name, fn)
