"""ctypes binding of libpolar_b200.so (the C ABI in include/polar_b200.h).

The product path has no CPU fallback: if the library is missing, or a
tensor is not on a CUDA device, calls raise immediately.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .exceptions import CapacityError, EmptyCacheError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpolar_b200.so")
if os.environ.get("PS_LIB_PATH"):  # experiment variants (tools/build_variant.sh); not the product path
    LIB_PATH = os.environ["PS_LIB_PATH"]

PS_DTYPE_F32 = 0
PS_DTYPE_BF16 = 1
PS_ACT_NONE = 0
PS_ACT_RELU = 1
PS_GG_A_READY = 1
PS_GG_BITMAP = 2

_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_f = ctypes.c_float
_sz = ctypes.c_size_t

# name -> (restype, argtypes); must cover every function in include/polar_b200.h
SIGNATURES = {
    "ps_version": (_i, []),
    "ps_status_string": (ctypes.c_char_p, [_i]),
    "ps_num_sms": (_i, []),
    "ps_debug_sha_mma": (None, [_i]),
    "ps_debug_sha_trace": (None, [_vp]),
    "ps_sha_workspace_bytes": (_sz, [_i, _i, _i, _i, _i, _i]),
    "ps_sha_auto_splits": (_i, [_i, _i, _i, _i, _i]),
    "ps_sha_decode": (_i, [_vp, _i64, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _f, _i, _i,
                           _vp, _i64, _i, _vp, _sz, _vp]),
    "ps_kv_append": (_i, [_vp, _vp, _vp, _vp, _vp, _i64, _i, _i, _i, _i, _vp, _vp]),
    "ps_sha_decode_paged": (_i, [_vp, _i64, _vp, _vp, _i, _i, _vp, _i64, _vp, _vp, _i, _i, _i, _i, _i, _i, _f, _i,
                                 _i, _vp, _i64, _i, _vp, _sz, _vp]),
    "ps_kv_append_paged": (_i, [_vp, _vp, _i, _vp, _i64, _vp, _vp, _vp, _i64, _i, _i, _i, _vp, _vp]),
    "ps_topk_rows": (_i, [_vp, _i, _i, _i64, _i, _vp, _vp, _vp]),
    "ps_threshold_rows": (_i, [_vp, _i, _i, _i64, _f, _vp, _vp]),
    "ps_select_union_workspace_bytes": (_sz, [_i, _i]),
    "ps_select_union": (_i, [_vp, _vp, _i, _i, _i64, _i, _f, _vp, _sz, _i, _i, _i, _vp, _vp, _vp]),
    "ps_select_union_bitmap": (_i, [_vp, _vp, _i, _i, _i64, _i, _f, _vp, _vp, _vp]),
    "ps_union_rows": (_i, [_vp, _i, _i, _i, _vp, _vp]),
    "ps_bitmap_compact": (_i, [_vp, _i, _i, _i, _i, _vp, _vp, _vp]),
    "ps_head_router_topk": (_i, [_vp, _i64, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp]),
    "ps_head_router_topk_append": (_i, [_vp, _i64, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                        _i64, _i, _i, _i, _vp, _vp]),
    "ps_head_router_topk_append_paged": (_i, [_vp, _i64, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp,
                                              _i64, _vp, _vp, _vp, _i64, _i, _i, _vp, _vp]),
    "ps_debug_gemm_trace": (None, [_vp, _i, _i]),
    "ps_debug_gemm_lsu_mode": (None, [_i]),
    "ps_debug_gemm_gemv": (None, [_i]),
    "ps_debug_topk_trace": (None, [_vp]),
    "ps_debug_topk_v2": (None, [_i]),
    "ps_gather_gemm_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "ps_gather_gemm_auto_splits": (_i, [_i, _i, _i]),
    "ps_gather_gemm": (_i, [_vp, _i, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i, _i, _i, _i, _i, _i,
                            _vp, _i64, _i, _vp, _sz, _vp]),
    "ps_gather_gemm_t": (_i, [_vp, _i, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i, _i, _i, _i, _i,
                              _vp, _i64, _i, _vp, _sz, _vp]),
    "ps_sparse_mlp_workspace_bytes": (_sz, [_i, _i, _i]),
    "ps_sparse_mlp": (_i, [_vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp, _i64, _i, _vp, _i64, _vp, _i64, _vp, _sz,
                           _vp]),
    "ps_router_mlp_workspace_bytes": (_sz, [_i, _i, _i]),
    "ps_router_mlp": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _i64, _i, _vp, _i64, _vp, _i64, _vp, _sz, _vp]),
    "ps_router_mlp_fused_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "ps_router_mlp_fused": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _i64, _i, _vp, _i64, _vp, _i64, _vp, _sz,
                                 _vp]),
    "ps_debug_router_trace": (None, [_vp]),
    "ps_allreduce_add_bf16": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _i64, _vp]),
    "ps_debug_chain_stages": (None, [_i]),
    "ps_debug_chain_trace": (None, [_vp]),
    "ps_set_pdl": (None, [_i]),
    "ps_layernorm": (_i, [_vp, _i64, _vp, _vp, _i, _i, _vp, _i64, _vp]),
    "ps_add_layernorm": (_i, [_vp, _i64, _vp, _vp, _vp, _i, _i, _vp, _i64, _vp]),
    "ps_embed": (_i, [_vp, _vp, _vp, _vp, _i, _i, _vp, _vp]),
    "ps_swiglu": (_i, [_vp, _i64, _i, _i, _vp, _i64, _vp]),
}

_LIB = None


def load():
    """Load the shared library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2505_14884_b200._build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        variant = "PS_LIB_PATH" in os.environ  # an older experiment build may lack newer entry points
        for name, (res, args) in SIGNATURES.items():
            if variant and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def check(status: int, what: str) -> None:
    """Map a PS_ERR_* status onto the reference's exception types."""
    if status == 0:
        return
    msg = f"{what}: {load().ps_status_string(status).decode()}"
    if status == 2:
        raise IndexError(msg)
    if status == 3:
        raise EmptyCacheError(msg)
    if status == 4:
        raise CapacityError(msg)
    if status == 7:
        raise RuntimeError(msg)
    raise ValueError(msg)


def ptr(t):
    """Raw device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"expected a torch tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise ValueError("libpolar_b200 operates on CUDA tensors only (no CPU fallback)")
    return t.data_ptr()


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
