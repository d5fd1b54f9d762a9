"""CPU-side tests: the C ABI library loads and exports every symbol declared
in include/polar_b200.h (no compute calls without a GPU), the ctypes
signatures cover the header, and host-side logic (policy rules, error
mapping, validation) behaves like the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "polar_b200.h")
LIB = os.path.join(ROOT, "paper_2505_14884_b200", "libpolar_b200.so")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2505_14884_b200 import _build

        _build.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_hot_path():
    fns = header_functions()
    for name in ("ps_sha_decode", "ps_topk_rows", "ps_select_union", "ps_bitmap_compact", "ps_head_router_topk",
                 "ps_gather_gemm", "ps_gather_gemm_t", "ps_kv_append"):
        assert name in fns


def test_library_exports_every_header_symbol(lib):
    for name in header_functions():
        assert hasattr(lib, name), f"{name} declared in polar_b200.h but not exported"


def test_ctypes_signatures_cover_header():
    from paper_2505_14884_b200 import _lib

    assert set(header_functions()) <= set(_lib.SIGNATURES)


def test_status_strings_and_pure_queries(lib):
    lib.ps_status_string.restype = ctypes.c_char_p
    assert lib.ps_status_string(0) == b"ok"
    assert b"capacity" in lib.ps_status_string(4)
    lib.ps_sha_workspace_bytes.restype = ctypes.c_size_t
    n1 = lib.ps_sha_workspace_bytes(64, 32, 32, 128, 16, 1)
    n4 = lib.ps_sha_workspace_bytes(64, 32, 32, 128, 16, 4)
    assert n4 > n1 > 0
    assert lib.ps_version() >= 1


def test_host_side_argument_errors(lib):
    """Invalid arguments are rejected before any launch (no GPU needed)."""
    nullp = ctypes.c_void_p(0)
    assert lib.ps_topk_rows(nullp, 0, 10, ctypes.c_int64(10), 1, nullp, nullp, nullp) == 1
    assert lib.ps_bitmap_compact(nullp, 64, 3, 64, 128, nullp, nullp, nullp) == 1
    assert lib.ps_head_router_topk(nullp, ctypes.c_int64(8), nullp, nullp, 1, 7, 8, 2, nullp, nullp, nullp) == 1
    # the union hand-off: no bitmap, k > cols, the bitmap aliasing the buffer it clears
    f = ctypes.c_float(0.0)
    p1, p2 = ctypes.c_void_p(64), ctypes.c_void_p(4096)
    assert lib.ps_select_union_bitmap(p1, nullp, 2, 64, ctypes.c_int64(64), 8, f, nullp, nullp, nullp) == 1
    assert lib.ps_select_union_bitmap(p1, nullp, 2, 64, ctypes.c_int64(64), 65, f, p2, nullp, nullp) == 1
    assert lib.ps_select_union_bitmap(p1, nullp, 2, 64, ctypes.c_int64(64), 8, f, p2, p2, nullp) == 1
    assert lib.ps_select_union_bitmap(p1, nullp, 2, 40000, ctypes.c_int64(40000), 8, f, p2, nullp, nullp) == 5
    # fused router: batches beyond its shared memory have no workspace size
    lib.ps_router_mlp_fused_workspace_bytes.restype = ctypes.c_size_t
    assert lib.ps_router_mlp_fused_workspace_bytes(129, 4096, 1024, 16384) == 0
    # allreduce: world out of range, rank outside the world
    assert lib.ps_allreduce_add_bf16(p2, p2, p2, p2, 0, 9, 1, 8, p2, ctypes.c_int64(8), nullp) == 1
    assert lib.ps_allreduce_add_bf16(p2, p2, p2, p2, 2, 2, 1, 8, p2, ctypes.c_int64(8), nullp) == 1


def test_status_to_exception_mapping():
    from paper_2505_14884_b200 import CapacityError, EmptyCacheError, _lib

    with pytest.raises(IndexError):
        _lib.check(2, "x")
    with pytest.raises(EmptyCacheError):
        _lib.check(3, "x")
    with pytest.raises(CapacityError):
        _lib.check(4, "x")
    with pytest.raises(ValueError):
        _lib.check(1, "x")
    with pytest.raises(RuntimeError):
        _lib.check(7, "x")
    assert issubclass(EmptyCacheError, ValueError) and issubclass(CapacityError, RuntimeError)


def test_policy_rules_match_reference():
    """engine.py:42-77: budget, layer-0 rule, sparse-MLP eligibility."""
    from oracle import polar_oracle as po
    from paper_2505_14884_b200.engine import SparsityPolicy
    from paper_2505_14884_b200.model import SHAPES

    for rho in (0.3, 0.5, 0.625, 1.0, 0.01):
        for n in (8, 32, 72):
            assert SparsityPolicy(mode="polar", head_density=rho).head_budget(n) == po.head_budget(rho, n)
    assert SparsityPolicy(mode="polar", head_density=0.3).head_budget(72) == 22
    p = SparsityPolicy(mode="polar", head_density=0.5)
    assert not p.wants_sparse_heads(0) and p.wants_sparse_heads(1)
    assert SparsityPolicy(mode="polar", head_density=0.5, layer0_dense_attention=False).wants_sparse_heads(0)
    assert not SparsityPolicy(mode="dejavu_mlp", head_density=0.5).wants_sparse_heads(3)
    assert not SparsityPolicy(mode="polar", head_density=1.0).wants_sparse_heads(3)
    assert not p.wants_sparse_mlp(SHAPES["opt-6.7b"])  # no k table
    p2 = SparsityPolicy(mode="polar", head_density=0.5, mlp_k_table={0: 10})
    assert p2.wants_sparse_mlp(SHAPES["opt-6.7b"]) and not p2.wants_sparse_mlp(SHAPES["llama-3.1-8b"])
    with pytest.raises(ValueError):
        SparsityPolicy(mode="bogus")
    with pytest.raises(ValueError):
        SparsityPolicy(head_density=0.0)


def test_batch_head_index_validation_matches_reference():
    from paper_2505_14884_b200 import kernels as pk

    with pytest.raises(ValueError):
        pk.BatchHeadIndex.__init__(object.__new__(pk.BatchHeadIndex), np.array([[1, 1]]))
    with pytest.raises(IndexError):
        pk.BatchHeadIndex.__init__(object.__new__(pk.BatchHeadIndex), np.array([[-1, 0]]))
    with pytest.raises(ValueError):
        pk.BatchHeadIndex.__init__(object.__new__(pk.BatchHeadIndex), np.zeros((0, 2), np.int64))
    with pytest.raises(ValueError):
        pk.BatchHeadIndex.__init__(object.__new__(pk.BatchHeadIndex), np.array([1, 2]))


def test_model_shapes():
    from paper_2505_14884_b200.model import SHAPES

    opt = SHAPES["opt-6.7b"]
    assert (opt.head_dim, opt.group_size, opt.kv_dim) == (128, 1, 4096)
    llama = SHAPES["llama-3.1-8b"]
    assert (llama.head_dim, llama.group_size, llama.activation) == (128, 4, "swiglu")
    assert SHAPES["opt-66b"].heads == 72 and SHAPES["llama-3.1-70b"].kv_heads == 8


def test_no_cpu_fallback_on_cpu_tensors():
    import torch

    from paper_2505_14884_b200 import _lib

    with pytest.raises(ValueError, match="CUDA"):
        _lib.ptr(torch.zeros(4))
