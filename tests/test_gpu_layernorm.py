"""LayerNorm glue (ps_layernorm / ps_add_layernorm, model.layernorm
model.py:168-175): bf16 output against an fp64 torch LayerNorm (within one
bf16 ulp), the pending bias written back into x, at the model widths and
batch sizes the engine runs."""

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

DEV = torch.device("cuda")


@pytest.mark.parametrize("B,d", [(1, 4096), (3, 4096), (64, 4096), (256, 4096), (64, 8192), (64, 9216), (5, 1024),
                                 (2, 16384)])
@pytest.mark.parametrize("with_add", [False, True])
def test_layernorm_matches_torch(B, d, with_add):
    from paper_2505_14884_b200 import _lib

    gen = torch.Generator(device=DEV).manual_seed(B * 7 + d)
    x0 = torch.randn(B, d, device=DEV, generator=gen) * 3 + 0.5
    g = torch.rand(d, device=DEV, generator=gen) + 0.5
    b = torch.randn(d, device=DEV, generator=gen) * 0.1
    add = torch.randn(d, device=DEV, generator=gen) if with_add else None
    xs = x0 + add if with_add else x0
    ref = torch.nn.functional.layer_norm(xs.double(), (d,), g.double(), b.double(), eps=1e-5)
    x = x0.clone()
    y = torch.full((B, d), float("nan"), device=DEV).bfloat16()
    if add is None:
        _lib.call("ps_layernorm", _lib.ptr(x), x.stride(0), _lib.ptr(g), _lib.ptr(b), B, d, _lib.ptr(y),
                  y.stride(0), _lib.stream_ptr())
    else:
        _lib.call("ps_add_layernorm", _lib.ptr(x), x.stride(0), _lib.ptr(add), _lib.ptr(g), _lib.ptr(b), B, d,
                  _lib.ptr(y), y.stride(0), _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all()
    err = (y.double() - ref).abs()
    assert (err <= ref.abs() * 2 ** -8 + 1e-3).all(), float(err.max())
    assert torch.equal(x, xs)  # the pending bias is written back (x unchanged without one)


def test_layernorm_rejects_bad_arguments():
    from paper_2505_14884_b200 import _lib

    L = _lib.load()
    x = torch.zeros(2, 64, device=DEV)
    g = torch.ones(64, device=DEV)
    y = torch.zeros(2, 64, device=DEV).bfloat16()
    st = _lib.stream_ptr()
    assert L.ps_layernorm(_lib.ptr(x), 64, _lib.ptr(g), _lib.ptr(g), 2, 62, _lib.ptr(y), 64, st) == 1  # PS_ERR_VALUE
    assert L.ps_layernorm(_lib.ptr(x), 32, _lib.ptr(g), _lib.ptr(g), 2, 64, _lib.ptr(y), 64, st) == 1  # PS_ERR_VALUE
    assert L.ps_layernorm(None, 64, _lib.ptr(g), _lib.ptr(g), 2, 64, _lib.ptr(y), 64, st) == 1  # PS_ERR_VALUE
