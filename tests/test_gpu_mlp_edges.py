"""Selective MLP through the device-count path (kernels.mlp_into: ps_gather_gemm
UP + ps_gather_gemm_t DOWN, the union size read on the device as in the
captured decode step) at the edges of the union size: empty (a threshold
router that selects nothing: the block reduces to residual + b2), one
neuron, tile boundaries 127/128/129, and every neuron -- for the GEMV
(B <= 4) and tcgen05 (B > 4) UP paths, against an fp64 torch reference of
kernels.py:353-373 (bf16 hidden activations, like the reference)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

DEV = torch.device("cuda")


@pytest.mark.parametrize("B", [1, 3, 8, 64])
@pytest.mark.parametrize("count", [0, 1, 127, 128, 129, 4096])
def test_mlp_device_count_edges(B, count):
    import paper_2505_14884_b200 as pb
    from paper_2505_14884_b200 import kernels as pk

    d, D = 1024, 4096
    gen = torch.Generator(device=DEV).manual_seed(B * 131 + count)
    w1 = (torch.randn(d, D, device=DEV, generator=gen) * 0.03).bfloat16().float()
    w2 = (torch.randn(d, D, device=DEV, generator=gen) * 0.03).bfloat16().float()
    b1 = torch.randn(D, device=DEV, generator=gen) * 0.05
    b2 = torch.randn(d, device=DEV, generator=gen) * 0.05
    packed = pb.PackedMLP.from_reference(w1, b1, w2, b2)
    x = torch.randn(B, d, device=DEV, generator=gen).bfloat16()
    res = torch.randn(B, d, device=DEV, generator=gen)
    rng = np.random.default_rng(count + 7)
    sel = np.sort(rng.choice(D, count, replace=False)).astype(np.int32)
    idx = torch.full((packed.D_pad,), 0, dtype=torch.int32, device=DEV)
    idx[:count] = torch.from_numpy(sel).to(DEV)
    cnt = torch.tensor([count], dtype=torch.int32, device=DEV)
    hidden = torch.full((B, packed.D_pad), float("nan"), device=DEV).bfloat16()
    out = res.clone()
    pk.mlp_into(packed, x, idx, cnt, hidden, out, residual=out)
    torch.cuda.synchronize()
    it = torch.from_numpy(sel.astype(np.int64)).to(DEV)
    h = torch.relu(x.double() @ w1[:, it].double() + b1[it].double())
    ref = res.double() + b2.double() + h.bfloat16().double() @ w2[:, it].double().T
    got = out.double()
    assert torch.isfinite(got).all()
    if count == 0:
        assert torch.allclose(got, ref, rtol=0, atol=1e-6)
    else:
        err = (got - ref).abs().max().item()
        assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err
