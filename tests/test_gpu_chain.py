"""The one-launch chained GEMMs (csrc/chain_gemm.cu): ps_sparse_mlp (the
selective MLP, kernels.py:353-373) and ps_router_mlp (routers.py:286-288),
against an f64 torch restatement over the same bf16 operands.

Tolerance (bf16 operands, f32 accumulation, hidden rounded to bf16 like the
reference's two-launch path): max|d| <= 2e-2 * max(1, max|ref|), rel-L2 <= 1e-2.
Also: repeats agree to f32 rounding (split tiles are summed with f32
reductions in arrival order), CUDA-graph replays (epoch flags,
self-resetting tickets and accumulators), an empty union, the dense (no ids)
form, ragged d / D, and batch 1..256."""

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2505_14884_b200.kernels import PackedMLP, ROW_PAD, _round_up, sparse_mlp_into  # noqa: E402
from paper_2505_14884_b200 import MlpRouter  # noqa: E402


def _mlp_case(B, d, D, k, seed=0, dense=False):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(seed)
    w1 = (torch.randn(D, d, device=dev, generator=g) * 0.05).bfloat16()
    w2 = (torch.randn(D, d, device=dev, generator=g) * 0.05).bfloat16()
    b1 = torch.randn(D, device=dev, generator=g) * 0.05
    b2 = torch.randn(d, device=dev, generator=g) * 0.05
    x = torch.randn(B, d, device=dev, generator=g).bfloat16()
    res = torch.randn(B, d, device=dev, generator=g)
    pk = PackedMLP(w1, b1, w2, b2)
    Dp = _round_up(D, ROW_PAD)
    if dense:
        ids = torch.arange(D, device=dev, dtype=torch.int32)
        idx = cnt = None
    else:
        ids = torch.randperm(D, device=dev, generator=g)[:k].sort().values.int()
        idx = torch.full((Dp,), int(ids[-1]) if k else 0, dtype=torch.int32, device=dev)
        idx[:k] = ids
        cnt = torch.tensor([k], dtype=torch.int32, device=dev)
    il = ids.long()
    h = torch.relu(x.double() @ w1[il].double().t() + b1[il].double())
    ref_h = h.bfloat16().double()
    ref = ref_h @ w2[il].double() + b2.double() + res.double()
    return pk, x, idx, cnt, res, ref, h, Dp


def _check(got, ref):
    got = got.double()
    scale = max(1.0, float(ref.abs().max()))
    assert float((got - ref).abs().max()) <= 2e-2 * scale
    assert float((got - ref).norm() / max(ref.norm(), 1e-30)) <= 1e-2


@pytest.mark.parametrize("B,d,D,k", [(8, 256, 1024, 300), (1, 4096, 16384, 1638), (16, 4096, 16384, 4000),
                                     (64, 4096, 16384, 6543), (128, 4096, 16384, 8600), (256, 1024, 4096, 2000),
                                     (5, 200, 520, 77), (64, 4096, 16384, 16384), (3, 256, 1024, 1)])
def test_sparse_mlp_matches_f64(B, d, D, k):
    pk, x, idx, cnt, res, ref, h, Dp = _mlp_case(B, d, D, k)
    hidden = torch.full((B, Dp), float("nan"), dtype=torch.bfloat16, device="cuda")
    out = res.clone()
    sparse_mlp_into(pk, x, idx, cnt, hidden, out, residual=out)
    torch.cuda.synchronize()
    _check(out, ref)
    # hidden: the union columns (bf16), then zeros up to the next 128
    kk = h.shape[1]
    assert float((hidden[:, :kk].double() - h).abs().max()) <= 1e-2 * max(1.0, float(h.abs().max()))
    assert bool((hidden[:, kk:_round_up(kk, 128)] == 0).all())


def test_sparse_mlp_dense_form():
    pk, x, idx, cnt, res, ref, h, Dp = _mlp_case(32, 512, 2048, 0, dense=True)
    hidden = torch.zeros((32, Dp), dtype=torch.bfloat16, device="cuda")
    out = res.clone()
    sparse_mlp_into(pk, x, None, None, hidden, out, residual=out)
    torch.cuda.synchronize()
    _check(out, ref)


def test_sparse_mlp_empty_union():
    pk, x, idx, cnt, res, ref, h, Dp = _mlp_case(8, 256, 1024, 10)
    cnt.zero_()
    hidden = torch.zeros((8, Dp), dtype=torch.bfloat16, device="cuda")
    out = torch.empty(8, 256, device="cuda")
    sparse_mlp_into(pk, x, idx, cnt, hidden, out, residual=res)
    torch.cuda.synchronize()
    assert torch.allclose(out, res + pk.b2)


def test_sparse_mlp_repeats_and_residual_copy():
    pk, x, idx, cnt, res, ref, h, Dp = _mlp_case(64, 4096, 16384, 6543, seed=3)
    hidden = torch.zeros((64, Dp), dtype=torch.bfloat16, device="cuda")
    outs = []
    for _ in range(3):
        o = torch.empty(64, 4096, device="cuda")
        sparse_mlp_into(pk, x, idx, cnt, hidden, o, residual=res)
        outs.append(o)
    torch.cuda.synchronize()
    _check(outs[0], ref)
    for o in outs[1:]:
        assert float((o - outs[0]).abs().max()) <= 1e-4 * max(1.0, float(ref.abs().max()))


def test_sparse_mlp_graph_replays_changing_union():
    """Captured once, replayed with a different union each time (the count and
    ids live on the device): epochs / tickets must carry across replays."""
    B, d, D = 64, 1024, 4096
    pk, x, idx, cnt, res, _, _, Dp = _mlp_case(B, d, D, 1000, seed=5)
    hidden = torch.zeros((B, Dp), dtype=torch.bfloat16, device="cuda")
    out = torch.empty(B, d, device="cuda")
    sparse_mlp_into(pk, x, idx, cnt, hidden, out, residual=res)  # warm / size the workspace
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            for _ in range(3):  # three chained launches in one graph
                sparse_mlp_into(pk, x, idx, cnt, hidden, out, residual=res)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.Generator(device="cuda").manual_seed(11)
    for k in (1000, 37, 4096, 129, 2500):
        ids = torch.randperm(D, device="cuda", generator=g)[:k].sort().values.int()
        idx.fill_(int(ids[-1]))
        idx[:k] = ids
        cnt.fill_(k)
        gr.replay()
        torch.cuda.synchronize()
        il = ids.long()
        hh = torch.relu(x.double() @ pk.w1t[il].double().t() + pk.b1[il].double()).bfloat16().double()
        _check(out, hh @ pk.w2t[il].double() + pk.b2.double() + res.double())


@pytest.mark.parametrize("B,d,h,D", [(64, 4096, 1024, 16384), (1, 4096, 1024, 16384), (8, 256, 1024, 1024),
                                     (200, 512, 128, 3000)])
def test_router_mlp_matches_f64(B, d, h, D):
    r = MlpRouter(d, D, hidden_dim=h, seed=3)
    g = torch.Generator(device="cuda").manual_seed(1)
    r.b_in = torch.randn(h, device="cuda", generator=g) * 0.1
    r.b_out = torch.randn(D, device="cuda", generator=g) * 0.1
    x = torch.randn(B, d, device="cuda", generator=g).bfloat16()
    hid = torch.empty(B, h, dtype=torch.bfloat16, device="cuda")
    lg = torch.empty(B, D, device="cuda")
    r.logits_into(x, hid, lg, fused=True)
    torch.cuda.synchronize()
    hh = torch.relu(x.double() @ r.w_in_t.double().t() + r.b_in.double())
    assert float((hid.double() - hh).abs().max()) <= 1e-2 * max(1.0, float(hh.abs().max()))
    ref = hid.double() @ r.w_out_t.double().t() + r.b_out.double()  # from the kernel's own bf16 hidden
    assert float((lg.double() - ref).abs().max()) <= 1e-3 * max(1.0, float(ref.abs().max()))
    # the two-launch path agrees (its split-K sums in another order, so the
    # bf16 hidden can differ in the last place)
    lg2 = torch.empty_like(lg)
    hid2 = torch.empty_like(hid)
    r.logits_into(x, hid2, lg2, fused=False)
    torch.cuda.synchronize()
    assert float((hid.double() - hid2.double()).abs().max()) <= 1e-2 * max(1.0, float(hh.abs().max()))
    assert float((lg.double() - lg2.double()).norm() / ref.norm()) <= 1e-2
