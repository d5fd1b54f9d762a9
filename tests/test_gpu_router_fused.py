"""The one-launch MLP router (ps_router_mlp_fused, routers.py:286-288):
hid = relu(x W_in + b_in) in bf16 and logits = hid W_out + b_out in f32,
against an f64 torch reference; repeated launches and CUDA-graph replays (the
self-resetting grid barrier); shapes it does not cover report False."""

import pytest

torch = pytest.importorskip("torch")

from paper_2505_14884_b200 import MlpRouter  # noqa: E402

pytestmark = pytest.mark.gpu


def _router(d, D, h, seed=3):
    r = MlpRouter(d, D, hidden_dim=h, seed=seed)
    g = torch.Generator(device="cuda").manual_seed(seed)
    r.b_in = torch.randn(h, device="cuda", generator=g) * 0.1
    r.b_out = torch.randn(D, device="cuda", generator=g) * 0.1
    return r


def _check(r, x, hid, lg, with_bias=True):
    hh = torch.relu(x.double() @ r.w_in_t.double().t() + r.b_in.double())
    # hidden: bf16 rounding of an f32 split-K sum
    assert float((hid.double() - hh).abs().max()) <= 1e-2 * max(1.0, float(hh.abs().max()))
    ref = hid.double() @ r.w_out_t.double().t() + (r.b_out.double() if with_bias else 0.0)
    assert float((lg.double() - ref).abs().max()) <= 1e-3 * max(1.0, float(ref.abs().max()))


@pytest.mark.parametrize("B,d,h,D", [(64, 4096, 1024, 16384), (1, 4096, 1024, 16384), (16, 4096, 1024, 16384),
                                     (128, 4096, 1024, 16384), (8, 256, 1024, 1024), (33, 512, 256, 3000)])
def test_router_fused_matches_f64(B, d, h, D):
    r = _router(d, D, h)
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(B, d, device="cuda", generator=g).bfloat16()
    hid = torch.full((B, h), float("nan"), dtype=torch.bfloat16, device="cuda")
    lg = torch.full((B, D), float("nan"), device="cuda")
    assert r.fused_bytes(B) > 0
    for _ in range(3):  # the grid barrier word and partials are reused launch to launch
        assert r.fused_into(x, hid, lg)
        torch.cuda.synchronize()
        _check(r, x, hid, lg)
    lg2 = torch.empty_like(lg)
    assert r.fused_into(x, hid, lg2, with_bias=False)
    torch.cuda.synchronize()
    _check(r, x, hid, lg2, with_bias=False)


def test_router_fused_graph_replay_tracks_inputs():
    B, d, h, D = 64, 4096, 1024, 16384
    rs = [_router(d, D, h, seed=s) for s in (5, 6)]
    x = torch.zeros(B, d, dtype=torch.bfloat16, device="cuda")
    hid = torch.empty(B, h, dtype=torch.bfloat16, device="cuda")
    lgs = [torch.empty(B, D, device="cuda") for _ in rs]
    for r, lg in zip(rs, lgs):
        r.fused_into(x, hid, lg)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(gr, stream=st):
        for r, lg in zip(rs, lgs):  # two layers back to back share the workspace
            r.fused_into(x, hid, lg)
    torch.cuda.current_stream().wait_stream(st)
    g = torch.Generator(device="cuda").manual_seed(2)
    for _ in range(4):
        x.copy_(torch.randn(B, d, device="cuda", generator=g).bfloat16())
        gr.replay()
        torch.cuda.synchronize()
        r = rs[1]
        hh = torch.relu(x.double() @ r.w_in_t.double().t() + r.b_in.double())
        assert float((hid.double() - hh).abs().max()) <= 1e-2 * max(1.0, float(hh.abs().max()))
        _check(r, x, hid, lgs[1])


def test_router_fused_unsupported_shapes_fall_back():
    r = _router(4096, 16384, 1024)
    x = torch.zeros(300, 4096, dtype=torch.bfloat16, device="cuda")
    hid = torch.empty(300, 1024, dtype=torch.bfloat16, device="cuda")
    lg = torch.empty(300, 16384, device="cuda")
    assert r.fused_bytes(300) == 0
    assert r.fused_into(x, hid, lg) is False
    wide = _router(9216, 36864, 1024)  # OPT-66B: W_in slices of > 4 K-blocks, > 148 tiles
    assert wide.fused_bytes(64) == 0


@pytest.mark.parametrize("B", [129, 256])
def test_router_fused_declines_large_batches(B):
    """B > 128 does not fit the kernel's shared memory: no workspace size,
    PS_ERR_UNSUPPORTED from the entry point, fused_into returns False (the
    engine then runs the two GEMMs)."""
    from paper_2505_14884_b200 import _lib

    r = _router(4096, 16384, 1024)
    assert r.fused_bytes(B) == 0
    assert _lib.load().ps_router_mlp_fused_workspace_bytes(B, 4096, 1024, 16384) == 0
    x = torch.zeros(B, 4096, device="cuda").bfloat16()
    hid = torch.zeros(B, 1024, dtype=torch.bfloat16, device="cuda")
    lg = torch.zeros(B, 16384, device="cuda")
    assert r.fused_into(x, hid, lg) is False
