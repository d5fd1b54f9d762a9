"""Union hand-off (ps_select_union_bitmap + PS_GG_BITMAP, SURVEY.md §8 rows
a10-a13): the selection kernel only ORs the rows' top-k / threshold sets into
a bitmap and the UP / DOWN GEMMs derive the union ids on the device.  The
results must be bit-identical to the compacted-id path (same ids in the same
order, same summation order), the union size written by UP must equal the
compaction's count, the alternate buffer must be cleared, and the engine's
decode steps must not change with the hand-off on."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

DEV = torch.device("cuda")


@pytest.mark.parametrize("B,D,k,mode", [(8, 4096, 400, "topk"), (64, 16384, 1638, "topk"), (64, 16384, 0, "thr"),
                                        (17, 2048, 2048, "topk"), (128, 16384, 1638, "hot")])
def test_bitmap_handoff_matches_compacted_ids(B, D, k, mode):
    import paper_2505_14884_b200 as pb
    from paper_2505_14884_b200 import _lib, kernels as pk

    d = 1024
    L = _lib.load()
    gen = torch.Generator(device=DEV).manual_seed(B + D + k)
    logits = torch.randn(B, D, device=DEV, generator=gen)
    if mode == "hot":
        logits[:, torch.randperm(D, device=DEV, generator=gen)[:1000]] += 5.0
    bias = torch.randn(D, device=DEV, generator=gen) * 0.1
    thr = 1.5
    # compacted path
    ws_n = int(L.ps_select_union_workspace_bytes(B, D))
    ws = torch.zeros(ws_n, dtype=torch.uint8, device=DEV)
    dpad = (D + 127) // 128 * 128
    idx = torch.zeros(dpad, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int32, device=DEV)
    _lib.call("ps_select_union", _lib.ptr(logits), _lib.ptr(bias), B, D, D, k, thr, _lib.ptr(ws), ws_n, 0, D, 128,
              _lib.ptr(idx), _lib.ptr(cnt), _lib.stream_ptr())
    # bitmap path (the other buffer starts dirty: the launch must clear it)
    bms = torch.zeros(2, (D + 31) // 32, dtype=torch.int32, device=DEV)
    bms[1].fill_(-1)
    _lib.call("ps_select_union_bitmap", _lib.ptr(logits), _lib.ptr(bias), B, D, D, k, thr, _lib.ptr(bms[0]),
              _lib.ptr(bms[1]), _lib.stream_ptr())
    torch.cuda.synchronize()
    assert int(bms[1].abs().sum()) == 0
    count = int(cnt)
    bits = bms[0].cpu().numpy().view(np.uint32)
    ids = np.nonzero(np.unpackbits(bits.view(np.uint8), bitorder="little"))[0]
    assert np.array_equal(ids, idx[:count].cpu().numpy())
    # the MLP through both paths
    w1 = (torch.randn(d, D, device=DEV, generator=gen) * 0.03).bfloat16().float()
    w2 = (torch.randn(d, D, device=DEV, generator=gen) * 0.03).bfloat16().float()
    b1 = torch.randn(D, device=DEV, generator=gen) * 0.05
    b2 = torch.randn(d, device=DEV, generator=gen) * 0.05
    packed = pb.PackedMLP.from_reference(w1, b1, w2, b2)
    x = torch.randn(B, d, device=DEV, generator=gen).bfloat16()
    res = torch.randn(B, d, device=DEV, generator=gen)
    hid_a = torch.zeros(B, packed.D_pad, dtype=torch.bfloat16, device=DEV)
    hid_b = torch.zeros_like(hid_a)
    out_a, out_b = res.clone(), res.clone()
    pk.mlp_into(packed, x, idx, cnt, hid_a, out_a, residual=out_a, expected=count)
    cnt_b = torch.full((1,), -7, dtype=torch.int32, device=DEV)
    pk.mlp_into_bitmap(packed, x, bms[0], cnt_b, hid_b, out_b, residual=out_b, expected=count)
    torch.cuda.synchronize()
    assert int(cnt_b) == count
    assert torch.equal(hid_a[:, :count], hid_b[:, :count])
    assert torch.equal(out_a, out_b)


@pytest.mark.parametrize("batch", [8, 64])
def test_engine_steps_identical_with_and_without_handoff(batch):
    import paper_2505_14884_b200 as pb
    from oracle import polar_oracle as po
    from paper_2505_14884_b200.engine import DecodeEngine, SparsityPolicy
    from paper_2505_14884_b200.model import DeviceModel, TransformerConfig

    cfg = TransformerConfig(2, 256, 1024, 8, 8, 512, 300, "relu")
    host = po.random_model(2, 256, 1024, 8, 8, 512, 300, seed=21)
    model = DeviceModel.from_host(cfg, host)
    outs = []
    for handoff in (False, True):
        policy = SparsityPolicy(mode="polar", mlp_k_table={0: 128, 1: 128}, head_density=0.5)
        hr = [pb.HeadRouter(256, 8, seed=40 + ell) for ell in range(2)]
        mr = [pb.MlpRouter(256, 1024, seed=30 + ell) for ell in range(2)]
        eng = DecodeEngine(model, batch, 300, policy, head_routers=hr, mlp_routers=mr, union_handoff=handoff)
        assert eng.union_handoff == handoff
        rng = np.random.default_rng(22)
        for c in eng.caches:
            c.fill_random(rng, 256)
        tokens = rng.integers(0, 512, batch, dtype=np.int64)
        eng.capture()
        steps = [eng.step(tokens).clone() for _ in range(4)]
        outs.append((steps, eng.union_counts.clone()))
    for a, b in zip(outs[0][0], outs[1][0]):
        assert torch.equal(a, b)
    assert torch.equal(outs[0][1], outs[1][1])
