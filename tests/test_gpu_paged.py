"""Paged KV cache: SHA through a block table is
bit-identical to SHA over the contiguous cache with the same contents (same
tiles, same partition, same merge order), matches the oracle, never reads
rows past a length or pages it does not map (NaN poison), and the paged
append writes the same rows as the contiguous one."""

import numpy as np
import pytest
import torch

from oracle import polar_oracle as po

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_14884_b200 as pb  # noqa: E402

DEV = torch.device("cuda")


def _t(a):
    return torch.as_tensor(np.asarray(a, np.float32), device=DEV)


@pytest.mark.parametrize("B,H,H_kv,d_h,N,P", [(6, 32, 32, 128, 300, 32), (5, 32, 8, 128, 700, 64),
                                              (3, 64, 8, 128, 1000, 128), (4, 8, 8, 32, 400, 128),
                                              (4, 8, 2, 64, 260, 64)])
def test_paged_sha_equals_contiguous_and_oracle(B, H, H_kv, d_h, N, P):
    rng = np.random.default_rng(B * 31 + H_kv + P)
    c = pb.KVCache(B, H_kv, N + 40, d_h, device=DEV)
    c.fill_random(rng, N)
    lens = rng.integers(1, N + 1, size=B)
    lens[0] = N
    lens[-1] = 1
    c.set_lengths(lens)
    # scattered pages in a pool with spare pages
    pc = pb.PagedKVCache.from_contiguous(c, page_rows=P, pool_pages=B * (-(-(N + 40) // P)) + 7, seed=5)
    assert (pc.host_table[0][: -(-N // P)] >= 0).all()
    q = po.round_bf16(rng.normal(size=(B, H, 1, d_h)).astype(np.float32))
    k = max(1, H_kv // 2)
    sel = np.stack([np.sort(rng.choice(H_kv, k, replace=False)) for _ in range(B)])
    bhi = pb.BatchHeadIndex(sel)
    ref_dev = pb.gqa_selective_attention_decode(_t(q), c, bhi).cpu()
    got = pb.gqa_selective_attention_decode(_t(q), pc, bhi).cpu()
    assert torch.equal(got, ref_dev)
    ref = po.naive_attention_reference(q, c.keys.float().cpu().numpy(), c.values.float().cpu().numpy(), lens,
                                       sel, H // H_kv)
    assert np.abs(got.numpy() - ref).max() <= 1e-2
    # poison: unmapped pages, rows past each length inside mapped pages, and
    # non-selected groups -- none of it may be read
    mapped = set(int(p) for p in pc.host_table[pc.host_table >= 0].ravel())
    for pg in range(pc.pool_pages):
        if pg not in mapped:
            pc.k_pool[pg] = float("nan")
            pc.v_pool[pg] = float("nan")
    for b in range(B):
        n = int(lens[b])
        for j in range(pc.max_pages):
            pg = int(pc.host_table[b, j])
            if pg < 0:
                continue
            lo = max(0, n - j * P)
            if lo < P:
                pc.k_pool[pg, :, lo:] = float("nan")
                pc.v_pool[pg, :, lo:] = float("nan")
            for g in range(H_kv):
                if g not in sel[b]:
                    pc.k_pool[pg, g] = float("nan")
                    pc.v_pool[pg, g] = float("nan")
    poisoned = pb.gqa_selective_attention_decode(_t(q), pc, bhi).cpu()
    assert torch.isfinite(poisoned).all()
    assert torch.equal(poisoned, got)


def test_paged_append_matches_contiguous():
    rng = np.random.default_rng(3)
    B, H_kv, d_h, P = 5, 4, 128, 32
    c = pb.KVCache(B, H_kv, 130, d_h, device=DEV)
    c.fill_random(rng, 30)
    c.set_lengths([30, 31, 32, 63, 64])  # appends land mid-page, at page ends and on fresh pages
    pc = pb.PagedKVCache.from_contiguous(c, page_rows=P, seed=1)
    for _ in range(3):
        kn = torch.randn(B, H_kv, d_h, device=DEV).bfloat16()
        vn = torch.randn(B, H_kv, d_h, device=DEV).bfloat16()
        c.append_step(kn, vn)
        pc.append_step(kn, vn)
    assert pc.lengths.cpu().tolist() == c.lengths.cpu().tolist() == [33, 34, 35, 66, 67]
    for b in range(B):
        for h in range(H_kv):
            assert torch.equal(pc.keys_for(b, h), c.keys_for(b, h))
            assert torch.equal(pc.values_for(b, h), c.values_for(b, h))
    # a fused strided source (the engine's QKV buffer layout) works too
    qkv = torch.randn(B, 3 * H_kv * d_h, device=DEV).bfloat16()
    kq, vq = qkv[:, H_kv * d_h:], qkv[:, 2 * H_kv * d_h:]
    pc.append_step(kq, vq, src_ld=qkv.stride(0))
    assert torch.equal(pc.keys_for(2, 1)[-1], kq[2, d_h:2 * d_h])


def test_paged_capacity_and_validation():
    pc = pb.PagedKVCache(2, 2, 64, 128, page_rows=32, pool_pages=3, device=DEV)
    pc.set_lengths([64, 0])
    with pytest.raises(pb.CapacityError):  # pool exhausted
        pc.set_lengths([64, 64])
    pc.release(0)
    pc.set_lengths([0, 64])
    kn = torch.zeros(2, 2, 128, device=DEV).bfloat16()
    with pytest.raises(pb.CapacityError):
        pc.append_step(kn, kn)
    with pytest.raises(ValueError):
        pb.PagedKVCache(2, 2, 64, 128, page_rows=48, device=DEV)  # not a tile multiple


def test_append_into_unmapped_page_is_refused():
    """unmapped pages are -1 on the device; the C-ABI append (no
    host reserve) refuses them -- nothing written, length kept, err 2 --
    instead of overwriting whichever sequence owns page 0."""
    from paper_2505_14884_b200 import _lib
    pc = pb.PagedKVCache(2, 2, 128, 128, page_rows=32, pool_pages=8, device=DEV)
    pc.set_lengths([32, 5])  # sequence 0: page 0 full, page 1 unmapped
    assert pc.block_table[0, 1].item() == -1
    before = pc.k_pool.clone()
    kn = torch.ones(2, 2, 128, device=DEV).bfloat16()
    _lib.call("ps_kv_append_paged", _lib.ptr(pc.k_pool), _lib.ptr(pc.v_pool), pc.page_rows,
              _lib.ptr(pc.block_table), pc.max_pages, _lib.ptr(pc.lengths), _lib.ptr(kn), _lib.ptr(kn),
              2 * 128, 2, 2, 128, _lib.ptr(pc._err), _lib.stream_ptr())
    assert pc.lengths.cpu().tolist() == [32, 6]  # sequence 1 appended, sequence 0 refused
    changed = (pc.k_pool != before).any(dim=(1, 2, 3)).nonzero().flatten().tolist()
    assert changed == [int(pc.host_table[1, 0])]  # only sequence 1's page was written
    with pytest.raises(ValueError, match="unmapped"):
        pc.check_errors()
    pc.check_errors()  # the flag was reset


@pytest.mark.parametrize("kv_heads,mode", [(8, "polar"), (2, "polar"), (8, "dense")])
def test_engine_step_paged_equals_contiguous(kv_heads, mode):
    """The decode engine over paged caches (scattered pages, separate paged
    append) produces the contiguous engine's logits, eager and from the
    captured graph."""
    from paper_2505_14884_b200.engine import DecodeEngine, SparsityPolicy
    from paper_2505_14884_b200.model import DeviceModel, TransformerConfig

    cfg = TransformerConfig(2, 256, 1024, 8, kv_heads, 512, 400, "relu")
    model = DeviceModel.from_host(cfg, po.random_model(2, 256, 1024, 8, kv_heads, 512, 400, seed=21))
    polar = mode == "polar"
    pol = SparsityPolicy(mode=mode, mlp_k_table={0: 128, 1: 128} if polar else None,
                         head_density=0.5 if polar else 1.0)
    hr = [pb.HeadRouter(256, kv_heads, seed=40 + e) for e in range(2)]
    mr = [pb.MlpRouter(256, 1024, seed=30 + e) for e in range(2)]
    engs = []
    for pr, rv in ((0, "full"), (128, "full"), (128, "on_demand")):  # head_dim 32: the SHA tile is 128 rows
        e = DecodeEngine(model, 8, 400, pol, head_routers=hr, mlp_routers=mr, kv_page_rows=pr, kv_reserve=rv)
        rng = np.random.default_rng(22)
        for c in e.caches:
            c.fill_random(rng, 252)
        engs.append(e)
    assert engs[1].paged and not engs[0].paged
    engs[0].enable_trace()  # its own selections force the oracle (eager and replayed steps)
    host = po.random_model(2, 256, 1024, 8, kv_heads, 512, 400, seed=21)
    rng = np.random.default_rng(22)
    ocaches = []
    for _ in range(2):
        c = po.KVCache(8, kv_heads, 400, 32)
        c.fill_random(rng, 252)
        ocaches.append(c)
    routers = [po.init_mlp_router(256, 1024, seed=30 + e) for e in range(2)]

    def oracle_step(tokens):
        tr = engs[0].trace
        forced = {"heads": {}, "union": {}}
        if polar:
            forced["heads"][1] = tr["heads"][1].cpu().numpy()
            forced["union"] = {e: tr["union"][e][: int(engs[0].union_counts[e].item())].cpu().numpy()
                               for e in range(2)}
        return po.decode_step(host, ocaches, tokens, mode=mode, head_density=pol.head_density,
                              k_table=pol.mlp_k_table, head_routers=[None, None], mlp_routers=routers,
                              forced=forced)

    def rel(a, b):
        a = a.cpu().numpy().astype(np.float64)
        return np.linalg.norm(a - b) / np.linalg.norm(b)

    tokens = np.random.default_rng(1).integers(0, 512, 8)
    for _ in range(2):
        outs = [e.step(tokens).clone() for e in engs]
        ref = oracle_step(tokens)
        assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
        assert rel(outs[0], ref) <= 2e-2
    for e in engs:
        e.capture()
    assert (engs[2].caches[1].host_table >= 0).sum() == 2 * 8  # on demand: only pages 0-1 so far
    for _ in range(140):  # 254 -> 394 rows: past the 256-row page and > 1 SHA tile past the capture window
        outs = [e.step(tokens).clone() for e in engs]
        ref = oracle_step(tokens)
        assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
        assert rel(outs[0], ref) <= 2e-2
    assert engs[1].caches[1].lengths.cpu().tolist() == [394] * 8
    assert (engs[2].caches[1].host_table >= 0).sum() == 4 * 8  # pages 2-3 mapped as the appends entered them


def test_head_router_fused_append_into_pages():
    """ps_head_router_topk_append_paged: same selections as the contiguous
    fused launch, and the same K/V rows land in the pages."""
    rng = np.random.default_rng(11)
    B, H_kv, d_h, d = 6, 8, 128, 512
    c = pb.KVCache(B, H_kv, 200, d_h, device=DEV)
    c.fill_random(rng, 60)
    c.set_lengths([60, 63, 64, 95, 96, 127])  # mid-page, page ends and fresh pages (32-row pages)
    pc = pb.PagedKVCache.from_contiguous(c, page_rows=32, seed=3)
    hr = pb.HeadRouter(d, H_kv, seed=2)
    x = torch.randn(B, d, device=DEV).bfloat16()
    qkv = torch.randn(B, 3 * H_kv * d_h, device=DEV).bfloat16()
    kq, vq = qkv[:, H_kv * d_h:], qkv[:, 2 * H_kv * d_h:]
    sel_a = torch.zeros(B, 3, dtype=torch.int32, device=DEV)
    sel_b = torch.zeros(B, 3, dtype=torch.int32, device=DEV)
    for b in range(B):  # the caller maps the page each append lands in (as the engine does)
        pc.reserve(b, int(pc.host_lengths[b]) + 1)
    hr.select_append_into(x, 3, sel_a, c, kq, vq, qkv.stride(0))
    hr.select_append_into(x, 3, sel_b, pc, kq, vq, qkv.stride(0))
    c.host_lengths += 1
    pc.host_lengths += 1
    torch.cuda.synchronize()
    assert torch.equal(sel_a, sel_b)
    assert pc.lengths.cpu().tolist() == c.lengths.cpu().tolist() == [61, 64, 65, 96, 97, 128]
    for b in range(B):
        for h in range(H_kv):
            assert torch.equal(pc.keys_for(b, h), c.keys_for(b, h))
            assert torch.equal(pc.values_for(b, h), c.values_for(b, h))
