"""Tensor-parallel decode step on the device path: 2 ranks sharing one GPU
(gloo carries the CUDA partial sums; NCCL needs distinct GPUs), each running
its shard engine (group_base-offset SHA, [lo, hi) union compaction, shard
GEMMs, bf16 partial sums all-reduced).

The check is the oracle decode step (oracle/polar_oracle.py, restating
sparsedecode/engine.py:314-392) run with the TP engine's OWN selections:
the global head selection (identical on every rank: replicated routers)
and the global union (the ranks' local unions rebased and concatenated).
Comparing TP against the TP=1 engine instead is not a parity check: the
bf16 partials shift the router inputs by ~1e-3 and near-tie neurons flip."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

CFG = (2, 256, 1024, 8, 512, 288)  # layers, d, D, H, vocab, max_seq
B, CTX, CAP, D_H = 8, 256, 288, 32


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _kv_draws(kv_heads):
    rng = np.random.default_rng(22)
    draws = []
    for _ in range(CFG[0]):
        k = rng.standard_normal((B, kv_heads, CTX, D_H), dtype=np.float32)
        v = rng.standard_normal((B, kv_heads, CTX, D_H), dtype=np.float32)
        draws.append((k, v))
    tokens = rng.integers(0, CFG[4], B, dtype=np.int64)
    return draws, tokens


def _policy_kw(mode):
    polar = mode == "polar"
    return dict(mlp_k_table={0: 128, 1: 128} if polar else None, head_density=0.5 if polar else 1.0)


def _build(kv_heads, mode, tp=None, plan=None):
    from oracle import polar_oracle as po
    import paper_2505_14884_b200 as pb
    from paper_2505_14884_b200.engine import DecodeEngine, SparsityPolicy
    from paper_2505_14884_b200.model import DeviceModel, TransformerConfig
    from paper_2505_14884_b200.parallel import shard_model

    L, d, D, H, V, S = CFG
    cfg = TransformerConfig(L, d, D, H, kv_heads, V, S, "relu")
    host = po.random_model(L, d, D, H, kv_heads, V, S, seed=21)
    model = DeviceModel.from_host(cfg, host)
    if plan is not None:
        model = shard_model(model, plan)
    policy = SparsityPolicy(mode=mode, **_policy_kw(mode))
    hr = [pb.HeadRouter(d, kv_heads, seed=40 + e) for e in range(L)]
    mr = [pb.MlpRouter(d, D, seed=30 + e) for e in range(L)]
    eng = DecodeEngine(model, B, CAP, policy, head_routers=hr, mlp_routers=mr, tp=tp)
    draws, tokens = _kv_draws(kv_heads)
    g0 = 0 if plan is None else plan.group_base
    nl = kv_heads if plan is None else plan.kv_heads_local
    for c, (k, v) in zip(eng.caches, draws):
        c.keys[:, :, :CTX] = torch.from_numpy(k[:, g0:g0 + nl]).to(c.keys.device).bfloat16()
        c.values[:, :, :CTX] = torch.from_numpy(v[:, g0:g0 + nl]).to(c.keys.device).bfloat16()
        c.set_lengths([CTX] * B)
    return eng, tokens


def oracle_logits(kv_heads, mode, tokens, heads, unions, steps_before=()):
    """The oracle decode step over the same (bf16-rounded) history, forced to
    the given per-layer selections.  ``steps_before``: earlier steps'
    (tokens, heads, unions) replayed first so the histories line up."""
    from oracle import polar_oracle as po

    L, d, D, H, V, S = CFG
    host = po.random_model(L, d, D, H, kv_heads, V, S, seed=21)
    draws, _ = _kv_draws(kv_heads)
    caches = []
    for k, v in draws:
        c = po.KVCache(B, kv_heads, CAP, D_H)
        c.keys[:, :, :CTX] = po.round_bf16(k)
        c.values[:, :, :CTX] = po.round_bf16(v)
        c.lengths[:] = CTX
        caches.append(c)
    kw = dict(mode=mode, head_density=_policy_kw(mode)["head_density"], k_table=_policy_kw(mode)["mlp_k_table"],
              head_routers=[None] * L, mlp_routers=[po.init_mlp_router(d, D, seed=30 + e) for e in range(L)])
    out = None
    for tk, hd, un in list(steps_before) + [(tokens, heads, unions)]:
        forced = {"heads": hd, "union": un}
        out = po.decode_step(host, caches, tk, forced=forced, **kw)
    return out


def _selections(eng, plan, world):
    """Global per-layer head selections and unions of this step (gathered)."""
    import torch.distributed as dist

    rec = eng.record
    heads = {}
    li = [ell for ell in range(CFG[0]) if eng.k_heads[ell]]
    for j, ell in enumerate(li):
        heads[ell] = rec["heads"][j].cpu().numpy()
    unions = {}
    for ell, u in enumerate(rec.get("union", [])):
        mine = (u.cpu().numpy().astype(np.int64) + plan.ffn_range[0]) if plan else u.cpu().numpy()
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        unions[ell] = np.concatenate(parts)
    return heads, unions


def selections_from_trace(eng, plan, world):
    """Same as the record, from the engine's device trace (graph replays)."""
    import torch.distributed as dist

    heads = {ell: eng.trace["heads"][ell].cpu().numpy() for ell in range(CFG[0]) if eng.k_heads[ell]}
    unions = {}
    if eng.sparse_mlp:
        counts = eng.union_counts.cpu().numpy()
        for ell in range(CFG[0]):
            u = eng.trace["union"][ell][: int(counts[ell])].cpu().numpy().astype(np.int64)
            mine = u + (plan.ffn_range[0] if plan else 0)
            parts = [None] * world
            dist.all_gather_object(parts, mine)
            unions[ell] = np.concatenate(parts)
    return heads, unions


def _rank(rank, world, port, kv_heads, mode, q, collective="nccl"):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2505_14884_b200.model import TransformerConfig
        from paper_2505_14884_b200.parallel import TPPlan, TensorParallel

        L, d, D, H, V, S = CFG
        cfg = TransformerConfig(L, d, D, H, kv_heads, V, S, "relu")
        plan = TPPlan.make(cfg, world, rank)
        eng, tokens = _build(kv_heads, mode, tp=TensorParallel(plan, dist.group.WORLD, collective=collective),
                             plan=plan)
        eng.record = {}
        logits = eng.step(tokens).cpu().numpy()
        heads, unions = _selections(eng, plan, world)
        if rank == 0:
            ref = oracle_logits(kv_heads, mode, tokens, heads, unions)
            q.put((float(np.linalg.norm(logits - ref) / np.linalg.norm(ref)), float(np.abs(logits - ref).max()),
                   float(np.abs(ref).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kv_heads,mode,collective", [(8, "polar", "nccl"), (2, "polar", "nccl"),
                                                     (8, "dense", "nccl"), (8, "polar", "p2p"),
                                                     (2, "polar", "p2p")])
def test_tp2_device_matches_oracle(kv_heads, mode, collective):
    """collective "nccl": the torch.distributed all-reduce (gloo here: the
    ranks share one GPU); "p2p": the fused peer-memory all-reduce + residual
    add (ps_allreduce_add_bf16) over CUDA IPC mappings."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, kv_heads, mode, q, collective)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
        assert p.exitcode == 0
    rel, mx, scale = q.get(timeout=10)
    # the oracle tolerance of tests/test_gpu_engine.py (bf16 weights, bf16
    # partial sums in the all-reduce, f32 residual)
    assert rel <= 2e-2, (rel, mx)
    assert mx <= 2e-2 * max(1.0, scale), (rel, mx)
