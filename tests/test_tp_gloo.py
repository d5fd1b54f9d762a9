"""Tensor-parallel sharding math on CPU: world_size 2, gloo backend.

Each rank takes its shard of the tiny model exactly as ``TPPlan`` (the
product's plan) prescribes -- local q/k/v columns and KV groups, W_o rows,
neuron rows of W1/W2 -- computes its partial residual updates with the CPU
oracle primitives, and all-reduces them.  The sharded step must reproduce the
unsharded oracle decode step (selections are replicated, so they are
identical on every rank by construction)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import polar_oracle as po

F32 = np.float32


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _tp_step(rank, world, port, kv_heads, mode, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_14884_b200.model import TransformerConfig
        from paper_2505_14884_b200.parallel import TPPlan

        cfg = TransformerConfig(2, 256, 1024, 8, kv_heads, 512, 288, "relu")
        plan = TPPlan.make(cfg, world, rank)
        m = po.random_model(2, 256, 1024, 8, kv_heads, 512, 288, seed=21)
        rng = np.random.default_rng(22)
        full_caches = []
        for _ in range(2):
            c = po.KVCache(8, kv_heads, 288, 32)
            c.fill_random(rng, 256)
            full_caches.append(c)
        tokens = rng.integers(0, 512, 8, dtype=np.int64)
        hr = [po.init_head_router(256, kv_heads, seed=40 + e) for e in range(2)]
        mr = [po.init_mlp_router(256, 1024, seed=30 + e) for e in range(2)]
        polar = mode == "polar"
        rho, k_mlp = (0.5, 128) if polar else (1.0, None)

        d, H, d_h, G = 256, 8, 32, plan.group_size
        B = 8
        q0, q1 = plan.q_cols
        k0, k1 = plan.kv_cols
        f0, f1 = plan.ffn_range
        g0 = plan.group_base
        # local caches: this rank's KV groups only
        caches = []
        for c in full_caches:
            lc = po.KVCache(B, plan.kv_heads_local, 288, d_h)
            lc.keys[:] = c.keys[:, g0:g0 + plan.kv_heads_local]
            lc.values[:] = c.values[:, g0:g0 + plan.kv_heads_local]
            lc.lengths[:] = c.lengths
            caches.append(lc)
        pos = caches[0].lengths.copy()
        x = m["embed"][tokens] + m["pos_embed"][pos]
        for ell, lw in enumerate(m["layers"]):
            cache = caches[ell]
            h1 = po.layernorm(x, lw["ln1_g"], lw["ln1_b"])
            q = (po.matmul(h1, lw["w_q"][:, q0:q1]) + lw["b_q"][q0:q1]).reshape(B, plan.heads_local, 1, d_h)
            kk = (po.matmul(h1, lw["w_k"][:, k0:k1]) + lw["b_k"][k0:k1]).reshape(B, plan.kv_heads_local, d_h)
            vv = (po.matmul(h1, lw["w_v"][:, k0:k1]) + lw["b_v"][k0:k1]).reshape(B, plan.kv_heads_local, d_h)
            cache.append_step(kk, vv)
            if polar and ell > 0:  # replicated router -> identical global selection
                sel = po.topk_indices_rows(po.head_router_forward(hr[ell]["w"], hr[ell]["b"], h1),
                                           po.head_budget(rho, kv_heads))
            else:
                sel = np.tile(np.arange(kv_heads), (B, 1))
            attn = np.zeros((B, plan.heads_local, 1, d_h), F32)
            for b in range(B):
                mine = plan.groups_of(sel[b])
                if mine:
                    one = po.KVCache(1, plan.kv_heads_local, 288, d_h)
                    one.keys[0], one.values[0], one.lengths[0] = cache.keys[b], cache.values[b], cache.lengths[b]
                    attn[b] = po.gqa_selective_attention_decode(q[b:b + 1], one, np.array([[g - g0 for g in mine]]))[0]
            o_part = po.matmul(attn[:, :, 0, :].reshape(B, q1 - q0), lw["w_o"][q0:q1, :])
            if rank == 0:
                o_part = o_part + lw["b_o"]
            t = torch.from_numpy(np.ascontiguousarray(o_part))
            dist.all_reduce(t)
            x = x + t.numpy()
            h2 = po.layernorm(x, lw["ln2_g"], lw["ln2_b"])
            if polar:
                logits = po.mlp_router_forward(mr[ell]["w_in"], mr[ell]["b_in"], mr[ell]["w_out"], mr[ell]["b_out"], h2)
                union = po.union_neuron_indices(list(po.topk_indices_rows(logits, k_mlp)))
            else:
                union = np.arange(1024)
            local = np.array(plan.union_local(union), np.int64) + f0
            part = np.zeros((B, d), F32)
            if local.size:
                hmid = np.maximum(h2.astype(np.float64) @ lw["mlp_w1"][:, local].astype(np.float64)
                                  + lw["mlp_b1"][local], 0.0)
                part = (hmid @ lw["mlp_w2"][:, local].astype(np.float64).T).astype(F32)
            if rank == 0:
                part = part + lw["mlp_b2"]
            t = torch.from_numpy(np.ascontiguousarray(part))
            dist.all_reduce(t)
            x = x + t.numpy()
        logits = po.matmul(po.layernorm(x, m["lnf_g"], m["lnf_b"]), m["unembed"])
        if rank == 0:
            ref = po.decode_step(m, full_caches, tokens, mode=mode, head_density=rho,
                                 k_table={0: 128, 1: 128} if polar else None, head_routers=hr, mlp_routers=mr)
            out_q.put((float(np.abs(logits - ref).max()), float(np.abs(ref).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kv_heads,mode", [(8, "polar"), (2, "polar"), (8, "dense")])
def test_tp2_matches_unsharded_oracle(kv_heads, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tp_step, args=(r, 2, port, kv_heads, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    err, scale = q.get(timeout=10)
    assert err <= 1e-4 * max(1.0, scale), err


def test_plan_partitions_everything_once():
    from paper_2505_14884_b200.model import SHAPES
    from paper_2505_14884_b200.parallel import TPPlan

    for name in ("opt-66b", "llama-3.1-70b", "tiny"):
        cfg = SHAPES[name]
        for world in (1, 2, 4, 8):
            if cfg.kv_heads % world or cfg.ffn_dim % (32 * world):
                continue
            groups, neurons, qcols = [], [], []
            for r in range(world):
                p = TPPlan.make(cfg, world, r)
                groups += list(range(p.group_base, p.group_base + p.kv_heads_local))
                neurons += list(range(*p.ffn_range))
                qcols += list(range(*p.q_cols))
                assert p.heads_local == p.kv_heads_local * cfg.group_size
            assert groups == list(range(cfg.kv_heads))
            assert neurons == list(range(cfg.ffn_dim))
            assert qcols == list(range(cfg.model_dim))
    with pytest.raises(ValueError):
        TPPlan.make(SHAPES["llama-3.1-8b"], 16, 0)
