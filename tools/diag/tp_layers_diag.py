"""TP=2 (gloo, one GPU) vs TP=1: the residual stream / LN output at every LayerNorm."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import torch.multiprocessing as mp
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_gpu_tp as T

CUR = {"l": None}


def patch():
    from paper_2505_14884_b200 import engine as E
    orig = E.DecodeEngine._ln

    def _ln(self, g, b, pending):
        x = self.x.clone()
        if pending is not None:
            x += pending
        CUR["l"].append(("x", x.cpu().numpy()))
        r = orig(self, g, b, pending)
        CUR["l"].append(("h", self.h.float().cpu().numpy()))
        return r
    E.DecodeEngine._ln = _ln


def _rank(rank, world, port, kv_heads, mode):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2505_14884_b200.model import TransformerConfig
    from paper_2505_14884_b200.parallel import TPPlan, TensorParallel
    cfg = TransformerConfig(2, 256, 1024, 8, kv_heads, 512, 288, "relu")
    plan = TPPlan.make(cfg, world, rank)
    patch()
    tp_rec = []
    CUR["l"] = tp_rec
    eng, tokens = T._build(kv_heads, mode, tp=TensorParallel(plan), plan=plan)
    eng.record = {}
    eng.step(tokens)
    if rank == 0:
        ref_rec = []
        CUR["l"] = ref_rec
        ref_eng, _ = T._build(kv_heads, mode)
        ref_eng.record = {}
        ref_eng.step(tokens)
        for i, ((n, a), (_, b)) in enumerate(zip(tp_rec, ref_rec)):
            print(i, n, "rel", float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30)), flush=True)
        for e in range(len(ref_eng.record.get("heads", []))):
            print("heads eq", bool(torch.equal(ref_eng.record["heads"][e], eng.record["heads"][e])))
        for e in range(len(ref_eng.record.get("union", []))):
            a, b = ref_eng.record["union"][e], eng.record["union"][e]
            print("union", a.numel(), b.numel(), "eq-shard0", bool(torch.equal(a[a < 512], b)))
    dist.destroy_process_group()


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    for kv in (8, 2):
        port = T._port()
        ps = [ctx.Process(target=_rank, args=(r, 2, port, kv, "polar")) for r in range(2)]
        for p in ps: p.start()
        for p in ps: p.join(timeout=300)
