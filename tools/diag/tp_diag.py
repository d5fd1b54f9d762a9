"""TP=2 on one GPU (gloo) vs TP=1: rel error with bf16 vs f32 partials, per case."""
import os, sys, socket
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import torch.multiprocessing as mp
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_gpu_tp as T


def _rank(rank, world, port, kv_heads, mode, q, f32, cg):
    import paper_2505_14884_b200.parallel as P
    if f32:
        def _partial(self, eng, name):
            t = self._tmp.get(name)
            if t is None:
                t = torch.zeros_like(eng.x)
                self._tmp[name] = t
            return t
        P.TensorParallel._partial = _partial
    T._rank(rank, world, port, kv_heads, mode, q)


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    for kv, mode in [(8, "polar"), (2, "polar"), (8, "dense")]:
        for f32 in (0, 1):
            q = ctx.Queue()
            port = T._port()
            ps = [ctx.Process(target=_rank, args=(r, 2, port, kv, mode, q, f32, 0)) for r in range(2)]
            for p in ps: p.start()
            for p in ps: p.join(timeout=300)
            try:
                print(kv, mode, "f32" if f32 else "bf16", q.get(timeout=10), flush=True)
            except Exception as e:
                print(kv, mode, f32, "ERR", e, [p.exitcode for p in ps], flush=True)
