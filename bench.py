"""Decode throughput benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config opt-6.7b] [--batch 64] [--ctx 1920] [--rho 0.5]
                    [--union 0.5] [--k-frac 0.1] [--dp] [--no-extra]

Metric (BASELINE.json): decode tokens/s of the polar sparse step vs the dense
step, at the OPT-6.7B shape (configs[1]) by default: random-init weights
N(0, 0.02), synthetic N(0,1) KV history of ``ctx`` tokens, batch 64, head
density rho = 0.5 (16 of 32 heads from the head router's top-k; layer 0
dense).  Neuron selection follows the reference's heavy-tailed
"hot-neuron" recipe (analysis.py:124-140): every token keeps its top
k = 0.1*D router logits; a fixed hot set (7.2 % of D: the batch union is
~0.5*D at B = 64) fires on every token, the remaining picks vary token by
token, so |S| grows with the batch as in the paper.  A "step"
= one full decode step (embed -> L x [LN, QKV, KV append, head router +
top-k, SHA, O-proj, LN, MLP router, top-k, union, selective MLP] -> LN ->
LM head -> argmax), replayed from one CUDA graph.  Inputs exceed L2
(tens of GB of KV), so no explicit L2 flush.

* value        -- polar tok/s, device-timed (CUDA events), max over ranks;
* dense        -- the same engine at full density (every head, every
                  neuron; cuBLAS dense MLP) on the same caches;
* e2e          -- ``DecodeEngine.step()`` (the public API) with HOST tokens:
                  per step the pinned H2D copy of the tokens, the graph
                  replay, the D2H read of the next tokens and a host sync,
                  all inside the timed region;
* roofline     -- the SHA kernel (dominant) timed alone on the same caches:
                  algorithmic bytes / CUDA-event duration vs
                  MEASURED_PEAKS.json hbm_gbs;
* cpu_baseline -- the UNMODIFIED reference package (``sparsedecode``,
                  installed into baseline/_ref) running its own
                  ``engine.decode_step`` on one layer of the same workload
                  on the host cores, x L layers;
* configs      -- further driver-observed points (other batch sizes, the
                  LLaMA-3.1-8B shape), each with the byte-model ideal ratio.

``--impl reference`` runs only the reference arm (rank 0; other ranks exit).
N > 1 (torchrun): tensor parallelism over the ranks on the same workload
(one global batch, heads + neurons sharded, routers replicated, NCCL
all-reduce of bf16 partials after the O- and down-projections; strong
scaling); ``--dp`` runs independent data-parallel replicas instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="opt-6.7b")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=1920)
    ap.add_argument("--rho", type=float, default=0.5)
    ap.add_argument("--union", type=float, default=0.5, help="hot-set recipe: |S|/D (= k/D)")
    ap.add_argument("--hot-frac", type=float, default=0.072,
                    help="hot-cold recipe: hot-set size / D (0.072: |S|/D ~ 0.5 at B=64, OPT-6.7B)")
    ap.add_argument("--k-frac", type=float, default=0.1, help="per-token neuron budget k / D")
    ap.add_argument("--union-recipe", default="hot-cold", choices=["hot-cold", "hot-set"],
                    help="hot-cold: per-token top-k over a fixed hot set + varying cold picks (default); "
                         "hot-set: every token's top-k is exactly the same hot set (k = |S|)")
    ap.add_argument("--kv-ring", type=int, default=0, help="alias KV storage over this many buffers (0 = auto)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the extra driver-observed configs")
    ap.add_argument("--dp", action="store_true", help="N > 1: data-parallel replicas instead of TP")
    ap.add_argument("--tp", action="store_true", help="(default for N > 1) tensor parallelism over the ranks")
    ap.add_argument("--tp-collective", default="nccl", choices=["nccl", "p2p"],
                    help="TP exchange: NCCL all-reduce, or the fused peer-memory all-reduce + residual add")
    ap.add_argument("--distinct-layers", type=int, default=0,
                    help="TP: distinct weight sets cycled over the layers (0 = all distinct)")
    ap.add_argument("--cpu-batch", type=int, default=0, help="batch of the CPU sample (0 = the workload batch)")
    ap.add_argument("--router-backend", default=None, choices=[None, "cublas", "fused", "native", "native_in"])
    ap.add_argument("--kv-page-rows", type=int, default=0,
                    help="paged KV caches with this many rows per page (0 = contiguous)")
    ap.add_argument("--kv-reserve", default="full", choices=["full", "on_demand"],
                    help="paged KV: map every page up front, or each page as the appends enter it")
    ap.add_argument("--union-handoff", choices=("auto", "on", "off"), default="auto",
                    help="selection writes only the union bitmap and UP / DOWN derive the ids on the device "
                    "(auto = the engine default: off)")
    ap.add_argument("--concurrent-head-router", choices=("auto", "on", "off"), default="auto", nargs="?",
                    const="on", help="head router as a concurrent graph branch (+ a separate KV append) instead of "
                    "fused with the KV append; auto = on for B <= 8 without TP (the engine default)")
    return ap.parse_args(argv)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._ready = threading.Event()  # set once the sampler is live (NVML init can take ~100 ms)
        self._t = None

    def _run(self):
        try:  # NVML directly: 20 ms sampling (nvidia-smi costs ~100 ms per call)
            import pynvml as nv

            nv.nvmlInit()
            hd = nv.nvmlDeviceGetHandleByIndex(self.index)
            bits = [nv.nvmlClocksThrottleReasonHwSlowdown, nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                    nv.nvmlClocksThrottleReasonSwThermalSlowdown, nv.nvmlClocksThrottleReasonSwPowerCap]
            nv.nvmlDeviceGetClockInfo(hd, nv.NVML_CLOCK_SM)
            self._ready.set()
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(hd, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(hd, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(hd)
                self.samples.append([str(sm), str(mx), "0"] + ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.02)
            return
        except Exception:
            pass
        self._ready.set()
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(timeout=10)
        self.samples.clear()  # only samples taken inside the timed region count
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------- workload recipe
def neuron_recipe(args, D: int):
    """(k per token, hot-set size) of the MLP selection.

    hot-cold (default; the reference's heavy-tailed profile,
    analysis.py:124-140): every token keeps its top k = k_frac*D router
    logits.  A hot set of hot_frac*D neurons carries a large router bias, so
    it fires on every token (hot_p ~ 1); the remaining picks come from the
    centered random router and vary token by token, so the batch union |S|
    grows with the batch.  hot_frac = 0.072 gives |S|/D ~ 0.5 at B = 64 on the
    OPT-6.7B shape (measured on B200 with tools/union_calib.py: 1000 hot ->
    0.60, 1500 -> 0.32); the measured |S| is reported next to every number.
    hot-set: every token's top-k is exactly the hot set (k = |S| = union*D).
    """
    if args.union_recipe == "hot-set":
        k = max(1, int(round(args.union * D)))
        return k, k
    k = max(1, int(round(args.k_frac * D)))
    return k, min(k, int(round(args.hot_frac * D)))


def workload_config(args, cfg, batch=None, config=None, ctx=None, world=1, tp=False):
    """The workload keys shared by both arms (GPU-only facts live elsewhere)."""
    config = config or args.config
    batch = batch or args.batch
    ctx = ctx or args.ctx
    D = cfg.ffn_dim
    k, n_hot = neuron_recipe(args, D)
    return {"workload": f"{config} polar decode step", "model_shape": config, "global_batch": batch,
            "seq_len": ctx, "head_density": args.rho,
            "neuron_selection": (f"per-token top-{k} (k/D={k / D:.3f}): a hot set of {n_hot} on every token + "
                                 f"per-token picks of a centered random router (analysis.py:124-140 profile)"
                                 if args.union_recipe == "hot-cold" else f"every token's top-{k} = one hot set")
            if cfg.activation == "relu" else "dense SwiGLU MLP (never sparsified, engine.py:67-70)",
            "layers": cfg.layers, "d_model": cfg.model_dim, "ffn": cfg.ffn_dim, "heads": cfg.heads,
            "kv_heads": cfg.kv_heads, "parallelism": (f"tp{world}" if tp else f"dp{world}"),
            "l2": "inputs larger than L2 (KV cache >> 126 MB); no flush"}


# ---------------------------------------------------------------- byte model
def step_bytes(cfg, B, ctx, k_h, S, dense: bool, tp: int = 1) -> float:
    """HBM bytes one decode step must move per GPU (bf16 weights and KV):
    every layer's QKV / O weights, the selected K/V rows, the routers and
    the gathered MLP rows (polar) or every MLP weight (dense), plus the LM
    head.  Layer 0 attention is dense in polar mode (SparsityPolicy)."""
    d, D, H_kv, d_h = cfg.model_dim, cfg.ffn_dim, cfg.kv_heads, cfg.head_dim
    dk = H_kv * d_h
    attn_w = (d * (d + 2 * dk) + d * d) * 2 / tp
    kv_full = B * ctx * H_kv * d_h * 4 / tp
    total = 0.0
    for ell in range(cfg.layers):
        total += attn_w
        if dense or ell == 0:
            total += kv_full
        else:
            total += kv_full * k_h / H_kv + d * H_kv * 2
        if cfg.activation == "swiglu":
            total += 3 * D * d * 2 / tp
        elif dense:
            total += 2 * D * d * 2 / tp
        else:
            h_r = min(1024, 4 * d)
            total += (d * h_r + h_r * D) * 2 + 2 * S * d * 2 / tp + B * D * 4
    total += cfg.vocab * d * 2
    return total


def ideal_ratio(cfg, B, ctx, rho, S):
    k_h = max(1, math.ceil(rho * cfg.kv_heads - 1e-9))
    return step_bytes(cfg, B, ctx, k_h, S, True) / step_bytes(cfg, B, ctx, k_h, S, False)


# ---------------------------------------------------------------- reference (CPU) leg
def import_reference():
    """The unmodified reference package: baseline/_ref (pip-installed from
    /root/reference, travels to the GPU box), else None."""
    if REF_DIR not in sys.path and os.path.isdir(os.path.join(REF_DIR, "sparsedecode")):
        sys.path.insert(0, REF_DIR)
    try:
        import sparsedecode  # noqa: F401
        return sparsedecode
    except Exception:
        return None


def cpu_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        blas = int(max(n)) if n else None
    except Exception:
        pass
    return {"cpu_count": os.cpu_count(), "cpu_model": model, "blas_threads": blas}


def reference_layer_sample(args, cfg, batch, reps=2, warm=1, seed=0):
    """One polar decode layer of the workload through the reference's own
    ``engine.decode_step`` (a 1-layer model of the same shape, vocab 512 so
    the LM head is negligible, layer-0 attention routed like every other
    layer).  Returns (seconds per layer, kind, sample text); falls back to
    the oracle port only if the reference package is not importable."""
    rng = np.random.default_rng(seed)
    d, D, H, H_kv, d_h = cfg.model_dim, cfg.ffn_dim, cfg.heads, cfg.kv_heads, cfg.head_dim
    relu = cfg.activation == "relu"
    k, n_hot = neuron_recipe(args, D)
    cap = args.ctx + warm + reps + 2
    sd = import_reference()
    if sd is not None:
        from sparsedecode import engine as sde, model as sdm
        c1 = sdm.TransformerConfig(1, d, D, H, H_kv, 512, cap, cfg.activation)
        model = sdm.random_model(c1, seed)
        cache = sd.KVCache(batch, H_kv, cap, d_h)
        cache.fill_random(rng, args.ctx)
        hr = [sd.HeadRouter(d, H_kv, seed=100)]
        mr = None
        table = None
        if relu:
            mr = [sd.MlpRouter(d, D, seed=200)]
            if args.union_recipe == "hot-cold":  # the same centered router as the GPU arm
                mr[0].b_out_ -= mr[0].w_out_.sum(axis=0) / math.sqrt(math.pi)
            mr[0].b_out_[rng.choice(D, n_hot, replace=False)] += 20.0
            table = sd.LayerKTable(((0, k, 1.0),))
        policy = sd.SparsityPolicy(mode="polar", mlp_k_table=table, head_density=args.rho,
                                   layer0_dense_attention=False)
        sess = sd.DecodeSession(caches=[cache], policy=policy, mlp_routers=mr, head_routers=hr)

        def layer():
            sde.decode_step(sess, model, rng.integers(0, 512, batch))
        kind, what = "reference", "sparsedecode.engine.decode_step (unmodified reference, baseline/_ref)"
    else:
        from oracle import polar_oracle as po
        host = po.random_model(1, d, D, H, H_kv, 512, cap, cfg.activation, seed=seed)
        cache = po.KVCache(batch, H_kv, cap, d_h)
        cache.fill_random(rng, args.ctx)
        mrs = None
        if relu:
            mrs = [po.init_mlp_router(d, D, seed=200)]
            if args.union_recipe == "hot-cold":
                mrs[0]["b_out"] -= mrs[0]["w_out"].sum(axis=0) / math.sqrt(math.pi)
            mrs[0]["b_out"][rng.choice(D, n_hot, replace=False)] += 20.0
        hrs = [po.init_head_router(d, H_kv, seed=100)]

        def layer():
            po.decode_step(host, [cache], rng.integers(0, 512, batch), mode="polar", head_density=args.rho,
                           layer0_dense=False, k_table={0: k} if relu else None, head_routers=hrs,
                           mlp_routers=mrs)
        kind, what = "port", "oracle/polar_oracle.py decode_step (numpy port; reference not importable)"
    for _ in range(warm):
        layer()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        layer()
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    sample = (f"{what}: one decode layer of {args.config} at B={batch}, ctx {args.ctx}, rho {args.rho}, "
              f"per-token top-{k if relu else 0} neurons, median of {reps} after {warm} warm-up, x {cfg.layers} "
              f"layers (embed / LM head excluded)")
    return t, kind, sample


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2505_14884_b200.model import SHAPES

    cfg = SHAPES[args.config]
    batch = args.cpu_batch or args.batch
    t_setup = time.perf_counter()
    reps = max(1, min(args.steps, 3))
    s, kind, sample = reference_layer_sample(args, cfg, batch, reps=reps, warm=min(args.warmup, 1))
    step_s = s * cfg.layers
    value = batch / step_s
    info = cpu_info()
    line = {"impl": "reference", "metric": "decode_tokens_per_s", "value": value, "unit": "tok/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
            "higher_is_better": True, "scaling": "weak" if (args.gpus == 1 or args.dp) else "strong",
            "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
            "config": workload_config(args, cfg, world=args.gpus, tp=args.gpus > 1 and not args.dp),
            "cpu_baseline": {"value": value, "unit": "tok/s", "cores": info["blas_threads"] or info["cpu_count"],
                             "kind": kind, "sample": sample + (f" (batch {batch} of {args.batch}: tok/s per "
                                                               f"host-step scales with the batch)"), **info},
            "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_setup}
    print(json.dumps(line), flush=True)


def ncu_traffic(kernel, args):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel`
    from the committed `ncu --set full` capture of this same workload
    (profiles/r02_ncu_traffic.json), else None."""
    if (args.config, args.batch, args.ctx, args.rho) != ("opt-6.7b", 64, 1920, 0.5):
        return None, None
    for name in ("r02_ncu_traffic.json", "r01_ncu_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                doc = json.load(f)
            for k in doc["kernels"]:
                if kernel in k["kernel"]:
                    return k["dram_read_bytes"] + k["dram_write_bytes"], f"profiles/{name}"
        except Exception:
            continue
    return None, None


# ---------------------------------------------------------------- our arm
def sha_algorithmic_bytes(lengths, k_h, G, d_h, B, H):
    """selected K+V rows + Q + O (zeros included) + ids + lengths."""
    kv = float(np.sum(lengths)) * k_h * d_h * 2 * 2
    return kv + B * k_h * G * d_h * 2 + B * H * d_h * 2 + B * k_h * 4 + B * 4


class Setup:
    """Engines (polar + dense on shared caches) for one workload point."""

    def __init__(self, args, config, B, ctx, dev, world, rank, tp_on, steps, warmup, model=None):
        import torch

        import paper_2505_14884_b200 as pb
        from paper_2505_14884_b200.engine import DecodeEngine, SparsityPolicy
        from paper_2505_14884_b200.model import SHAPES, DeviceModel

        self.cfg = cfg = SHAPES[config]
        self.B, self.ctx = B, ctx
        L, H_kv, d_h, D = cfg.layers, cfg.kv_heads, cfg.head_dim, cfg.ffn_dim
        self.cap = cap = ctx + warmup * 2 + steps * 3 + 16
        free = torch.cuda.mem_get_info(dev)[0]
        self.tp = None
        if tp_on:
            from paper_2505_14884_b200.parallel import TPPlan, TensorParallel, random_shard

            plan = TPPlan.make(cfg, world, rank)
            import torch.distributed as dist

            self.tp = TensorParallel(plan, dist.group.WORLD if world > 1 else None,
                                     collective=getattr(args, "tp_collective", "nccl"))
            self.model = model or random_shard(cfg, plan, seed=1234, device=dev,
                                               distinct_layers=args.distinct_layers or None)
            self.H_loc, self.Hkv_loc, self.D_loc = plan.heads_local, plan.kv_heads_local, plan.ffn_local
        else:
            self.model = model or DeviceModel.random(cfg, seed=1234 + rank, device=dev)
            self.H_loc, self.Hkv_loc, self.D_loc = cfg.heads, H_kv, D
        kv_layer = B * self.Hkv_loc * cap * d_h * 2 * 2
        budget = free - (0 if model is not None else self.model.weight_bytes()) - 14 * 2 ** 30
        ring = args.kv_ring or (L if kv_layer * L <= budget else max(2, int(budget // kv_layer)))
        self.ring = min(ring, L)
        self.k_h = math.ceil(args.rho * H_kv - 1e-9)
        self.relu = cfg.activation == "relu"
        k, n_hot = neuron_recipe(args, D)
        self.k_mlp, self.n_hot = k, n_hot
        gen = np.random.default_rng(7)  # same on every TP rank: routers are replicated
        hr = [pb.HeadRouter(cfg.model_dim, H_kv, seed=100 + ell, device=dev) for ell in range(L)]
        mr = None
        if self.relu:
            mr = [pb.MlpRouter.random_device(cfg.model_dim, D, seed=200 + ell, device=dev,
                                             hot=gen.choice(D, n_hot, replace=False) if n_hot else None,
                                             center=args.union_recipe == "hot-cold")
                  for ell in range(L)]
        polar = SparsityPolicy(mode="polar", head_density=args.rho,
                               mlp_k_table={ell: k for ell in range(L)} if self.relu else None)
        self.eng = DecodeEngine(self.model, B, cap, polar, head_routers=hr, mlp_routers=mr, kv_ring=self.ring,
                                router_backend=args.router_backend,
                                concurrent_router={"on": True, "off": False}.get(args.concurrent_head_router),
                                union_handoff={"on": True, "off": False}.get(args.union_handoff),
                                tp=self.tp, kv_page_rows=args.kv_page_rows, kv_reserve=args.kv_reserve)
        self.eng.fill_random(ctx, seed=99 + (0 if tp_on else rank))
        self.dense = DecodeEngine(self.model, B, cap, SparsityPolicy(mode="dense"), caches=self.eng.caches,
                                  tp=self.tp)
        self.tokens_host = torch.randint(0, cfg.vocab, (B,), dtype=torch.int32,
                                         generator=torch.Generator().manual_seed(5)).pin_memory()
        self.graphs, self.graph_error = True, None
        self.eng.tokens.copy_(self.tokens_host)
        self.dense.tokens.copy_(self.tokens_host)
        try:
            self.eng.capture()
            self.dense.capture()
        except Exception as exc:  # reported in the JSON line (TP collectives that cannot be captured)
            if self.tp is None:
                raise
            self.graphs, self.graph_error = False, f"{type(exc).__name__}: {exc}"[:200]
            self.eng.graph = self.dense.graph = None

    def union_density(self):
        """Mean over layers of the device union size / D (after timing)."""
        if not self.relu:
            return None
        c = self.eng.union_counts.float()
        if self.tp is not None and self.tp.plan.world > 1:
            import torch.distributed as dist
            dist.all_reduce(c)  # each rank holds the count of its neuron shard
        return float(c.mean().item()) / self.cfg.ffn_dim


def replay(engine):
    def f():
        if engine.graph is not None:
            engine.graph.replay()
        else:
            engine.step_launches()
        engine._advance()
    return f


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PS_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0 with a gloo
    # group, so the TP path (sharding, graph capture with the p2p collective,
    # the JSON line) runs end to end on a one-GPU box; its timings are meaningless
    share = os.environ.get("PS_BENCH_SHARE_GPU") == "1" and world > 1
    if share:
        local = 0
    if world > 1:
        if share:
            dist.init_process_group("gloo", init_method="env://")
        else:
            dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tp_on = (world > 1 and not args.dp) or args.tp

    import paper_2505_14884_b200 as pb
    from paper_2505_14884_b200 import kernels as pk

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            fn()
        e.record()
        barrier()
        ms = s.elapsed_time(e)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    su = Setup(args, args.config, args.batch, args.ctx, dev, world, rank, tp_on, args.steps, args.warmup)
    cfg, B, eng, dense = su.cfg, su.B, su.eng, su.dense
    L, H, H_kv, d_h, D = cfg.layers, cfg.heads, cfg.kv_heads, cfg.head_dim, cfg.ffn_dim
    for _ in range(args.warmup):
        replay(dense)()
        replay(eng)()
    torch.cuda.synchronize()
    # every measurement starts from the same KV lengths (the caches are
    # shared and each step appends a row: later measurements would attend
    # over longer histories).  The dense baseline is the median of three
    # K-step measurements, one before and two after the polar one; the polar
    # value is one K-step measurement
    saved = [(c.lengths.clone(), c.host_lengths.copy()) for c in eng.caches]

    def reset_lengths():
        for c, (dl, hl) in zip(eng.caches, saved):
            c.lengths.copy_(dl)
            c.host_lengths[:] = hl
        torch.cuda.synchronize()

    reset_lengths()
    dense_ms = [timed(replay(dense), args.steps)]
    reset_lengths()
    with ClockSampler(local) as clk:
        ms_polar = timed(replay(eng), args.steps)
    clocks = clk.summary()
    union_density = su.union_density()

    # per-rank load (TP): selected KV groups and union neurons owned by this rank
    load = None
    if su.tp is not None:
        lo = su.tp.group_base
        sel = eng.sel[:, :su.k_h]
        heads_mine = float(((sel >= lo) & (sel < lo + su.Hkv_loc)).sum().item())
        neurons_mine = float(eng.union_counts.float().mean().item()) if su.relu else 0.0
        t = torch.tensor([heads_mine, neurons_mine], device=dev)
        if world > 1:
            allv = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(allv, t)
            allv = torch.stack(allv).cpu().numpy()
        else:
            allv = t[None].cpu().numpy()
        load = {"selected_kv_units_per_rank": allv[:, 0].tolist(),
                "union_neurons_per_rank": allv[:, 1].tolist(),
                "units_max_over_mean": float(allv[:, 0].max() / max(1e-9, allv[:, 0].mean())),
                "neurons_max_over_mean": float(allv[:, 1].max() / max(1e-9, allv[:, 1].mean())) if su.relu else None}

    # e2e: the public API (DecodeEngine.step) with host tokens in / next tokens out
    out_host = torch.empty(B, dtype=torch.int64).pin_memory()

    def e2e_step():
        eng.step(su.tokens_host)
        out_host.copy_(eng.next_tokens, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    reset_lengths()  # the same histories as the device-timed polar measurement
    for _ in range(2):
        e2e_step()
    barrier()
    t0 = time.perf_counter()
    ms_e2e = timed(e2e_step, args.steps)
    wall_e2e = (time.perf_counter() - t0) * 1e3

    for _ in range(2):
        reset_lengths()
        dense_ms.append(timed(replay(dense), args.steps))
    ms_dense = sorted(dense_ms)[1]

    # roofline: the SHA kernel alone on the same caches, one launch per layer
    qkv = eng.qkv
    k_loc = max(1, min(su.k_h, su.Hkv_loc))
    g = torch.Generator(device=dev).manual_seed(3)
    sel = torch.stack([torch.randperm(su.Hkv_loc, device=dev, generator=g)[:k_loc].sort().values
                       for _ in range(B)]).to(torch.int32)
    dq = su.H_loc * d_h
    out = torch.empty(B, dq, dtype=torch.bfloat16, device=dev)
    lens = [c.host_lengths.copy() for c in eng.caches]
    for c in eng.caches[:2]:
        pk.sha_decode_into(qkv, qkv.shape[1], c, sel, su.H_loc, eng.scale, out, dq,
                           max_len_hint=int(c.host_lengths.max()))
    torch.cuda.synchronize()
    sha_graph = torch.cuda.CUDAGraph()
    cap_stream = torch.cuda.Stream(device=dev)
    cap_stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap_stream):
        with torch.cuda.graph(sha_graph, stream=cap_stream):
            for c in eng.caches:
                pk.sha_decode_into(qkv, qkv.shape[1], c, sel, su.H_loc, eng.scale, out, dq,
                                   max_len_hint=int(c.host_lengths.max()))
    torch.cuda.current_stream().wait_stream(cap_stream)
    sha_graph.replay()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    sha_runs = []
    for _ in range(3):
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record(st)
        sha_graph.replay()
        e_ev.record(st)
        torch.cuda.synchronize()
        sha_runs.append(s_ev.elapsed_time(e_ev) / L)
    sha_ms = float(np.median(sha_runs))
    sha_bytes = float(np.mean([sha_algorithmic_bytes(l, k_loc, H // H_kv, d_h, B, su.H_loc) for l in lens]))
    hbm_peak, _, peak_kind = load_peaks()
    achieved = sha_bytes / (sha_ms * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic("sha_mma_kernel", args)

    # selective MLP kernels alone (UP + DOWN gathered GEMMs), one pair per
    # layer, over the union the polar step actually produced (last layer)
    mlp = None
    if su.relu:
        x2 = torch.randn(B, cfg.model_dim, device=dev).to(torch.bfloat16)
        y = torch.empty(B, cfg.model_dim, dtype=torch.float32, device=dev)
        cnt = eng.union_counts[L - 1:L].clone()
        S = int(cnt.item())
        idx = eng.union_idx.clone()
        hidden = eng.hidden
        pk.mlp_into(su.model.layers[0].mlp, x2, idx, cnt, hidden, y, expected=S)
        torch.cuda.synchronize()
        mlp_graph = torch.cuda.CUDAGraph()
        cap_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap_stream):
            with torch.cuda.graph(mlp_graph, stream=cap_stream):
                for lw in su.model.layers:
                    pk.mlp_into(lw.mlp, x2, idx, cnt, hidden, y, expected=S)
        torch.cuda.current_stream().wait_stream(cap_stream)
        mlp_graph.replay()
        torch.cuda.synchronize()
        runs = []
        for _ in range(3):
            s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_ev.record(st)
            mlp_graph.replay()
            e_ev.record(st)
            torch.cuda.synchronize()
            runs.append(s_ev.elapsed_time(e_ev) / L)
        mlp_ms = float(np.median(runs))
        mlp_bytes = 2 * S * cfg.model_dim * 2 + S * 2 + cfg.model_dim * 4 + 2 * B * cfg.model_dim * 2 + S * 4
        mlp = {"sparse_mlp_us_per_layer": mlp_ms * 1e3, "sparse_mlp_GBps": mlp_bytes / (mlp_ms * 1e-3) / 1e9,
               "sparse_mlp_frac": mlp_bytes / (mlp_ms * 1e-3) / 1e9 / hbm_peak, "union_size": S,
               "union_density": S / su.D_loc}
    n_launch = int(eng.launches_per_step)
    toks = (1 if su.tp is not None else world) * B * args.steps
    value = toks / (ms_polar * 1e-3)
    dense_value = toks / (ms_dense * 1e-3)
    S_meas = (union_density or 0.0) * D if su.relu else D
    main_ideal = ideal_ratio(cfg, B, args.ctx, args.rho, S_meas)
    setup_info = {"kv_storage_buffers": su.ring, "graph_captured": su.graphs, "graph_error": su.graph_error,
                  "kv_aliasing": ("none" if su.ring == L else f"K/V storage aliased over {su.ring} buffers"),
                  "hot_set": su.n_hot, "k_per_token": su.k_mlp,
                  "head_router": "concurrent branch" if su.eng.concurrent_router else "fused with the KV append",
                  "mlp_router": su.eng.router_backend, "o_proj": su.eng.o_backend,
                  "union_handoff": su.eng.union_handoff}
    del su, eng, dense, sha_graph
    torch.cuda.empty_cache()

    # further driver-observed points (N = 1 only; same recipe, shorter runs)
    extra = []
    if world == 1 and not args.no_extra and args.config == "opt-6.7b":
        points = [("opt-6.7b", 1), ("opt-6.7b", 16), ("opt-6.7b", 128), ("opt-6.7b", 256),
                  ("llama-3.1-8b", 64), ("llama-3.1-8b", 512)]
        ks, kw = min(args.steps, 8), 3
        for config, b in points:
            if b == args.batch and config == args.config:
                continue
            try:
                s2 = Setup(args, config, b, args.ctx, dev, world, rank, False, ks, kw)
                for _ in range(kw):
                    replay(s2.dense)()
                    replay(s2.eng)()
                mp = timed(replay(s2.eng), ks)
                md = timed(replay(s2.dense), ks)
                ud = s2.union_density()
                Sx = (ud or 0.0) * s2.cfg.ffn_dim if s2.relu else s2.cfg.ffn_dim
                extra.append({"config": config, "global_batch": b, "seq_len": args.ctx, "steps": ks, "warmup": kw,
                              "value": b * ks / (mp * 1e-3), "dense_value": b * ks / (md * 1e-3),
                              "speedup_vs_dense": md / mp, "union_density_measured": ud,
                              "ideal_ratio_byte_model": ideal_ratio(s2.cfg, b, args.ctx, args.rho, Sx),
                              "kv_storage_buffers": s2.ring})
                del s2
            except Exception as exc:  # report, never hide
                extra.append({"config": config, "global_batch": b, "error": f"{type(exc).__name__}: {exc}"[:200]})
            torch.cuda.empty_cache()

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cb = args.cpu_batch or B
            t_layer, kind, sample = reference_layer_sample(args, cfg, cb, reps=2, warm=1)
            info = cpu_info()
            cpu = {"value": cb / (t_layer * L), "unit": "tok/s", "cores": info["blas_threads"] or info["cpu_count"],
                   "kind": kind, "sample": sample, **info}
        line = {
            "metric": "decode_tokens_per_s", "value": value, "unit": "tok/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_polar / args.steps,
            "higher_is_better": True, "scaling": "strong" if tp_on and world > 1 else "weak", "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random-init weights N(0,0.02); N(0,1) KV history; hot/cold neuron router bias)",
            "config": workload_config(args, cfg, world=world, tp=tp_on),
            "setup": setup_info,
            "dense": {"value": dense_value, "ms_per_step": ms_dense / args.steps,
                      "ms_per_step_samples": [m / args.steps for m in dense_ms]},
            "speedup_vs_dense": value / dense_value,
            "ideal_ratio_byte_model": main_ideal,
            "union_density_measured": union_density,
            "tp_load": load,
            "e2e": {"value": toks / (ms_e2e * 1e-3), "unit": "tok/s", "h2d_bytes_per_step": B * 4,
                    "d2h_bytes_per_step": B * 8, "wall_ms_per_step": wall_e2e / args.steps,
                    "api": "DecodeEngine.step(host tokens) + D2H of next tokens + sync"},
            "gpu_launches": n_launch * args.steps,
            "roofline": {"bound": "hbm", "kernel": "sha_mma_kernel", "achieved": achieved, "peak": hbm_peak,
                         "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
                         "traffic_source": traffic_src, "peak_kind": peak_kind, "bytes_per_launch": sha_bytes,
                         "us_per_launch": sha_ms * 1e3},
            "kernels": mlp,
            "configs": extra,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
