"""The reference's on-disk formats (sparsedecode/fileio.py:1-287) read into
this package's device objects -- SURVEY.md §8(f) row f4: routers trained and
k-tables calibrated offline by the reference CPU code drive the GPU path.

Little-endian, 4-byte magic + u32 version 1 (fileio.py:1-17):

* ``PSWT`` model weights (save_model / load_model, fileio.py:159-218): u32
  length-prefixed JSON ``TransformerConfig``, then f32 blocks -- embed
  (vocab, d), pos_embed (max_seq, d), per layer ln1_g, ln1_b, w_q, b_q, w_k,
  b_k, w_v, b_v, w_o, b_o, ln2_g, ln2_b, mlp_w1 (d, D), mlp_b1, mlp_w2 (d, D),
  mlp_b2 [, mlp_w3 for SwiGLU], then lnf_g, lnf_b, unembed (d, vocab);
* ``PSRT`` router checkpoint (save_router / load_router, fileio.py:80-117):
  kind byte (0 neuron router: u32 d, hidden, D; w_in, b_in, w_out, b_out --
  1 head router: u32 d, heads; w, b), f32 blocks;
* k-table TSV ``layer<TAB>k<TAB>recall`` (calibration.py:73-89), token
  streams (one id per line, fileio.py:220-240), run configs (JSON with
  ``model`` and ``policy`` objects, fileio.py:243-287).

The readers return host arrays (``read_*``, numpy, CPU-testable) or device
objects (``load_*``: ``DeviceModel`` neuron-major bf16, ``HeadRouter`` /
``MlpRouter``).  Errors follow the reference: ``ValueError`` for bad magic,
version, truncation or trailing bytes; ``ConfigurationError`` from
``LayerKTable.k_for`` for a layer without a budget.
"""

from __future__ import annotations

import json
import struct

import numpy as np

from .exceptions import ConfigurationError
from .model import TransformerConfig

FORMAT_VERSION = 1

# per-layer block order of a PSWT file (fileio.py:197-202)
LAYER_BLOCKS = ("ln1_g", "ln1_b", "w_q", "b_q", "w_k", "b_k", "w_v", "b_v", "w_o", "b_o",
                "ln2_g", "ln2_b", "mlp_w1", "mlp_b1", "mlp_w2", "mlp_b2")


class _Cursor:
    """Bounds-checked little-endian reads over one file's bytes."""

    def __init__(self, data: bytes, path):
        self.data, self.pos, self.path = data, 0, path

    def bytes(self, n: int) -> bytes:
        end = self.pos + n
        if n < 0 or end > len(self.data):
            raise ValueError(f"{self.path}: truncated file")
        out = self.data[self.pos:end]
        self.pos = end
        return out

    def u8(self) -> int:
        return self.bytes(1)[0]

    def u32(self) -> int:
        return struct.unpack("<I", self.bytes(4))[0]

    def f32(self, shape) -> np.ndarray:
        n = int(np.prod(shape))
        return np.frombuffer(self.bytes(4 * n), dtype="<f4").astype(np.float32).reshape(shape)

    def header(self, magic: bytes) -> None:
        got = self.bytes(4)
        if got != magic:
            raise ValueError(f"{self.path}: bad magic {got!r}, expected {magic!r}")
        ver = self.u32()
        if ver != FORMAT_VERSION:
            raise ValueError(f"{self.path}: unsupported version {ver}")

    def end(self) -> None:
        if self.pos != len(self.data):
            raise ValueError(f"{self.path}: trailing bytes after payload")


def _read(path) -> bytes:
    with open(path, "rb") as f:
        return f.read()


def _f32(a) -> bytes:
    return np.ascontiguousarray(a, dtype="<f4").tobytes()


# ---------------------------------------------------------------------- config
def config_from_dict(d: dict) -> TransformerConfig:
    """TransformerConfig.from_dict (model.py:65-67): every field required."""
    names = ("layers", "model_dim", "ffn_dim", "heads", "kv_heads", "vocab", "max_seq", "activation")
    missing = [n for n in names if n not in d]
    if missing:
        raise KeyError(missing[0])
    return TransformerConfig(**{n: d[n] for n in names})


# ---------------------------------------------------------------------- PSWT
def read_model(path) -> dict:
    """PSWT -> host dict in the oracle's ``random_model`` layout (f32 numpy,
    input-major weights as stored) plus ``config`` (a TransformerConfig)."""
    r = _Cursor(_read(path), path)
    r.header(b"PSWT")
    cfg = config_from_dict(json.loads(r.bytes(r.u32()).decode()))
    d, D, dk = cfg.model_dim, cfg.ffn_dim, cfg.kv_dim
    shapes = {"ln1_g": (d,), "ln1_b": (d,), "w_q": (d, d), "b_q": (d,), "w_k": (d, dk), "b_k": (dk,),
              "w_v": (d, dk), "b_v": (dk,), "w_o": (d, d), "b_o": (d,), "ln2_g": (d,), "ln2_b": (d,),
              "mlp_w1": (d, D), "mlp_b1": (D,), "mlp_w2": (d, D), "mlp_b2": (d,), "mlp_w3": (d, D)}
    embed = r.f32((cfg.vocab, d))
    pos = r.f32((cfg.max_seq, d))
    layers = []
    for _ in range(cfg.layers):
        lw = {n: r.f32(shapes[n]) for n in LAYER_BLOCKS}
        lw["mlp_w3"] = r.f32(shapes["mlp_w3"]) if cfg.activation == "swiglu" else None
        layers.append(lw)
    lnf_g, lnf_b = r.f32((d,)), r.f32((d,))
    unembed = r.f32((d, cfg.vocab))
    r.end()
    return {"config": cfg, "layers": layers, "embed": embed, "pos_embed": pos, "unembed": unembed,
            "lnf_g": lnf_g, "lnf_b": lnf_b}


def write_model(host: dict, path) -> None:
    """Host dict (``read_model`` / ``random_model`` layout) -> PSWT, byte-for-
    byte the reference's save_model (fileio.py:159-178)."""
    cfg = host["config"]
    cfg = cfg if isinstance(cfg, TransformerConfig) else config_from_dict(cfg)
    cj = json.dumps(cfg.to_dict()).encode()
    parts = [b"PSWT", struct.pack("<I", FORMAT_VERSION), struct.pack("<I", len(cj)), cj,
             _f32(host["embed"]), _f32(host["pos_embed"])]
    for lw in host["layers"]:
        parts += [_f32(lw[n]) for n in LAYER_BLOCKS]
        if cfg.activation == "swiglu":
            parts.append(_f32(lw["mlp_w3"]))
    parts += [_f32(host["lnf_g"]), _f32(host["lnf_b"]), _f32(host["unembed"])]
    with open(path, "wb") as f:
        f.write(b"".join(parts))


def load_model(path, device="cuda"):
    """PSWT -> DeviceModel (neuron-major bf16 weights, f32 norms/biases)."""
    from .model import DeviceModel

    host = read_model(path)
    return DeviceModel.from_host(host["config"], host, device=device)


# ---------------------------------------------------------------------- PSRT
def read_router(path) -> tuple:
    """PSRT -> ("mlp" | "head", weights dict in declaration order)."""
    r = _Cursor(_read(path), path)
    r.header(b"PSRT")
    kind = r.u8()
    if kind == 0:
        d, h, D = r.u32(), r.u32(), r.u32()
        shapes = {"w_in": (d, h), "b_in": (h,), "w_out": (h, D), "b_out": (D,)}
        name = "mlp"
    elif kind == 1:
        d, H = r.u32(), r.u32()
        shapes = {"w": (d, H), "b": (H,)}
        name = "head"
    else:
        raise ValueError(f"{path}: unknown router kind {kind}")
    w = {k: r.f32(s) for k, s in shapes.items()}
    r.end()
    return name, w


def write_router(kind: str, weights: dict, path) -> None:
    """(kind, weights) -> PSRT, byte-for-byte the reference's save_router."""
    parts = [b"PSRT", struct.pack("<I", FORMAT_VERSION)]
    if kind == "mlp":
        d, h = np.shape(weights["w_in"])
        D = np.shape(weights["w_out"])[1]
        parts += [struct.pack("<B", 0), struct.pack("<III", d, h, D)]
        order = ("w_in", "b_in", "w_out", "b_out")
    elif kind == "head":
        d, H = np.shape(weights["w"])
        parts += [struct.pack("<B", 1), struct.pack("<II", d, H)]
        order = ("w", "b")
    else:
        raise TypeError(f"unknown router kind {kind!r}")
    parts += [_f32(weights[k]) for k in order]
    with open(path, "wb") as f:
        f.write(b"".join(parts))


def load_router(path, device=None):
    """PSRT -> HeadRouter | MlpRouter on the device."""
    from .routers import HeadRouter, MlpRouter

    kind, w = read_router(path)
    if kind == "mlp":
        return MlpRouter.from_weights(w["w_in"], w["b_in"], w["w_out"], w["b_out"], device=device)
    return HeadRouter.from_weights(w["w"], w["b"], device=device)


# ---------------------------------------------------------------------- k-table
class LayerKTable:
    """Calibrated per-layer neuron budgets (calibration.py:47-89)."""

    def __init__(self, rows):
        rows = tuple((int(ell), int(k), float(rec)) for ell, k, rec in rows)
        for ell, k, _ in rows:
            if k < 1:
                raise ValueError(f"layer {ell}: k must be >= 1, got {k}")
        if len({r[0] for r in rows}) != len(rows):
            raise ValueError("duplicate layer index in k table")
        self.rows = rows

    def k_for(self, layer: int) -> int:
        for ell, k, _ in self.rows:
            if ell == layer:
                return k
        raise ConfigurationError(f"no calibrated k for layer {layer}")

    def __len__(self) -> int:
        return len(self.rows)

    def save(self, path) -> None:
        with open(path, "w") as f:
            for ell, k, rec in self.rows:
                f.write(f"{ell}\t{k}\t{rec:.6f}\n")

    @classmethod
    def load(cls, path) -> "LayerKTable":
        rows = []
        with open(path) as f:
            for line in f:
                line = line.strip()
                if not line or line.startswith("#"):
                    continue
                ell, k, rec = line.split("\t")
                rows.append((int(ell), int(k), float(rec)))
        return cls(rows)


# ---------------------------------------------------------------------- tokens / run config
def load_token_stream(path) -> np.ndarray:
    """Newline-delimited non-negative ids (fileio.py:231-240) -> int64."""
    vals = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line:
                vals.append(int(line))
    arr = np.array(vals, dtype=np.int64)
    if arr.size and arr.min() < 0:
        raise ValueError(f"{path}: token ids must be non-negative")
    return arr


def save_token_stream(tokens, path) -> None:
    tokens = np.asarray(tokens)
    if tokens.ndim != 1:
        raise ValueError("token stream must be 1-dimensional")
    if tokens.size and int(tokens.min()) < 0:
        raise ValueError("token ids must be non-negative")
    with open(path, "w") as f:
        f.writelines(f"{int(t)}\n" for t in tokens)


def policy_from_dict(doc: dict):
    """fileio.py:255-268 -> engine.SparsityPolicy.  ``mlp_k_table`` may be a
    path to a k-table TSV or inline rows.  Only router head ranking is on the
    decode hot path; "oracle" ranking is rejected."""
    from .engine import SparsityPolicy

    table = doc.get("mlp_k_table")
    if isinstance(table, str):
        table = LayerKTable.load(table)
    elif table is not None:
        table = LayerKTable(table)
    ranking = doc.get("head_ranking", "router")
    if ranking != "router":
        raise ConfigurationError(f"head_ranking {ranking!r} is a study tool, not on the decode path")
    return SparsityPolicy(mode=doc.get("mode", "dense"), mlp_k_table=table,
                          head_density=float(doc.get("head_density", 1.0)),
                          layer0_dense_attention=bool(doc.get("layer0_dense_attention", True)))


def load_run_config(path) -> tuple:
    """Run config JSON (fileio.py:278-287) -> (TransformerConfig, SparsityPolicy)."""
    with open(path) as f:
        doc = json.load(f)
    if "model" not in doc:
        raise ValueError(f"{path}: missing 'model' object")
    return config_from_dict(doc["model"]), policy_from_dict(doc.get("policy", {}))
