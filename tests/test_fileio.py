"""On-disk formats: this package's readers vs files the
REFERENCE's writers produced (tests/golden/make_fileio_fixtures.py), byte
for byte, plus the reference's error behaviour (fileio.py:38-71)."""

import json
import os

import numpy as np
import pytest

from paper_2505_14884_b200 import fileio as F
from paper_2505_14884_b200.exceptions import ConfigurationError

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fileio")


@pytest.fixture(scope="module")
def expected():
    return np.load(os.path.join(G, "expected.npz"))


@pytest.mark.parametrize("tag,kvh", [("relu", 2), ("swiglu", 1)])
def test_read_model_matches_reference_arrays(expected, tag, kvh):
    host = F.read_model(os.path.join(G, f"model_{tag}.pswt"))
    cfg = host["config"]
    assert (cfg.layers, cfg.model_dim, cfg.ffn_dim, cfg.heads, cfg.kv_heads, cfg.vocab, cfg.max_seq) == \
        (2, 64, 128, 2, kvh, 40, 12)
    assert cfg.activation == tag
    for name in ("embed", "pos_embed", "unembed", "lnf_g", "lnf_b"):
        assert np.array_equal(host[name], expected[f"{tag}_{name}"]), name
    for ell, lw in enumerate(host["layers"]):
        for name in F.LAYER_BLOCKS:
            assert np.array_equal(lw[name], expected[f"{tag}_l{ell}_{name}"]), (ell, name)
        if tag == "swiglu":
            assert np.array_equal(lw["mlp_w3"], expected[f"{tag}_l{ell}_mlp_w3"])
        else:
            assert lw["mlp_w3"] is None


@pytest.mark.parametrize("tag", ["relu", "swiglu"])
def test_write_model_is_byte_identical(tmp_path, tag):
    src = os.path.join(G, f"model_{tag}.pswt")
    out = tmp_path / "m.pswt"
    F.write_model(F.read_model(src), out)
    assert out.read_bytes() == open(src, "rb").read()


@pytest.mark.parametrize("kind,fname,prefix", [("mlp", "router_mlp.psrt", "mlp_router_"),
                                                ("head", "router_head.psrt", "head_router_")])
def test_routers_round_trip(tmp_path, expected, kind, fname, prefix):
    src = os.path.join(G, fname)
    got_kind, w = F.read_router(src)
    assert got_kind == kind
    for k, v in w.items():
        assert np.array_equal(v, expected[prefix + k]), k
    out = tmp_path / "r.psrt"
    F.write_router(kind, w, out)
    assert out.read_bytes() == open(src, "rb").read()


def test_k_table_and_run_config(tmp_path):
    kt = F.LayerKTable.load(os.path.join(G, "k_table.tsv"))
    assert kt.rows == ((0, 20, 0.95), (1, 24, 0.9))
    assert kt.k_for(1) == 24
    with pytest.raises(ConfigurationError):
        kt.k_for(2)
    kt.save(tmp_path / "k.tsv")
    assert (tmp_path / "k.tsv").read_text() == open(os.path.join(G, "k_table.tsv")).read()
    with pytest.raises(ValueError):
        F.LayerKTable([(0, 0, 1.0)])
    with pytest.raises(ValueError):
        F.LayerKTable([(0, 3, 1.0), (0, 4, 1.0)])
    cfg, pol = F.load_run_config(os.path.join(G, "run_config.json"))
    assert (cfg.model_dim, cfg.heads, cfg.activation) == (64, 2, "relu")
    assert pol.mode == "polar" and pol.head_density == 0.5 and pol.layer0_dense_attention
    assert pol.k_for(0) == 20 and pol.k_for(1) == 24
    doc = json.load(open(os.path.join(G, "run_config.json")))
    doc["policy"]["head_ranking"] = "oracle"
    p = tmp_path / "rc.json"
    p.write_text(json.dumps(doc))
    with pytest.raises(ConfigurationError):
        F.load_run_config(p)
    p.write_text(json.dumps({"policy": {}}))
    with pytest.raises(ValueError):
        F.load_run_config(p)


def test_token_stream(tmp_path):
    toks = F.load_token_stream(os.path.join(G, "tokens.txt"))
    assert toks.dtype == np.int64 and toks.tolist() == [3, 1, 4, 1, 5, 9, 2, 6]
    F.save_token_stream(toks, tmp_path / "t.txt")
    assert (tmp_path / "t.txt").read_text() == open(os.path.join(G, "tokens.txt")).read()
    (tmp_path / "bad.txt").write_text("1\n-2\n")
    with pytest.raises(ValueError):
        F.load_token_stream(tmp_path / "bad.txt")
    with pytest.raises(ValueError):
        F.save_token_stream(np.zeros((2, 2), np.int64), tmp_path / "x.txt")


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXXX" + b[4:], "bad magic"),
    (lambda b: b[:4] + (2).to_bytes(4, "little") + b[8:], "unsupported version"),
    (lambda b: b[:-4], "truncated"),
    (lambda b: b + b"\0", "trailing bytes"),
])
def test_format_errors(tmp_path, mutate, msg):
    for fname, reader in (("model_relu.pswt", F.read_model), ("router_mlp.psrt", F.read_router)):
        p = tmp_path / fname
        p.write_bytes(mutate(open(os.path.join(G, fname), "rb").read()))
        with pytest.raises(ValueError, match=msg):
            reader(p)
    p = tmp_path / "kind.psrt"
    b = bytearray(open(os.path.join(G, "router_head.psrt"), "rb").read())
    b[8] = 7
    p.write_bytes(bytes(b))
    with pytest.raises(ValueError, match="unknown router kind"):
        F.read_router(p)
