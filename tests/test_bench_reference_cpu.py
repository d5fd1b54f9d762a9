"""bench.py's reference arm on the host (no GPU needed): the unmodified
reference engine from baseline/_ref on the tiny config prints one contract
line with impl = "reference", its own cpu_baseline and a zero-copy e2e; and
under torchrun-style env with RANK != 0 the arm exits 0 without output.
Skipped when the reference has not been installed into baseline/_ref."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "sparsedecode")):
    pytest.skip("reference not installed in baseline/_ref", allow_module_level=True)


def _run(env_extra=None, *args):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, cwd=ROOT, env=env)


def test_reference_arm_line_on_cpu():
    out = _run(None, "--impl", "reference", "--config", "tiny", "--batch", "8", "--ctx", "200", "--steps", "1",
               "--warmup", "1")
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["value"] > 0 and j["unit"] == "tok/s"
    assert j["metric"] == "decode_tokens_per_s" and j["higher_is_better"] is True
    assert j["e2e"]["value"] == j["value"]
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0
    cb = j["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] == j["value"] and cb["cores"] >= 1 and cb["sample"]


def test_reference_arm_other_ranks_exit_quietly():
    out = _run({"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"}, "--impl", "reference", "--config", "tiny",
               "--gpus", "2", "--steps", "1", "--warmup", "1")
    assert out.returncode == 0, out.stderr[-2000:]
    assert not [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
