"""Summarise tools/gpu_ab_lib.sh logs: polar / dense ms per step and the ratio."""
import glob
import json

for f in sorted(glob.glob("gpurun_out/ab_*_*.log")):
    if "pytest" in f:
        continue
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print(f, "no result")
        continue
    d = json.loads(lines[-1])
    print(f"{f:42s} polar {d['ms_per_step']:.4f} ms  dense {d['dense']['ms_per_step']:.4f} ms  "
          f"ratio {d['speedup_vs_dense']:.4f}  e2e {d['e2e']['value']:.1f}")
