"""Per-kernel duration and DRAM traffic from `ncu --set full` reports ->
profiles/<round>_ncu_traffic.json (bench.py reads roofline.traffic from it).

    python tools/ncu_traffic.py out.json gpurun_out/full_sha.ncu-rep gpurun_out/full_sel_gg.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "msecond": 1e-3, "second": 1.0}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    lines = out.splitlines()
    r = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, units, data = r[0], r[1], r[2:]
    for d in data:
        rec = {}
        for h, u, v in zip(hdr, units, d):
            rec[h] = (v, u)
        yield rec


def val(rec, name):
    v, u = rec[name]
    return float(v.replace(",", "")) * UNITS.get(u, 1.0)


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    ks = []
    for rep in reps:
        for rec in rows(rep):
            name = rec["Kernel Name"][0]
            base = name.split("(")[0].replace("void ", "")
            for pre in ("ps::<unnamed>::", "ps::(anonymous namespace)::", "<unnamed>::", "unnamed>::"):
                base = base.replace(pre, "")
            ks.append({"kernel": base,
                       "duration_s": val(rec, "gpu__time_duration.sum"),
                       "dram_read_bytes": val(rec, "dram__bytes_read.sum"),
                       "dram_write_bytes": val(rec, "dram__bytes_write.sum"),
                       "grid": rec.get("launch__grid_size", ("", ""))[0]})
    doc = {"source": "ncu --set full --clock-control none (cold cache, serialized); one launch each, OPT-6.7B "
                     "B=64 ctx 1920 rho=0.5 |S|/D=0.5 (tools/gpu_profiles.sh)", "kernels": ks}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    for k in ks:
        print(f"{k['kernel'][:50]:50s} {k['duration_s'] * 1e6:8.1f} us  read {k['dram_read_bytes'] / 1e6:9.1f} MB")


if __name__ == "__main__":
    main()
