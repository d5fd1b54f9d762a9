"""Key metrics of every kernel in one or more `ncu --set full` reports, as
CSV (one row per profiled launch): duration, DRAM bytes read / written,
DRAM throughput, tensor-pipe activity, warps active, registers, grid.

    python tools/ncu_summary.py gpurun_out/r02_full_sha.ncu-rep ... > profiles/r02_ncu_kernels.csv
"""
import csv
import io
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_us",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_rt_pct",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"duration_us": ("nsecond", 1e-3, "usecond", 1.0, "msecond", 1e3),
         "dram_read_MB": ("byte", 1e-6, "Kbyte", 1e-3, "Mbyte", 1.0, "Gbyte", 1e3),
         "dram_write_MB": ("byte", 1e-6, "Kbyte", 1e-3, "Mbyte", 1.0, "Gbyte", 1e3)}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"report": path.split("/")[-1], "kernel": row[hdr.index("Kernel Name")][:60]}
        for m, name in WANT.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = row[i].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                d[name] = v
                continue
            if name in SCALE:
                sc = SCALE[name]
                u = units[i]
                for k in range(0, len(sc), 2):
                    if sc[k] == u:
                        x *= sc[k + 1]
            d[name] = round(x, 3)
        res.append(d)
    return res


def main():
    allr = []
    for p in sys.argv[1:]:
        allr += rows(p)
    cols = ["report", "kernel"] + [v for v in WANT.values() if any(v in r for r in allr)]
    w = csv.DictWriter(sys.stdout, fieldnames=cols, extrasaction="ignore")
    w.writeheader()
    for r in allr:
        w.writerow(r)


if __name__ == "__main__":
    main()
