"""One-line-per-kernel summary of ncu --set full reports (read here, no GPU)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe % (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "fp64 pipe % (elapsed)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "cycles/issued inst"),
]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?").split("(")[0]
        vals = []
        for k, label in KEYS:
            if k in d and d[k] != "":
                vals.append(f"{label}={d[k]} {u.get(k, '')}".strip())
        res.append(f"{name}: " + "; ".join(vals))
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"## {p}")
        for line in summarize(p):
            print("  " + line)
