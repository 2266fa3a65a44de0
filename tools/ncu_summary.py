"""Key metrics from ncu reports (one kernel each) as a markdown table.
usage: python tools/ncu_summary.py name=path.ncu-rep ..."""
import csv
import io
import subprocess
import sys

WANT = [
    ("duration (us)", "gpu__time_duration.sum", 1e-3),
    ("DMMA issue (% of peak)", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
    ("DRAM read (MB)", "dram__bytes_read.sum", 1e-6),
    ("DRAM write (MB)", "dram__bytes_write.sum", 1e-6),
    ("DRAM throughput (% of peak)", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("shared wavefronts (% of peak)", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1),
    ("shared bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("registers / thread", "launch__registers_per_thread", 1),
    ("block", "launch__block_size", 1),
    ("grid", "launch__grid_size", 1),
    ("dyn smem (KB)", "launch__shared_mem_per_block_dynamic", 1),
]
cols = []
for arg in sys.argv[1:]:
    name, path = arg.split("=", 1)
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    col = []
    for label, key, scale in WANT:
        v = d.get(key, "")
        try:
            x = float(v.replace(",", ""))
            unit = u.get(key, "")
            if key == "gpu__time_duration.sum":
                x = x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
            elif key.startswith("dram__bytes"):
                x = x * {"byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0, "Gbyte": 1e3, "GB": 1e3}.get(unit, 1e-6)
            else:
                x = x * scale
            col.append(f"{x:.4g}")
        except ValueError:
            col.append(v or "-")
    cols.append((name, col))
print("| metric | " + " | ".join(n for n, _ in cols) + " |")
print("|---|" + "---|" * len(cols))
for i, (label, _, _) in enumerate(WANT):
    print(f"| {label} | " + " | ".join(c[i] for _, c in cols) + " |")
