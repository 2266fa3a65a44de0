"""Brief of one kernel in an ncu report: duration, DRAM, pipes, L1 wavefronts / writeback,
occupancy, warp stall breakdown and the hottest SASS lines. usage: ncu_brief.py REPORT [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "inst_executed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sectors.sum", "l1tex__t_requests.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size"]
for k, x in zip(h, v):
    if k in want:
        print(f"{k:70s} {x}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hh = src[1]
ix = {k: i for i, k in enumerate(hh)}
stalls = collections.Counter()
lines = []
for r in src[2:]:
    if len(r) < len(hh):
        continue
    for k in hh:
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                stalls[k] += int(float(r[ix[k]] or 0))
            except ValueError:
                pass
    try:
        lines.append((int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Instructions Executed"]],
                      r[ix["Source"]].strip()))
    except ValueError:
        continue
tot = sum(stalls.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {100 * c / tot:.1f}%" for k, c in stalls.most_common(8)))
ops = collections.Counter()
for s, ie, t in lines:
    w = t.split()
    op = w[1] if w and w[0].startswith("@") and len(w) > 1 else (w[0] if w else "")
    ops[op] += int(ie or 0)
print("ops:", ops.most_common(14))
for s, ie, t in sorted(lines, reverse=True)[:top]:
    print(f"{s:6d} {ie:>10s}  {t}")
