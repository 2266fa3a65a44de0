"""Per-CUDA-source-line warp-stall samples from `ncu -i rep --page source --csv --print-source cuda,sass`
(pick one launch with --launch-skip/--launch-count). usage: ... | python tools/ncu_lines.py [N]"""
import csv
import sys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rows = list(csv.reader(sys.stdin))
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
out = []


def num(v):
    try:
        return int(float(v))
    except ValueError:
        return 0


for r in rows:
    if len(r) != len(hdr) or r[0] == "Line No":
        continue
    if r[0]:  # CUDA line row (aggregated over its SASS)
        out.append([r[0], r[1].strip()[:80], num(r[si]), num(r[ie])])
tot = sum(x[2] for x in out) or 1
for x in sorted(out, key=lambda x: -x[2])[:n]:
    print(f"{x[0]:>5} {x[2]:6d} {100 * x[2] / tot:5.1f}% {x[3]:8d}  {x[1]}")
