"""Top SASS lines by warp-stall samples per kernel from `ncu -i rep --page source --csv`.
usage: ncu -i X.ncu-rep --page source --csv | python tools/ncu_hot.py [N]"""
import csv
import sys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 15
lines = sys.stdin.read().split("\n")
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
for b in blocks:
    print(b[0][:110])
    r = list(csv.reader(b[1:]))
    h = r[0]
    rows = [dict(zip(h, x)) for x in r[1:] if len(x) == len(h)]
    tot = sum(int(x["Instructions Executed"] or 0) for x in rows)
    samp = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in rows)
    print(f"  warp-instr {tot}  samples {samp}  sass lines {len(rows)}")
    rows.sort(key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))
    for x in rows[:n]:
        reasons = sorted(((k, int(v or 0)) for k, v in x.items() if k.startswith("stall_") and "Not Issued" not in k),
                         key=lambda kv: -kv[1])[:2]
        print(f"  {x['Address'][-5:]} {x['Instructions Executed']:>7} {x['Warp Stall Sampling (All Samples)']:>5} "
              f"{x['Source'].strip()[:60]:60s} {reasons}")
