#!/usr/bin/env python3
"""Top SASS lines by warp-stall samples from `ncu --page source --csv` output.
usage: ncu -i rep --page source --csv --kernel-name regex:K --launch-count 1 > x.csv; python tools/ncu_hot.py x.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
i_s = hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows if len(r) > i_s and r[i_s].isdigit()]
tot = sum(int(r[i_s]) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -int(r[i_s]))[:n]:
    print(f"{int(r[i_s]):6d} {100.0 * int(r[i_s]) / max(tot, 1):5.1f}%  {r[0][-5:]}  {r[1][:100]}")

stall = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = {hdr[i]: sum(int(r[i]) for r in data if r[i].isdigit()) for i in stall}
print("stall totals:", ", ".join(f"{k[6:]}={v}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v))
