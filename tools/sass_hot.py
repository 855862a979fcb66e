"""Summarise an ncu --page source --print-source sass CSV: top instructions by stall samples."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
tot_s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
tot_i = sum(int(d["Instructions Executed"] or 0) for d in data)
print("instructions executed", tot_i, "samples", tot_s)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = Counter()
for d in data:
    for c in stall_cols:
        agg[c] += int(d[c] or 0)
print("stalls:", ", ".join(f"{k[6:]}={v*100/max(1,tot_s):.1f}%" for k, v in agg.most_common(8)))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
data.sort(key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))
for d in data[:top]:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    st = Counter({c[6:]: int(d[c] or 0) for c in stall_cols}).most_common(2)
    print(f"{d['Address']:>6} {s*100/max(1,tot_s):5.1f}% ex={d['Instructions Executed']:>10} {d['Source'][:70]:70} {st}")
