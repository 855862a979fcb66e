"""Per-CUDA-line totals from `ncu -i rep --page source --csv --print-source cuda,sass`:
instructions executed and stall samples attributed to each kernels.cu line (top N)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ins = defaultdict(int)
smp = defaultdict(int)
text = {}
cur = None
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        continue
    if not r[0].isdigit():  # SASS rows and headers; the line rows carry the totals
        continue
    cur = int(r[0])
    text[cur] = r[1]
    v = r[hdr.index("Instructions Executed")]
    ins[cur] += int(v) if v.isdigit() else 0
    v = r[hdr.index("Warp Stall Sampling (All Samples)")]
    smp[cur] += int(v) if v.isdigit() else 0
ti, ts = sum(ins.values()), sum(smp.values())
print(f"instructions {ti}  samples {ts}")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for ln in sorted(ins, key=lambda k: -ins[k])[:top]:
    print(f"{ln:5d} ins {ins[ln]*100/ti:5.1f}%  smp {smp[ln]*100/max(ts,1):5.1f}%  {text.get(ln, '')[:90]}")
