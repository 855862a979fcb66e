"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: launches, mean and share per kernel."""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")) if r]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
t = defaultdict(list)
for r in rows[1:]:
    if len(r) != len(hdr):
        continue
    name = re.sub(r"<unnamed>::|\(anonymous namespace\)::", "", r[ki])
    name = re.sub(r"\(<unnamed>::KParams.*|\(KParams.*|\(.*\*.*\)$", "", name).strip()
    v = float(r[vi].replace(",", ""))
    name = re.sub(r"^void ", "", name)
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r[ui]]
    t[name].append(v * scale)  # -> us
tot = sum(sum(v) for v in t.values())
print(f"# ncu launch list {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("# gpu__time_duration.sum, --clock-control none; cold-cache serialised launches: compare shares, not absolutes\n")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:90]:90s} launches={len(v):4d} mean={sum(v) / len(v):9.1f} us  share={100 * sum(v) / tot:5.1f}%")
spmv = [v for k, v in t.items() if k.startswith("cb_spmv_kernel")]
zero = [v for k, v in t.items() if k.startswith("cb_zero_kernel")]
if spmv and zero:
    s, z = sum(map(sum, spmv)) / sum(map(len, spmv)), sum(map(sum, zero)) / sum(map(len, zero))
    print(f"\nSpMV kernel share of one step (zero + spmv): {100 * s / (s + z):.1f}%  (spmv {s:.1f} us, zero {z:.1f} us)")
