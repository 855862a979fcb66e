"""Summarise tools/ncu_metrics.sh CSVs into one table (profiles/r1_ncu_metrics.txt)."""
import csv
import glob
import io
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
NNZ = {"clustered": 407534668, "rmat": 131159768, "laplace": 4996000}
print("# ncu --metrics (SURVEY §8(d)), one cb_spmv_kernel launch, --clock-control none; tools/ncu_metrics.sh")
print("# cold = --cache-control all (caches flushed before the launch); warm = --cache-control none (3rd launch)")
for f in sorted(glob.glob(os.path.join(d, "ncu_metrics_*.csv"))):
    name = os.path.basename(f)[len("ncu_metrics_"):-4]
    txt = open(f).read()
    i = txt.find('"ID"')
    if i < 0:
        print(name, "no data")
        continue
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    v = {r["Metric Name"]: (r["Metric Value"], r["Metric Unit"]) for r in rows}
    cfg = name.split("_")[0]
    def g(k):
        return float(v[k][0].replace(",", "")) if k in v else float("nan")
    red = g("lts__t_requests_op_red.sum")
    print(f"\n[{name}]")
    for k in sorted(v):
        print(f"  {k:55s} {v[k][0]:>18s} {v[k][1]}")
    if cfg in NNZ:
        print(f"  RED requests per nnz: {red / NNZ[cfg]:.3f}   gather sectors per nnz: "
              f"{g('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum') / NNZ[cfg]:.3f}")
