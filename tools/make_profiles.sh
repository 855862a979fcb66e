#!/bin/bash
# Summarise the gpurun_out/ captures of tools/gpu_profiles.sh + tools/ncu_metrics.sh into profiles/<tag>_*
# (run here, on the CPU box, after the GPU call):  bash tools/make_profiles.sh r2
tag=${1:-r2}
set -e
for c in clustered rmat laplace uniform; do
  rep=gpurun_out/prof_$c.ncu-rep
  [ -f $rep ] || continue
  {
    echo "# ncu --set full --clock-control none, one cb_spmv_kernel launch, BASELINE $c fp64 (tools/prof_kernel.py; tools/gpu_profiles.sh)"
    python tools/ncu_summary.py $rep
    echo; echo "# per source line (tools/src_lines.py: instructions executed / warp-stall samples)"
    ncu -i $rep --page source --csv --print-source cuda,sass > /tmp/_src.csv 2>/dev/null
    python tools/src_lines.py /tmp/_src.csv 25
    echo; echo "# stall reasons (tools/sass_hot.py)"
    ncu -i $rep --page source --csv --print-source sass > /tmp/_sass.csv 2>/dev/null
    python tools/sass_hot.py /tmp/_sass.csv 12
  } > profiles/${tag}_ncu_$c.txt
done
cp gpurun_out/launches_bench.csv profiles/${tag}_launches_bench.csv
python tools/launch_summary.py gpurun_out/launches_bench.csv "(bench.py --steps 5 --warmup 3, clustered fp64)" > profiles/${tag}_launches_summary.txt
python tools/ncu_metrics_summary.py gpurun_out > profiles/${tag}_ncu_metrics.txt
python - <<PY
import json, subprocess, csv
out = {}
for c in ("clustered", "rmat", "laplace"):  # uniform: all panels, tools/ncu_uniform_traffic.sh
    raw = subprocess.run(["ncu", "-i", f"gpurun_out/prof_{c}.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h, u, v = rows[0], rows[1], rows[2]
    def g(k):
        i = h.index(k)
        return float(v[i].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[i]]
    out[f"{c}_f64"] = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
import os
if os.path.exists("gpurun_out/ncu_uniform_traffic.csv"):  # one whole SpMV = P panel launches
    rows = list(csv.reader(l for l in open("gpurun_out/ncu_uniform_traffic.csv") if l.startswith('"')))
    h = rows[0]
    mi, ui, vi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out["uniform_f64"] = sum(float(r[vi].replace(",", "")) * scale[r[ui]] for r in rows[1:]
                             if r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(out)
PY
