"""Key metrics of an ncu report (details page) as compact text."""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Active Warps Per SM", "Registers Per Thread", "Eligible Warps Per Scheduler",
        "No Eligible", "Executed Instructions", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Mem Busy", "Max Bandwidth", "Warp Cycles Per Issued Instruction"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(out.splitlines())
hdr = next(r)
for row in r:
    d = dict(zip(hdr, row))
    if d.get("Metric Name") in KEYS:
        print(f"  {d['Metric Name']:40s} {d['Metric Value']:>16s} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "lts__t_request_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "gpu__time_duration.sum", "lts__t_requests_op_red.sum",
        "lts__t_sectors_op_red.sum", "smsp__inst_executed.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]
for k in want:
    for i, name in enumerate(h):
        if name == k:
            print(f"  {k:40s} {v[i]:>16s} {u[i]}")
