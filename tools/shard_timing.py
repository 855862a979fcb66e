"""Single-GPU projection of the row-sharded scaling run: for P = 1, 2, 4, 8, build
every rank's nnz-balanced row shard (bench.py's cut, dist.shard_bounds) and time its SpMV alone
(zero + kernel, CUDA events, back-to-back).  Aggregate GFLOP/s = 2 nnz / max-shard time is a
projection (one GPU, no concurrent ranks), not a measured multi-GPU number."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402
from paper_2605_18515_b200 import dist as cbd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "clustered"
only = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else None  # "P,rank": one shard only
A = synth.make(name)
steps = 50
out = {"workload": name, "nnz": int(A.nnz), "note": "projection: every rank's shard timed alone on one B200, aggregate = 2 nnz / max shard time", "P": {}}
agg = cb.decide_agg(*cb.block_stats(A))  # the global th0 decision
def time_shard(r0, r1):
    S = cbd.slice_rows(A, r0, r1)
    h = cb.build(S, device=0, agg_mode=agg, keep_host=0)
    x = torch.from_numpy(synth.vector(A.n, 0, 7)).to("cuda:0")
    y = torch.empty(S.m, dtype=torch.float64, device="cuda:0")
    for _ in range(5):
        cb.spmv(h, x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        cb.spmv(h, x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    cb.destroy(h)
    return ms, int(S.row_ptr[-1])


if only:
    P, r = only
    cuts = cbd.shard_bounds(A.row_ptr, P)
    ms, k = time_shard(int(cuts[r]), int(cuts[r + 1]))
    print(json.dumps({"workload": name, "P": P, "rank": r, "ms": ms, "nnz": k}))
    sys.exit(0)
for P in (1, 2, 4, 8):
    cuts = cbd.shard_bounds(A.row_ptr, P)
    res = [time_shard(int(cuts[r]), int(cuts[r + 1])) for r in range(P)]
    ms = [t for t, _ in res]
    out["P"][P] = {"shard_ms": ms, "shard_nnz": [k for _, k in res], "max_ms": max(ms),
                   "projected_aggregate_gflops": 2.0 * A.nnz / (max(ms) * 1e-3) / 1e9}
base = out["P"][1]["projected_aggregate_gflops"]
for P, v in out["P"].items():
    v["projected_efficiency"] = v["projected_aggregate_gflops"] / (P * base)
print(json.dumps(out))
