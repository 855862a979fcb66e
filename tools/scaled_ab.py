"""Time cbspmv_spmv_add, cbspmv_spmv (zero y + add) and cbspmv_spmv_scaled on one workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "uniform"
n_it = int(sys.argv[2]) if len(sys.argv) > 2 else 10
A = synth.make(name)
h = cb.build(A, device=0, keep_host=0)
x = torch.from_numpy(synth.vector(A.n, 0, 7)).to("cuda:0")
y = torch.empty(A.m, dtype=torch.float64, device="cuda:0")
ss = torch.full((1,), float(A.n), dtype=torch.float64, device="cuda:0")
calls = {"spmv_add": lambda: cb.spmv_add(h, x, y), "spmv": lambda: cb.spmv(h, x, y),
         "spmv_scaled": lambda: cb.spmv_scaled(h, x, ss, y)}
for rep in range(2):
    for k, f in calls.items():
        for _ in range(2):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n_it):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} {k}: {e0.elapsed_time(e1) / n_it:.3f} ms", flush=True)
