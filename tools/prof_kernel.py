"""Build one BASELINE workload and launch the SpMV a few times (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rmat")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--launches", type=int, default=3)
ap.add_argument("--small", action="store_true")
a = ap.parse_args()
A = synth.make(a.config, small=a.small)
tdt = torch.float32 if a.dtype == "f32" else torch.float64
h = cb.build(A, dtype=a.dtype, device=0, keep_host=0)
x = torch.from_numpy(synth.vector(A.n, 0, 7)).to("cuda:0", tdt)
y = torch.empty(A.m, dtype=tdt, device="cuda:0")
for _ in range(a.launches):
    cb.spmv(h, x, y)
torch.cuda.synchronize()
print(h.info)
