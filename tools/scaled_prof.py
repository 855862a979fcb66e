"""Launch spmv and spmv_scaled on R-MAT a few times each (for an ncu duration comparison)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402

A = synth.make(sys.argv[1] if len(sys.argv) > 1 else "rmat")
h = cb.build(A, device=0, keep_host=0)
x = torch.from_numpy(synth.vector(A.n, 0, 7)).to("cuda:0")
y = torch.empty(A.m, dtype=torch.float64, device="cuda:0")
ss = torch.full((1,), float(A.n), dtype=torch.float64, device="cuda:0")
for _ in range(3):
    cb.spmv(h, x, y)
    cb.spmv_scaled(h, x, ss, y)
torch.cuda.synchronize()
