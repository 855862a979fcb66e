"""Small SpMV runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402

cases = [(synth.fig1(), {}), (synth.rmat(10, 16, 3), {}), (synth.clustered(1 << 11), {}),
         (synth.laplace5(64), {}), (synth.random_csr(77, 300, 0.05, 3, pattern="hub"), {"force_format": 1}),
         (synth.random_csr(50, 50, 0.4, 4, pattern="blockdense"), {"force_format": 2}),
         (synth.random_csr(50, 600, 0.2, 5), {"col_panels": 3}),
         (synth.uniform(1 << 10, 1 << 10, 20, 5, 1), {"agg_mode": 0})]
for A, opts in cases:
    for dt in ("f64", "f32"):
        tdt = torch.float64 if dt == "f64" else torch.float32
        h = cb.build(A, dtype=dt, device=0, **opts)
        x = torch.from_numpy(synth.vector(A.n, 0, 1)).to("cuda:0", tdt)
        y = torch.empty(A.m, dtype=tdt, device="cuda:0")
        cb.spmv(h, x, y)
        ss = torch.tensor([2.0], dtype=torch.float64, device="cuda:0")
        cb.spmv_scaled(h, x, ss, y)
        torch.cuda.synchronize()
        cb.destroy(h)
print("sanitize run ok")
