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
# stage reuse (many 4 KB pages per CTA), with dynamic and static page claiming
reuse = [(synth.clustered(1 << 13), {}), (synth.rmat(12, 16, 3), {})]
for env in ({"CBSPMV_PAGE_BYTES": "4096", "CBSPMV_DYNAMIC_PAGES": "1"},
            {"CBSPMV_PAGE_BYTES": "4096", "CBSPMV_DYNAMIC_PAGES": "0"}):
    os.environ.update(env)
    for A, opts in reuse:
        for dt in ("f64", "f32"):
            tdt = torch.float64 if dt == "f64" else torch.float32
            h = cb.build(A, dtype=dt, device=0, **opts)
            x = torch.from_numpy(synth.vector(A.n, 0, 1)).to("cuda:0", tdt)
            y = torch.empty(A.m, dtype=tdt, device="cuda:0")
            for _ in range(2):
                cb.spmv(h, x, y)
            torch.cuda.synchronize()
            cb.destroy(h)
    for k in env:
        del os.environ[k]
# row-run slices with a forced hot x cache (full and 32 columns), host- and device-filled
for env in ({"CBSPMV_HOT_MIN_PCT": "0"}, {"CBSPMV_HOT_MIN_PCT": "0", "CBSPMV_HOT_BYTES": "256", "CBSPMV_RUN_MAX": "3"}):
    os.environ.update(env)
    A = synth.rmat(12, 16, 3)
    for dt in ("f64", "f32"):
        for dbuild in (0, 1):
            tdt = torch.float64 if dt == "f64" else torch.float32
            h = cb.build(A, dtype=dt, device=0, device_build=dbuild)
            assert h.info["n_hot"] > 0
            x = torch.from_numpy(synth.vector(A.n, 0, 1)).to("cuda:0", tdt)
            y = torch.empty(A.m, dtype=tdt, device="cuda:0")
            cb.spmv(h, x, y)
            torch.cuda.synchronize()
            cb.destroy(h)
    for k in env:
        del os.environ[k]
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
# pipelined host batch (two staging slots, copy streams)
A = synth.clustered(1 << 11)
h = cb.build(A, device=0)
xs = [synth.vector(A.n, 0, k) for k in range(3)]
ys = [np.empty(A.m) for _ in range(3)]
cb.spmv_host_batch(h, xs, ys)
cb.destroy(h)
# fused finalize + exchange: 2 ranks simulated in one process, 3 steps
from paper_2605_18515_b200 import dist as cbd  # noqa: E402
A = synth.uniform(1 << 11, 1 << 11, 20, 6, 1)
m2 = A.m // 2
hs = [cb.build(cbd.slice_rows(A, r * m2, (r + 1) * m2), device=0) for r in range(2)]
xcs = [cb.Exchange(A.n, "f64", 2, r, 0) for r in range(2)]
for xc in xcs:
    xc.connect(peer_bases=[c.base() for c in xcs])
    xc.buffer(0).fill_(1.0)
    xc.buffer(1).zero_()
sss = [torch.tensor([float(A.n)], dtype=torch.float64, device="cuda:0") for _ in range(2)]
for k in range(3):
    for r in range(2):
        if k:
            xcs[r].wait(k, sss[r], 5.0)
        cb.spmv_scaled(hs[r], xcs[r].buffer(k & 1), sss[r], xcs[r].buffer((k + 1) & 1)[r * m2:(r + 1) * m2])
        xcs[r].publish((k + 1) & 1, r * m2, m2, k + 1)
for r in range(2):
    xcs[r].wait(3, sss[r], 5.0)
torch.cuda.synchronize()
assert not any(xc.timed_out() for xc in xcs)
for h in hs:
    cb.destroy(h)
for xc in xcs:
    xc.destroy()
print("sanitize run ok")
