"""In-process A/B of per-build env knobs on one workload: the matrix is generated once, then one
handle per variant is built (the launch-shape / layout env knobs are read per build) and timed
with CUDA events.   python tools/ab_inproc.py rmat "CBSPMV_STAGES=6;CBSPMV_STAGES=12" [launches]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1]
variants = sys.argv[2].split(";")
launches = int(sys.argv[3]) if len(sys.argv) > 3 else 50
dtype = os.environ.get("AB_DTYPE", "f64")
A = synth.make(name)
tdt = torch.float32 if dtype == "f32" else torch.float64
x = torch.from_numpy(synth.vector(A.n, 0, 7)).to("cuda:0", tdt)
y = torch.empty(A.m, dtype=tdt, device="cuda:0")
ref = None
for v in variants:
    saved = dict(os.environ)
    for kv in filter(None, v.split(",")):
        k, val = kv.split("=", 1)
        os.environ[k] = val
    try:
        h = cb.build(A, dtype=dtype, device=0, keep_host=0)
    finally:
        os.environ.clear()
        os.environ.update(saved)
    for _ in range(5):
        cb.spmv(h, x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(launches):
        cb.spmv(h, x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / launches
    if ref is None:
        ref = y.clone()
    err = (y - ref).abs().max().item() / max(ref.abs().max().item(), 1e-300)
    print(f"{name} {v or 'default'}: {ms:.4f} ms  {2 * A.nnz / ms / 1e6:.1f} GFLOP/s  max rel diff vs first {err:.2e}",
          flush=True)
    cb.destroy(h)
