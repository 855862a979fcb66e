"""Step time (cbspmv_spmv: zero y + SpMV) of per-build env variants, CUDA events, in-process.
    python tools/step_ab.py laplace "CBSPMV_PDL=0;" [launches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402

name, variants = sys.argv[1], sys.argv[2].split(";")
n_it = int(sys.argv[3]) if len(sys.argv) > 3 else 200
A = synth.make(name)
x = torch.from_numpy(synth.vector(A.n, 0, 7)).to("cuda:0")
y = torch.empty(A.m, dtype=torch.float64, device="cuda:0")
for rep in range(2):
    for v in variants:
        saved = dict(os.environ)
        for kv in filter(None, v.split(",")):
            k, val = kv.split("=", 1)
            os.environ[k] = val
        try:
            h = cb.build(A, device=0, keep_host=0)
        finally:
            os.environ.clear()
            os.environ.update(saved)
        for _ in range(5):
            cb.spmv(h, x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n_it):
            cb.spmv(h, x, y)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} {v or 'default'}: step {e0.elapsed_time(e1) / n_it * 1e3:.1f} us", flush=True)
        cb.destroy(h)
