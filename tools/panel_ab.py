"""A/B of the column-panel count for the uniform matrix (configs[4]): SpMV time per panel count."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_18515_b200 as cb
import synth
A = synth.make("uniform")
x = torch.from_numpy(synth.vector(A.n, synth.VEC_UNIFORM, seed=7)).to("cuda:0")
y = torch.empty(A.m, dtype=torch.float64, device="cuda:0")
for P in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "3,4,6,8,12").split(",")]:
    h = cb.build(A, device=0, keep_host=0, col_panels=P)
    for _ in range(3):
        cb.spmv(h, x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10):
        cb.spmv(h, x, y)
    e1.record(); torch.cuda.synchronize()
    print(f"panels {P}: {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
    cb.destroy(h)
