"""Host build phases (CBSPMV_BUILD_TIMING=1) of BASELINE workloads with a device upload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CBSPMV_BUILD_TIMING"] = "1"
import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402

for name in (sys.argv[1:] or ["clustered", "rmat"]):
    t = time.perf_counter()
    A = synth.make(name)
    gen = time.perf_counter() - t
    t = time.perf_counter()
    h = cb.build(A, device=0, keep_host=0, device_build=int(os.environ.get("DEVICE_BUILD", "0")))
    wall = time.perf_counter() - t
    i = h.info
    print(f"{name}: gen {gen:.2f} s, build wall {wall:.2f} s (build_seconds {i['build_seconds']:.2f}, "
          f"upload {i['upload_seconds']:.2f}, panels {i['n_panels']}, nnz {i['nnz']}), cores {os.cpu_count()}",
          flush=True)
    cb.destroy(h)
