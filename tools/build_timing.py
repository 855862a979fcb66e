"""NEXT-3 (Fig. 13(b): preprocessing is "a small trade-off"):
wall time of the format build for the BASELINE workloads, host builder vs device builder
(device_build=1), with the builders' phase times (CBSPMV_BUILD_TIMING=1, captured from stderr),
the SpMV time of the built handle and the number of SpMVs the build costs.

    python tools/build_timing.py [--configs laplace,rmat,clustered,uniform] [--out file.json]

One JSON line per (config, builder); with --out, the list is also written as one JSON file."""
import argparse
import json
import os
import re
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CBSPMV_BUILD_TIMING"] = "1"
import torch  # noqa: E402

import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402


class StderrCapture:
    """Capture the C++ builders' phase lines (written to fd 2)."""

    def __enter__(self):
        self.tmp = tempfile.TemporaryFile(mode="w+b")
        sys.stderr.flush()
        self.saved = os.dup(2)
        os.dup2(self.tmp.fileno(), 2)
        return self

    def __exit__(self, *a):
        sys.stderr.flush()
        os.dup2(self.saved, 2)
        os.close(self.saved)
        self.tmp.seek(0)
        self.text = self.tmp.read().decode(errors="replace")
        self.tmp.close()


def phases(text):
    out = []
    for m in re.finditer(r"\[cbspmv build\] (.+?)\s+([0-9.]+) s", text):
        out.append([m.group(1).strip(), float(m.group(2))])
    return out


def spmv_ms(h, n, m, steps=10):
    x = torch.from_numpy(synth.vector(n, synth.VEC_UNIFORM, seed=7)).to("cuda:0")
    y = torch.empty(m, dtype=torch.float64, device="cuda:0")
    for _ in range(3):
        cb.spmv(h, x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        cb.spmv(h, x, y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="laplace,rmat,clustered,uniform")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = []
    for name in a.configs.split(","):
        t = time.perf_counter()
        A = synth.make(name)
        gen = time.perf_counter() - t
        for dev_build in (0, 1):
            torch.cuda.synchronize()
            with StderrCapture() as cap:
                t = time.perf_counter()
                h = cb.build(A, device=0, keep_host=0, device_build=dev_build)
                torch.cuda.synchronize()
                wall = time.perf_counter() - t
            i = h.info
            ms = spmv_ms(h, A.n, A.m)
            line = {"config": name, "builder": "device" if dev_build else "host", "nnz": int(i["nnz"]),
                    "gen_s": gen, "build_wall_s": wall, "build_s": i["build_seconds"], "upload_s": i["upload_seconds"],
                    "n_panels": int(i["n_panels"]), "spmv_ms": ms, "build_in_spmvs": wall / (ms * 1e-3),
                    "host_cores": os.cpu_count(), "phases": phases(cap.text)}
            print(json.dumps(line), flush=True)
            res.append(line)
            cb.destroy(h)
        del A
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"tool": "tools/build_timing.py", "gpu": torch.cuda.get_device_name(0), "runs": res}, f, indent=1)


if __name__ == "__main__":
    main()
