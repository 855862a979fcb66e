"""NEXT-2: the paper's ablation re-measured on B200 with the synthetic workloads.

Variants (build options of cbspmv_build):
  I    intra-block data aggregation only: no column aggregation, every block COO, no Alg. 2
  II   + column aggregation (th0 rule) + format selection, no Alg. 2
  full + TB-Load-Balance (Alg. 2) — the default pipeline
plus agg forced on / off with everything else default.
Prints one JSON line per (workload, variant): kernel time, GFLOP/s, blocks, alg bytes.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_18515_b200 as cb  # noqa: E402
import synth  # noqa: E402

VARIANTS = {
    "I": dict(agg_mode=0, force_format=0, balance=0),
    "II": dict(balance=0),
    "full": dict(),
    "agg_on": dict(agg_mode=1),
    "agg_off": dict(agg_mode=0),
}

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="clustered,rmat,laplace")
ap.add_argument("--steps", type=int, default=50)
a = ap.parse_args()
for name in a.configs.split(","):
    A = synth.make(name)
    x = torch.from_numpy(synth.vector(A.n, synth.VEC_UNIFORM, seed=7)).to("cuda:0")
    y = torch.empty(A.m, dtype=torch.float64, device="cuda:0")
    for vname, opts in VARIANTS.items():
        try:
            h = cb.build(A, device=0, keep_host=0, **opts)
        except cb.CBSpMVError as e:  # e.g. forced COO on 256-nnz blocks is still valid; report failures
            print(json.dumps({"workload": name, "variant": vname, "error": str(e)}), flush=True)
            continue
        for _ in range(5):
            cb.spmv(h, x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.steps):
            cb.spmv(h, x, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        i = h.info
        print(json.dumps({"workload": name, "variant": vname, "opts": opts, "ms": ms,
                          "gflops": 2.0 * i["nnz"] / (ms * 1e-3) / 1e9, "agg": i["agg"], "blocks": i["nb"],
                          "fmt_count": list(i["fmt_count"]), "alg_bytes": i["alg_bytes"],
                          "hbm_gbs": i["alg_bytes"] / (ms * 1e-3) / 1e9,
                          "tb_load_sd": i["tb_load_sd"], "tb_load_sd_natural": i["tb_load_sd_natural"]}),
              flush=True)
        cb.destroy(h)
