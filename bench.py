#!/usr/bin/env python
"""CB-SpMV benchmark (BASELINE.json metric) — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat|clustered|laplace|uniform]
                    [--dtype f64|f32|f32f64] [--impl cb|reference]

Default workload: BASELINE configs[3] (block-clustered, 2^22 rows, ~407M nnz,
fp64) — the large synthetic matrix whose HBM roofline the metric asks for and
the one config exercising all three warp paths (DESIGN.md §6 explains the
choice); R-MAT (configs[2]) and the Laplacian (configs[1]) are measured with the
same protocol in the same run and reported under "detail.also".

A step is one y := A·x over the whole (row-sharded) matrix through the C ABI
(cbspmv_spmv: zero y + the persistent SpMV kernel).  Inputs already resident in
HBM; the matrix stream (>= 2 GB on the default workload) is far larger than the
126 MB L2, so back-to-back steps read it from HBM; a cold-L2 figure (L2 flushed
between individually timed steps) is reported beside it.  Multi-GPU: one
process per GPU under torchrun, rows split by nnz at block-row boundaries (no
data-path collective for a single SpMV), time = max over ranks.

--impl reference times the oracle (plain single-threaded C, the CPU baseline of
this tier) on rank 0 on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 SpMV GFLOP/s and achieved HBM GB/s vs B200 peak at 1/2/4/8 GPUs"
WORKLOAD = {
    "rmat": "BASELINE configs[2]: synthetic R-MAT scale 23, edge factor 16 (8,388,608 rows, ~131M nnz after dedup)",
    "clustered": "BASELINE configs[3]: synthetic block-clustered 2^22 rows, ~407M nnz, dense/CSR/COO mix",
    "laplace": "BASELINE configs[1]: 5-point Laplacian on a 1000x1000 grid (1M rows, 4,996,000 nnz)",
    "uniform": "BASELINE configs[4]: power iteration on uniform random 2^25 x 2^25, 50 nnz/row",
}


def env_int(k, d):
    return int(os.environ.get(k, d))


# ----------------------------------------------------------------------------- clocks (NVML)
class ClockSampler:
    """Sample SM clock + throttle reasons with NVML every ~5 ms during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            time.sleep(0.02)
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- workload
def make_matrix(config: str, rank: int, world: int):
    """This rank's row shard, generated alone ("each rank generates and builds only
    its rows"): the cut comes from per-row counts (synth.row_counts, no matrix materialised;
    rows split by nnz at block-row boundaries, equal shards for the uniform matrix), then the
    counter-based generator produces rows [r0, r1) only.  Returns (shard, (r0, r1), total nnz,
    total rows); the nnz total is all-reduced by the caller when world > 1."""
    import numpy as np
    import synth
    from paper_2605_18515_b200 import dist
    if world == 1:
        A = synth.make(config)
        return A, (0, A.m), A.nnz, A.m
    counts = synth.row_counts(config)
    if config == "uniform":
        cuts = dist.equal_bounds(len(counts), world)
    else:
        rp = np.zeros(len(counts) + 1, np.int64)
        np.cumsum(counts, out=rp[1:])
        cuts = dist.shard_bounds(rp, world)
    r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
    S = synth.make(config, r0, r1)
    return S, (r0, r1), None, len(counts)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# Random x-gather ceiling measured on this pool's B200 (tools/mb_mixed.cu,
# profiles/r1_microbench_tma_mixed.txt): ~0.94 random 32-byte sector requests per SM-cycle,
# whether issued by LDG or TMA gather4.  An aggregated matrix needs one random gather per
# restore entry (aggregated column of a block row), so n_restore / (0.94 * SMs * clock) bounds
# its SpMV from below independently of HBM.
GATHER_REQ_PER_SM_CYCLE = 0.94


def gather_floor(info, kernel_ms, sms=148, mhz=1965.0):
    if not info["agg"]:
        return None
    n = int(info["n_restore"])
    floor_ms = n / (GATHER_REQ_PER_SM_CYCLE * sms * mhz * 1e6) * 1e3
    return {"x_gathers": n, "floor_ms": floor_ms, "frac": floor_ms / kernel_ms if kernel_ms else None,
            "basis": "0.94 random sector requests / SM-cycle (profiles/r1_microbench_tma_mixed.txt), 148 SMs, 1965 MHz"}


def ncu_traffic(config: str, dtype: str):
    """dram bytes per launch of the SpMV kernel from the committed ncu --set full capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{config}_{dtype}")
    except Exception:
        return None


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    import oracle
    import synth
    A = synth.make(args.config)
    x = synth.vector(A.n, synth.VEC_UNIFORM, seed=7)
    # bounded sample: leading block-aligned row range sized so the whole run ends in minutes
    t0 = time.perf_counter()
    probe_rows = min(A.m, max(16, (A.m // 64) // 16 * 16))
    from paper_2605_18515_b200.dist import slice_rows
    oracle.spmv_csr(slice_rows(A, 0, probe_rows), x)
    t_probe = max(time.perf_counter() - t0, 1e-6)
    budget = 150.0 / max(1, args.steps + args.warmup)  # seconds per step
    rows = int(min(A.m, probe_rows * budget / t_probe)) // 16 * 16
    rows = max(16, min(A.m, rows))
    S = slice_rows(A, 0, rows)
    nnz_s = int(S.row_ptr[-1])
    for _ in range(args.warmup):
        oracle.spmv_csr(S, x)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.spmv_csr(S, x)
    dt = (time.perf_counter() - t0) / max(1, args.steps)
    gflops = 2.0 * nnz_s / dt / 1e9
    sample = f"rows [0,{rows}) of {A.m} ({nnz_s} of {A.nnz} nnz), full oracle Alg. 1 per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": gflops, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "name": args.config, "m": A.m, "nnz": A.nnz},
        "cpu_baseline": {"value": gflops, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": gflops, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_cb(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as tdist

    import paper_2605_18515_b200 as cb
    from paper_2605_18515_b200 import dist
    import synth

    dev, cdev = init_ranks(local_rank, world)
    local_rank = dev.index

    def allreduce(a, op="sum"):
        if world == 1:
            return a
        t = torch.from_numpy(np.asarray(a)).to(cdev)
        tdist.all_reduce(t, op=tdist.ReduceOp.SUM if op == "sum" else tdist.ReduceOp.MAX)
        return t.cpu().numpy()

    def barrier():
        if world > 1:
            tdist.barrier()

    t0 = time.perf_counter()
    A, (r0, r1), nnz_total, m_total = make_matrix(args.config, rank, world)
    gen_s = time.perf_counter() - t0
    if nnz_total is None:
        nnz_total = int(allreduce(np.array([A.nnz], np.int64))[0])
    agg = dist.global_agg(A, lambda a: allreduce(a), dtype=args.dtype) if world > 1 else -1
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    h = cb.build(A, dtype=args.dtype, device=local_rank, agg_mode=agg, keep_host=0)
    info = h.info
    x_host = synth.vector(A.n, synth.VEC_UNIFORM, seed=7)
    x = torch.from_numpy(x_host).to(dev, tdt)
    y = torch.empty(A.m, dtype=tdt, device=dev)
    stream = torch.cuda.current_stream(dev)

    # warm-up
    for _ in range(max(args.warmup, 0)):
        cb.spmv(h, x, y)
    torch.cuda.synchronize()

    # ---- timed region: K back-to-back steps (inputs > L2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            cb.spmv(h, x, y)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / max(1, args.steps)
    ms_max = float(allreduce(np.array([ms]), "max")[0])

    # ---- dominant kernel alone (y += A x, same stream, events over K launches)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    k0.record(stream)
    for _ in range(args.steps):
        cb.spmv_add(h, x, y)
    k1.record(stream)
    torch.cuda.synchronize()
    kernel_ms = k0.elapsed_time(k1) / max(1, args.steps)

    # ---- cold L2: flush (write 2x L2) before each individually timed step
    flush = torch.empty(64 << 20, dtype=torch.float64, device=dev)  # 512 MB
    cold = []
    for _ in range(min(args.steps, 20)):
        flush.fill_(1.0)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        cb.spmv(h, x, y)
        c1.record(stream)
        torch.cuda.synchronize()
        cold.append(c0.elapsed_time(c1))
    del flush
    cold_ms = statistics.median(cold) if cold else None
    cold_ms_max = float(allreduce(np.array([cold_ms or 0.0]), "max")[0])

    # ---- end to end through the public API with host buffers (pinned)
    # K independent requests (a ring of 4 pinned x / y host buffers) through
    # cbspmv_spmv_host_batch: every step uploads its x and downloads its y inside the timed
    # region; the copies of neighbouring steps overlap the SpMV (two device staging slots)
    vt = np.float32 if args.dtype == "f32" else np.float64
    ring = 4
    xhs = [torch.from_numpy(x_host.astype(vt)).pin_memory().numpy() for _ in range(ring)]
    yhs = [torch.empty(A.m, dtype=tdt).pin_memory().numpy() for _ in range(ring)]
    cb.spmv_host_batch(h, xhs[:2], yhs[:2])
    barrier()
    t_e2e = time.perf_counter()
    cb.spmv_host_batch(h, [xhs[k % ring] for k in range(args.steps)], [yhs[k % ring] for k in range(args.steps)])
    e2e_s = (time.perf_counter() - t_e2e) / max(1, args.steps)
    e2e_max = float(allreduce(np.array([e2e_s]), "max")[0])
    y_dev = torch.empty(A.m, dtype=tdt, device=dev)
    cb.spmv(h, x, y_dev)
    # fp atomics make the two runs differ in rounding; rows with cancellation need an absolute
    # term scaled to the vector (the oracle-based per-row bound lives in the GPU tests)
    yd = y_dev.cpu().numpy()
    e2e_ok = bool(np.allclose(yhs[(args.steps - 1) % ring], yd, rtol=1e-5 if args.dtype == "f32" else 1e-10,
                              atol=(1e-5 if args.dtype == "f32" else 1e-12) * float(np.max(np.abs(yd), initial=0.0))))

    flops = 2.0 * nnz_total
    value = flops / (ms_max * 1e-3) / 1e9
    peak, peak_src = peaks()
    achieved = info["alg_bytes"] / (kernel_ms * 1e-3) / 1e9
    # ncu DRAM bytes of the whole-matrix launch (profiles/ncu_traffic.json): only a 1-GPU line
    traffic = ncu_traffic(args.config, args.dtype) if world == 1 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(A, x_host, args.dtype)
    also = {}
    if world == 1 and args.also:
        names = [n for n in args.also.split(",") if n and n not in (args.config, "uniform", "none")]
        cb.destroy(h)
        also = measure_also(names, args.dtype, args.steps, max(args.warmup, 3), local_rank)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded generators, synth/)",
            # config: the workload alone, identical to the reference arm's; run details under "detail"
            "config": {"workload": WORKLOAD[args.config], "name": args.config, "m": int(m_total), "nnz": int(nnz_total)},
            "detail": {
                "agg": int(info["agg"]), "blocks": int(info["nb"]),
                "fmt_count_coo_csr_dense": list(info["fmt_count"]), "parallelism": f"row-shard x{world}",
                **({"shared_gpu_test": True} if shared_gpu_test() else {}),
                "l2": "inputs larger than L2 (matrix stream %.2f GB vs 126 MB L2); cold_l2_ms flushes 512 MB "
                      "before each step" % (info["dev_stream_bytes"] / 1e9),
                "cold_l2_ms": cold_ms, "cold_l2_gflops": flops / (cold_ms_max * 1e-3) / 1e9 if cold_ms else None,
                "alg_bytes_per_spmv": int(info["alg_bytes"]), "dev_stream_bytes": int(info["dev_stream_bytes"]),
                "achieved_hbm_gbs_step": info["alg_bytes"] / (ms * 1e-3) / 1e9,
                "tb_load_sd": info["tb_load_sd"], "tb_load_sd_natural": info["tb_load_sd_natural"],
                "gen_s": gen_s, "build_s": info["build_seconds"], "upload_s": info["upload_seconds"],
                "grid": info["grid"], "gather_floor": gather_floor(info, kernel_ms), "also": also,
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": "cb_spmv_kernel",
                         "kernel_ms": kernel_ms, "peak_source": peak_src,
                         "bytes": "alg_bytes = 21 B/block meta + |mtx_data| + 4 B/restore entry + "
                                  "8 B/cols_offset + size(Val)*(n+m), per launch"},
            "e2e": {"value": flops / e2e_max / 1e9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(A.n) * xhs[0].itemsize, "d2h_bytes_per_step": int(A.m) * yhs[0].itemsize,
                    "matches_device_y": e2e_ok,
                    "path": "cbspmv_spmv_host_batch: K requests, pinned host x in / y out every step, "
                            "uploads and downloads of neighbouring steps overlapping the SpMV"},
            "gpu_launches": int(args.steps * info["launches_per_spmv"]),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        cb.destroy(h)
        tdist.destroy_process_group()


def measure_also(names, dtype, steps, warmup, local_rank):
    """Other BASELINE workloads, same protocol (K back-to-back steps, CUDA events), N=1 only."""
    import torch

    import paper_2605_18515_b200 as cb
    import synth
    out = {}
    dev = torch.device("cuda", local_rank)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    for name in names:
        A = synth.make(name)
        h = cb.build(A, dtype=dtype, device=local_rank, keep_host=0)
        x = torch.from_numpy(synth.vector(A.n, synth.VEC_UNIFORM, seed=7)).to(dev, tdt)
        y = torch.empty(A.m, dtype=tdt, device=dev)
        for _ in range(warmup):
            cb.spmv(h, x, y)
        st = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(steps):
            cb.spmv(h, x, y)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(st)
        for _ in range(steps):
            cb.spmv_add(h, x, y)
        k1.record(st)
        torch.cuda.synchronize()
        kms = k0.elapsed_time(k1) / steps
        peak, _ = peaks()
        i = h.info
        out[name] = {"workload": WORKLOAD[name], "nnz": int(i["nnz"]), "agg": int(i["agg"]),
                     "gflops": 2.0 * i["nnz"] / (ms * 1e-3) / 1e9, "ms_per_step": ms, "kernel_ms": kms,
                     "alg_bytes": int(i["alg_bytes"]),
                     "hbm_frac": i["alg_bytes"] / (kms * 1e-3) / 1e9 / peak,
                     "gather_floor": gather_floor(i, kms),
                     "l2_resident": i["alg_bytes"] < 126e6}
        cb.destroy(h)
        del A
    return out


def run_power(args, rank, world, local_rank):
    """BASELINE configs[4]: iterated SpMV (power iteration) on the uniform matrix, rows split in
    equal shards across ranks; a step = spmv_scaled + sumsq + (N>1) NCCL all-reduce + all-gather."""
    import torch
    import torch.distributed as tdist

    import paper_2605_18515_b200 as cb
    from paper_2605_18515_b200 import dist

    dev, cdev = init_ranks(local_rank, world)
    local_rank = dev.index
    if shared_gpu_test() and world > 1 and args.exchange != "fused":
        raise SystemExit("CBSPMV_BENCH_SHARED_GPU runs the power iteration with --exchange fused only (gloo host collectives)")
    t0 = time.perf_counter()
    A, (r0, r1), nnz_total, m_total = make_matrix("uniform", rank, world)
    gen_s = time.perf_counter() - t0
    if nnz_total is None:
        nnz_total = int(_allreduce_np(np.array([A.nnz], np.int64), cdev, world)[0])
    agg = dist.global_agg(A, lambda a: _allreduce_np(a, cdev, world), dtype=args.dtype) if world > 1 else -1
    # column panels: the auto count on one GPU (x slices L2-resident); with N ranks a multiple
    # of N so panel cuts fall on the x owners' boundaries (NEXT-1 (i) overlap)
    panels = 0 if world == 1 else world * max(1, -(-6 // world))  # 1 GPU: the auto count (6)
    h = cb.build(A, dtype=args.dtype, device=local_rank, agg_mode=agg, keep_host=0, col_panels=panels)
    info = h.info
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    x0 = torch.ones(A.n, dtype=tdt, device=dev)
    fused = None
    if args.exchange == "fused":
        # NEXT-1 (ii): y shards pushed into every peer's next iterate by one kernel over peer
        # memory (CUDA IPC mappings), the next step gated by device flags
        fused = dist.FusedPowerIteration(h, A.n, "f32" if args.dtype == "f32" else "f64", world, rank, local_rank)

        def run_steps(n):
            return fused.run(x0, n)
    elif args.exchange == "nccl" or args.no_overlap:
        def run_steps(n):
            return dist.power_iteration_device(h, x0, n, world)
    else:
        def run_steps(n):
            return dist.power_iteration_overlapped(h, x0, n, world, rank)
    run_steps(max(args.warmup, 3))
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(st)
        x, ss = run_steps(args.steps)
        e1.record(st)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    ms_max = float(_allreduce_np(np.array([ms]), cdev, world, "max")[0])
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    y = torch.empty(A.m, dtype=tdt, device=dev)
    k0.record(st)
    for _ in range(args.steps):
        cb.spmv_add(h, x0, y)
    k1.record(st)
    torch.cuda.synchronize()
    kernel_ms = k0.elapsed_time(k1) / args.steps
    lam = float(ss.item()) ** 0.5
    # per-step split (fused exchange): CUDA events after each enqueued phase of a separate run
    split = None
    if fused is not None:
        marks = []

        def mark(phase):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(st)
            marks.append((phase, ev))
        fused.run(x0, args.steps, mark=mark)
        torch.cuda.synchronize()
        acc = {}
        for (_, a), (ph, b) in zip(marks[:-1], marks[1:]):
            acc[ph] = acc.get(ph, 0.0) + a.elapsed_time(b)
        split = {k + "_ms": v / args.steps for k, v in acc.items()}
        split["note"] = ("per step, CUDA events on the stream after each enqueued phase: wait = device flag wait "
                         "for every rank's publish of the previous step (+ rank-order sum of squares), spmv = "
                         "zero y + the panels' SpMV kernels, publish = the fused finalize / peer-store kernel")
    # end to end through the public API: the start vector from pinned host memory, K steps, the
    # eigenvalue estimate read back (what a user of the power iteration gets)
    e2e = None
    if fused is not None:
        x0_host = torch.ones(A.n, dtype=tdt).pin_memory()
        if world > 1:
            tdist.barrier()
        t_e = time.perf_counter()
        x0_dev = x0_host.to(dev, non_blocking=True)
        _, ss_e = fused.run(x0_dev, args.steps)
        lam_e = float(ss_e.item()) ** 0.5
        e2e_s = time.perf_counter() - t_e
        e2e_max = float(_allreduce_np(np.array([e2e_s]), cdev, world, "max")[0])
        e2e = {"value": 2.0 * nnz_total * args.steps / e2e_max / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(A.n) * x0_host.element_size() / args.steps,
               "d2h_bytes_per_step": 8 / args.steps, "lambda": lam_e,
               "path": f"x0 from pinned host memory -> FusedPowerIteration.run({args.steps} steps) -> lambda read "
                       "back; host copies inside the timed region, amortised over the steps"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(A, np.ones(A.n), args.dtype)
        cpu["sample"] += " of this rank's rows, one SpMV of the power iteration"
    if fused is not None and fused.timed_out():
        raise RuntimeError("fused exchange: a device wait timed out (a peer never published)")
    peak, peak_src = peaks()
    if rank == 0:
        line = {
            "metric": METRIC, "value": 2.0 * nnz_total / (ms_max * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded generators, synth/)",
            "config": {"workload": WORKLOAD["uniform"], "name": "uniform", "m": int(m_total), "nnz": int(nnz_total)},
            "detail": {"rows_per_rank": int(A.m), "agg": int(info["agg"]),
                       "lambda": lam, "gen_s": gen_s, "build_s": info["build_seconds"],
                       "n_panels": int(info["n_panels"]), "gather_floor": gather_floor(info, kernel_ms),
                       "step_split": split, "rows_per_rank_range": [int(r0), int(r1)],
                       "exchange": args.exchange,
                       **({"shared_gpu_test": True} if shared_gpu_test() else {}),
                       "parallelism": f"row-shard x{world}, " + {
                           "fused": "one fused finalize+exchange kernel per step over peer memory (CUDA IPC / NVLink), device flags",
                           "nccl": "NCCL all-reduce + all-gather per step",
                           "overlap": "NCCL all-reduce + per-owner broadcasts overlapped with column panels"}[
                               "nccl" if args.no_overlap else args.exchange]},
            "roofline": {"bound": "hbm", "achieved": info["alg_bytes"] / (kernel_ms * 1e-3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": info["alg_bytes"] / (kernel_ms * 1e-3) / 1e9 / peak,
                         "traffic": ncu_traffic("uniform", args.dtype) if world == 1 else None,
                         "kernel": "cb_spmv_kernel",
                         "kernel_ms": kernel_ms, "peak_source": peak_src},
            "gpu_launches": int(args.steps * ((3 + info["n_panels"]) if args.exchange == "fused" else
                                              (2 + (1 if args.no_overlap else info["n_panels"])))),
            "clocks": clk.summary(), "cpu_baseline": cpu,
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    if fused is not None:
        if world > 1:
            tdist.barrier()  # no peer still stores into a mapping we are about to free
        fused.destroy()
    cb.destroy(h)
    if world > 1:
        tdist.destroy_process_group()


def shared_gpu_test() -> bool:
    """CBSPMV_BENCH_SHARED_GPU=1: a functional test of the multi-rank path on a box with fewer GPUs
    than ranks -- ranks share GPUs (local_rank mod device count) and the host-side collectives
    run over gloo.  Its timings are not scaling numbers (config.shared_gpu_test marks the line)."""
    return os.environ.get("CBSPMV_BENCH_SHARED_GPU") == "1"


def init_ranks(local_rank, world):
    """Device of this rank and the device of its collective buffers (NCCL: the GPU; gloo: CPU)."""
    import torch
    import torch.distributed as tdist
    shared = shared_gpu_test()
    ndev = max(1, torch.cuda.device_count())
    dev = torch.device("cuda", local_rank % ndev if shared else local_rank)
    torch.cuda.set_device(dev)
    if world > 1:
        if shared:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=dev)
    return dev, (torch.device("cpu") if shared else dev)


def _allreduce_np(a, dev, world, op="sum"):
    if world == 1:
        return np.asarray(a)
    import torch
    import torch.distributed as tdist
    t = torch.from_numpy(np.asarray(a)).to(dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.SUM if op == "sum" else tdist.ReduceOp.MAX)
    return t.cpu().numpy()


def cpu_baseline(A, x, dtype):
    """The oracle as it stands (single-threaded C, Alg. 1) on a bounded sample: ~10 s of CPU work."""
    import oracle
    import synth
    from paper_2605_18515_b200.dist import slice_rows
    if dtype in ("f32", "f32f64"):  # the oracle in fp64 on the rounded inputs
        A = synth.CSR(A.m, A.n, A.row_ptr, A.col, A.val.astype(np.float32).astype(np.float64))
    if dtype == "f32":
        x = x.astype(np.float32).astype(np.float64)
    t0 = time.perf_counter()
    oracle.spmv_csr(A, x)
    t1 = time.perf_counter() - t0
    if t1 > 10.0:  # one full pass is already past the budget: time a leading row sample instead
        rows = max(16, int(A.m * 10.0 / t1) // 16 * 16)
        S = slice_rows(A, 0, rows)
        t0 = time.perf_counter()
        oracle.spmv_csr(S, x)
        dt = time.perf_counter() - t0
        nnz = int(S.row_ptr[-1])
        return {"value": 2.0 * nnz / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
                "sample": f"rows [0,{rows}) ({nnz} nnz), 1 pass"}
    reps = int(max(1, min(20, 10.0 / max(t1, 1e-3))))
    t0 = time.perf_counter()
    for _ in range(reps):
        oracle.spmv_csr(A, x)
    dt = (time.perf_counter() - t0) / reps
    return {"value": 2.0 * A.nnz / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
            "sample": f"full matrix ({A.nnz} nnz), {reps} passes after 1 warm pass"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="clustered", choices=list(WORKLOAD))
    ap.add_argument("--also", default="rmat,laplace",
                    help="other BASELINE workloads timed the same way on N=1 (comma list, '' for none)")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32", "f32f64"])
    ap.add_argument("--impl", default="cb", choices=["cb", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="fused", choices=["fused", "overlap", "nccl"],
                    help="power iteration (--config uniform): fused peer-memory exchange kernel (default), "
                         "NCCL broadcasts overlapped with column panels, or plain NCCL all-reduce + all-gather")
    ap.add_argument("--no-overlap", action="store_true",
                    help="uniform power iteration: plain all-gather instead of per-owner broadcasts + panels")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config == "uniform":
        run_power(args, rank, world, local_rank)
    else:
        run_cb(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
