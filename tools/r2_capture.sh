# Round capture on one B200 (tools/make_profiles.sh summarises it into profiles/<tag>_*):
# full GPU suite, smoke, bench lines, ablation, build timing, ncu launch list of the default bench
# command, one ncu --set full capture per workload, the SURVEY §8(d) metric set.
set -x
make all > gpurun_out/make.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
  tail -3 gpurun_out/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?
for c in rmat uniform; do
  timeout 900 python bench.py --config $c --steps 50 --warmup 5 --also none > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?
done
for dt in f32 f32f64; do
  timeout 900 python bench.py --dtype $dt --steps 100 --warmup 5 --no-cpu-baseline --also rmat > gpurun_out/bench_clustered_$dt.log 2>&1; echo bench_$dt=$?
done
timeout 1800 python tools/ablation.py --configs clustered,rmat,laplace,uniform > gpurun_out/ablation.jsonl 2> gpurun_out/ablation.err; echo ablation_rc=$?
if [ "${SKIP_TIMING:-0}" != "1" ]; then
  timeout 1500 python tools/build_timing.py --out gpurun_out/build_timing.json > gpurun_out/build_timing.log 2>&1; echo timing_rc=$?
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 5 --warmup 3 --no-cpu-baseline --also "" > gpurun_out/bench_under_ncu.log 2>&1; echo launch_rc=$?
for c in clustered rmat laplace; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:cb_spmv_kernel -s 1 -c 1 -f -o gpurun_out/prof_$c python tools/prof_kernel.py --config $c > gpurun_out/ncu_$c.log 2>&1; echo prof_${c}_rc=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cb_spmv_kernel -s 12 -c 1 -f -o gpurun_out/prof_uniform python tools/prof_kernel.py --config uniform --launches 3 > gpurun_out/ncu_uniform.log 2>&1; echo prof_uniform_rc=$?
bash tools/ncu_metrics.sh > gpurun_out/ncu_metrics.log 2>&1; echo metrics_rc=$?
bash tools/ncu_uniform_traffic.sh
# the bounds-checking debug build over the GPU suite (compute-sanitizer is closed on the pool)
if [ -f ab/check/libcbspmv.so ]; then
  CBSPMV_LIB=$PWD/ab/check/libcbspmv.so timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > gpurun_out/check_pytest.log 2>&1; echo check_pytest_rc=$?
  CBSPMV_LIB=$PWD/ab/check/libcbspmv.so timeout 600 python tools/sanitize_run.py > gpurun_out/check_sanitize_run.txt 2>&1; echo check_run_rc=$?
fi
