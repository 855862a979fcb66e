# Round profiles: ncu launch list of the bench command + one --set full capture per workload.
set -x
make all > gpurun_out/make.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
   python bench.py --steps 5 --warmup 3 --no-cpu-baseline --also "" > gpurun_out/bench_under_ncu.log 2>&1; echo launch_rc=$?
for c in ${CONFIGS:-clustered rmat}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:cb_spmv_kernel -s 1 -c 1 -f -o gpurun_out/prof_$c python tools/prof_kernel.py --config $c > gpurun_out/ncu_$c.log 2>&1; echo prof_${c}_rc=$?
done
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_default.log
CBSPMV_BUILD_TIMING=1 timeout 900 python tools/build_timing.py clustered rmat uniform > gpurun_out/build_timing.log 2>&1; echo timing_rc=$?
