# usage: bash tools/gpu_check.sh [pytest-args]   (env BENCH="rmat clustered", STEPS=50)
set -x
make all > gpurun_out/make.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
  tail -3 gpurun_out/pytest_gpu.log
fi
for c in ${BENCH:-rmat}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 ${BENCH_ARGS:-} > gpurun_out/bench_$c.log 2>&1; echo bench_${c}_rc=$?
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', 'GFLOP/s=%.1f ms=%.3f kernel_ms=%.3f frac=%.3f e2e=%.1f clocks=%s' % (d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e']['value'], d['clocks']))" 2>&1 | tail -1
done
