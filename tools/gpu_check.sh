set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
make all > gpurun_out/make.log 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -3 gpurun_out/bench.log
