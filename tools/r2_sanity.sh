# compute-sanitizer over tools/sanitize_run.py (all four tools) and the N>1 bench paths run as two
# ranks sharing one B200 (CBSPMV_BENCH_SHARED_GPU=1: a functional test, not scaling numbers).
set -x
make all > gpurun_out/make.log 2>&1
for t in memcheck synccheck initcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $t python tools/sanitize_run.py > gpurun_out/sanitizer_$t.txt 2>&1; echo ${t}_rc=$?
  tail -2 gpurun_out/sanitizer_$t.txt
done
for c in clustered rmat uniform; do
  CBSPMV_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --config $c --no-cpu-baseline --also none > gpurun_out/mr_$c.log 2>&1
  echo mr_${c}_rc=$?
done
CBSPMV_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29612 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/mr_reference.log 2>&1; echo mr_ref_rc=$?
