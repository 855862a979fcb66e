# A/B of env settings on one bench config: AB="CBSPMV_COO_SEGRED=0;CBSPMV_COO_SEGRED=1" CONFIG=rmat
make all > gpurun_out/make.log 2>&1
IFS=';' read -ra VARIANTS <<< "${AB:-X=0}"
for c in ${CONFIGS:-rmat}; do
for v in "${VARIANTS[@]}"; do
  env $v timeout 600 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --also none > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', 'GFLOP/s=%.1f ms=%.3f kernel_ms=%.3f frac=%.3f cold_ms=%.3f' % (d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['detail']['cold_l2_ms']))" 2>&1 | tail -1
done; done
