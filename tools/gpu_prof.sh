set -x
make all > gpurun_out/make.log 2>&1
for c in ${CONFIGS:-rmat}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cb_spmv_kernel -s 1 -c 1 -f -o gpurun_out/prof_$c python tools/prof_kernel.py --config $c > gpurun_out/ncu_$c.log 2>&1; echo rc=$?
done
