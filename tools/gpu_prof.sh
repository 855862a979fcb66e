set -x
make all > gpurun_out/make.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cb_spmv_kernel -s 1 -c 1 -o gpurun_out/prof_rmat python tools/prof_kernel.py --config rmat > gpurun_out/ncu_rmat.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_rmat.log
