# DRAM bytes of one whole uniform SpMV (all P column panels: the 3rd SpMV's launches) for the bench
# line's roofline.traffic (profiles/ncu_traffic.json "uniform_f64"); metrics only, one GPU.
# P = the auto panel count of the 2^25-column matrix (capi.cpp: x slices of ~1/3 L2 -> 6).
P=${P:-6}
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:cb_spmv_kernel -s $((2 * P)) -c $P --csv python tools/prof_kernel.py --config uniform --launches 3 \
  > gpurun_out/ncu_uniform_traffic.csv 2> gpurun_out/ncu_uniform_traffic.err
echo uniform_traffic_rc=$?
