# SURVEY §8(d) metric set for one cb_spmv_kernel launch per workload, cold (--cache-control all)
# and warm (--cache-control none, 3rd launch): L1 / L2 sector and request hit rates, RED traffic,
# DRAM bytes, LSU gather sectors.  Summarised by tools/ncu_metrics_summary.py.
set -x
make all > gpurun_out/make.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_request_hit_rate.pct,l1tex__t_sector_hit_rate.pct,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed
for cfg in "clustered f64" "rmat f64" "laplace f64" "clustered f32"; do
  set -- $cfg
  for cc in all none; do
    timeout 600 ncu --metrics $M --clock-control none --cache-control $cc -k regex:cb_spmv_kernel -s 2 -c 1 --csv \
      python tools/prof_kernel.py --config $1 --dtype $2 > gpurun_out/ncu_metrics_$1_$2_$cc.csv 2> gpurun_out/ncu_metrics_$1_$2_$cc.err
    echo "$1 $2 $cc rc=$?"
  done
done
