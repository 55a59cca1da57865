timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__maximum_warps_per_active_cycle_pct \
  --cache-control all --clock-control none -k regex:"coo_rowptr|add_tile" --csv -c 6 \
  --log-file gpurun_out/ncu_add.csv python tools/time_add.py 3 > gpurun_out/ncu_add.log 2>&1
