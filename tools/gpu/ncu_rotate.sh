# ncu, one pass per launch (no replay-induced warming): DRAM bytes of every
# headline launch under the rotating-copies protocol, cache control none
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --cache-control none --clock-control none -k regex:spmv_ --csv -c 120 \
  --log-file gpurun_out/ncu_rotate.csv python bench.py --steps 20 --warmup 3 --no-formats > gpurun_out/ncu_rotate.log 2>&1
tail -3 gpurun_out/ncu_rotate.log
