for m in 1.5 4 8; do
  SL_BENCH_L2_MARGIN=$m timeout 600 python bench.py --steps 100 --no-formats > gpurun_out/bench_m$m.json 2>&1
done
SL_BENCH_L2_MARGIN=8 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --cache-control none --clock-control none -k regex:spmv_ --csv -c 100 \
  --log-file gpurun_out/ncu_rotate_m8.csv python bench.py --steps 20 --warmup 3 --no-formats > /dev/null 2>&1
