SL_COO_KERNEL=tile timeout 900 ncu --set full --import-source on --clock-control none -k regex:"spmv_coo_kernel" -c 1 \
  -o gpurun_out/coo_tile python tools/time_coo.py 2 > gpurun_out/ncu_coo.log 2>&1
