timeout 900 ncu --set full --import-source on --clock-control none -k regex:"add_tile" -c 2 \
  -o gpurun_out/add_full python tools/time_add.py 3 > gpurun_out/ncu_add_full.log 2>&1
