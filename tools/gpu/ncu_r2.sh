# round-2 ncu evidence: the bench's launch list, one full capture per hot kernel
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_plain.json 2> gpurun_out/r2_bench_plain.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 1500 \
  --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_under_ncu.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"spmv_csr_handoff|spmv_ell|spmv_dia_kernel|coo_rowptr|add_tile|mttkrp_c" -c 14 \
  -o gpurun_out/r2_full python tools/prof_kernels.py --reps 1 --no-table --only coo,csr,ell,dia,add,mttkrp_coo,mttkrp_csf > gpurun_out/r2_full.log 2>&1
ls -la gpurun_out/r2_full.ncu-rep
