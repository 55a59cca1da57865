# GPU: bench (driver-style K=20 and default), reference arm
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
timeout 600 python bench.py > gpurun_out/bench_def.json 2> gpurun_out/bench_def.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -5 gpurun_out/*.err
