# GPU: the format-property sweep + the API tests (after engine changes)
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/sweep_smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_api.py -m gpu -q -rf -p no:cacheprovider > gpurun_out/sweep_pytest.log 2>&1
tail -60 gpurun_out/sweep_pytest.log
