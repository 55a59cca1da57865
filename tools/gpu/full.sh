# GPU: smoke + the whole GPU suite
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/full_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/full_pytest.log 2>&1
tail -30 gpurun_out/full_pytest.log
tail -2 gpurun_out/full_smoke.log
