# GPU: smoke + the whole GPU suite (+ the A/B build's parity tests)
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/full_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/full_pytest.log 2>&1
SL_LIB_PATH=paper_1804_10112_b200/_lib/alt/libsl_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider > gpurun_out/full_pytest_alt.log 2>&1
tail -3 gpurun_out/full_pytest.log gpurun_out/full_pytest_alt.log
tail -2 gpurun_out/full_smoke.log
