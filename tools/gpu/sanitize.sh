# compute-sanitizer over the reduced-size GPU suite (no full-size tests)
export PYTHONDONTWRITEBYTECODE=1
timeout 2400 compute-sanitizer --tool memcheck --target-processes all --print-limit 200 \
  --log-file gpurun_out/r2_memcheck.log \
  python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/r2_memcheck_pytest.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/r2_memcheck_pytest.log
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report analysis --target-processes all --print-limit 200 \
  --log-file gpurun_out/r2_racecheck.log \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_convert.py tests/test_gpu_widen.py -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/r2_racecheck_pytest.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/r2_racecheck_pytest.log
timeout 1200 compute-sanitizer --tool synccheck --target-processes all --print-limit 200 \
  --log-file gpurun_out/r2_synccheck.log \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/r2_synccheck_pytest.log 2>&1
echo "synccheck rc=$?" >> gpurun_out/r2_synccheck_pytest.log
tail -3 gpurun_out/r2_*_pytest.log; grep -c "ERROR SUMMARY" gpurun_out/r2_memcheck.log; grep "ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/r2_*check.log | sort | uniq -c | head
