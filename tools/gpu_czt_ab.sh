# CZT A/B on the box: parity tests of the CZT paths, then cfg2 timing with each variant
set -x
timeout 600 python -m pytest tests/test_gpu_czt.py tests/test_gpu_fullbatch.py -q -x -k "czt or cfg2" > gpurun_out/czt_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/czt_tests.log
timeout 120 python tools/czt_time.py 30
SKG_CZT_NO_TM=1 timeout 120 python tools/czt_time.py 30
