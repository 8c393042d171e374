# CZT A/B on the box: parity tests of the CZT paths, then cfg2 timing with each variant (+ optional ncu)
set -x
timeout 600 python -m pytest tests/test_gpu_czt.py tests/test_gpu_fullbatch.py -q -x -k "czt or cfg2" > gpurun_out/czt_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/czt_tests.log
for v in "" SKG_CZT_NO_TWT=1 SKG_CZT_NO_TM=1; do echo "== $v"; env $v timeout 120 python tools/czt_time.py 30; done
[ -n "$PROF" ] && TAG=${TAG:-r2a} CAPS="$PROF" NOLAUNCH=1 bash tools/gpu_prof.sh > gpurun_out/prof.log 2>&1
true
