# zoom A/B on the box: parity tests of the zoom routes, then cfg3 timing per route (+ optional ncu)
set -x
timeout 900 python -m pytest tests/test_gpu_zoom.py tests/test_gpu_fullbatch.py tests/test_gpu_guards.py -q -x -k "zoom or cfg3" > gpurun_out/zoom_tests.log 2>&1; echo tests_rc=$?
tail -3 gpurun_out/zoom_tests.log
for v in "" SKG_ZOOM_NO_FUSE=1 SKG_ZOOM_NO_PCFIR=1; do echo "== $v"; env $v timeout 120 python tools/zoom_time.py 30; done
[ -n "$PROF" ] && TAG=${TAG:-r2b} CAPS="$PROF" NOLAUNCH=1 bash tools/gpu_prof.sh > gpurun_out/prof.log 2>&1
true
