timeout 900 python -m pytest tests/test_gpu_multipass.py -x -q -k "fused_ring" > gpurun_out/r5_multipass.log 2>&1; echo "multipass rc=$?" >> gpurun_out/r5_multipass.log
tail -5 gpurun_out/r5_multipass.log
(
timeout 300 python tools/fft4_time.py
SKG_ROWH_DBG=2 timeout 300 python tools/fft4_time.py
SKG_4STEP_DELTA_X10=15 timeout 300 python tools/fft4_time.py
) > gpurun_out/r5_fft4_time.log 2>&1
cat gpurun_out/r5_fft4_time.log
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k4_rfused -c 1 -o gpurun_out/r5_fused32 -f python tools/fft4_one.py f32 65536 4096 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k4_rfused -c 1 -o gpurun_out/r5_fused64 -f python tools/fft4_one.py f64 262144 1024 > /dev/null 2>&1
