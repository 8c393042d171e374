timeout 1200 python -m pytest tests/test_gpu_multipass.py tests/test_gpu_guards.py tests/test_gpu_fft.py -x -q 2>&1 | tail -3
timeout 300 python tools/fft4_time.py
timeout 300 python tools/fft_long_time.py
