timeout 900 python -m pytest tests/test_gpu_multipass.py -x -q -k "real_fourstep" 2>&1 | tail -2
timeout 300 python tools/fft4_time.py
