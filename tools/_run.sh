timeout 1200 python -m pytest tests/test_gpu_zoom.py -x -q 2>&1 | tail -3
timeout 1200 python tools/sweep.py --kinds zoom --precs f64 --ns 65536 --out gpurun_out/r11_sweep_zoom64.json 2>&1 | tail -3 | cut -c1-250
