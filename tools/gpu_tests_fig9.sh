# (GPU box) full gpu test suite, cube timing and the Fig. 9 sweep
# full GPU gate + timing helpers + the Fig. 9 sweep
timeout 1300 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest_rc=$?; tail -4 gpurun_out/pytest_gpu_full.log
timeout 300 python tools/cube_time.py 10
timeout 900 python tools/fig9_sweep.py gpurun_out/fig9_sweep.json > gpurun_out/fig9.log 2>&1; echo fig9_rc=$?; tail -3 gpurun_out/fig9.log
